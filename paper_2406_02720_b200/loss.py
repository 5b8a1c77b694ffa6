"""Training loss on the GPU: (1 - lambda) L1 + lambda (1 - SSIM) and its exact
gradient, the cotangent d_color that the backward blend consumes.

Drop-in for the reference's `halfsplat.loss` (loss.py:1-106): the same names,
argument meaning, return types and errors (`ShapeMismatch`, `ImageTooSmall`,
`ValueError` for lambda outside [0, 1]).  The host functions take numpy images
and return float64 numpy gradients like the reference; `DeviceLoss` is the
allocation-free form for device-resident training loops (torch CUDA tensors in,
loss scalars and the float32 cotangent out, no host synchronisation).

All arithmetic runs in `hs_loss` (csrc/hs_loss.cu) in FP64; float32 images are
read as float32 (exact in FP64), anything else as float64 (`hs_loss_f64`), so a
reference caller's float64 renders and uint8/255 targets are not rounded.
There is no CPU path.
"""

import ctypes

import numpy as np
import torch

from . import _native, errors

SSIM_WINDOW = 11    # loss.py:13
SSIM_SIGMA = 1.5    # loss.py:14
SSIM_C1 = 0.01**2   # loss.py:15
SSIM_C2 = 0.03**2   # loss.py:16


def _stream():
    return ctypes.c_void_p(torch.cuda.current_stream().cuda_stream)


def _ptr(t):
    return ctypes.c_void_p(t.data_ptr()) if t is not None else None


class DeviceLoss:
    """compute_loss on device tensors with a persistent workspace.

    `__call__(rendered, target)` takes (H,W,C) or (H,W) CUDA tensors (float32,
    or float64 when either is float64: then both are read as float64) and returns `(stats, d_rendered)`: stats is a (4,) float64 device tensor
    [loss, L1, mean SSIM, MSE] and d_rendered the float32 gradient, shaped like
    `rendered`.  Nothing is copied to the host.
    """

    def __init__(self, lambda_ssim=0.2):
        if not 0.0 <= lambda_ssim <= 1.0:
            raise ValueError("lambda_ssim must lie in [0, 1]")
        self.lambda_ssim = float(lambda_ssim)
        self._ws = None
        self._shape = None

    def _workspace(self, h, w, c, device):
        if self._shape != (h, w, c, device) or self._ws is None:
            nbytes = _native.load().hs_loss_workspace_size(h, w, c)
            self._ws = torch.empty(max(nbytes, 1), dtype=torch.uint8, device=device)
            self._shape = (h, w, c, device)
        return self._ws

    def __call__(self, rendered, target, d_out=None, stats=None, d_out_f64=None):
        if rendered.shape != target.shape:
            raise errors.ShapeMismatch(f"{tuple(rendered.shape)} vs {tuple(target.shape)}")
        if rendered.dim() not in (2, 3):
            raise errors.ShapeMismatch("expected HxW or HxWxC images")
        if not (rendered.is_cuda and target.is_cuda):
            raise ValueError("DeviceLoss takes CUDA tensors")
        f64 = torch.float64 in (rendered.dtype, target.dtype)
        x = rendered.contiguous().to(torch.float64 if f64 else torch.float32)
        y = target.contiguous().to(x.dtype)
        h, w = x.shape[0], x.shape[1]
        c = x.shape[2] if x.dim() == 3 else 1
        if stats is None:
            stats = torch.empty(4, dtype=torch.float64, device=x.device)
        if d_out is None and d_out_f64 is None:
            d_out = torch.empty(x.shape, dtype=torch.float32, device=x.device)
        ws = self._workspace(h, w, c, x.device)
        lib = _native.load()
        fn = lib.hs_loss_f64 if f64 else lib.hs_loss
        _native.check(fn(_ptr(x), _ptr(y), h, w, c, self.lambda_ssim, _ptr(stats),
                         _ptr(d_out), _ptr(d_out_f64), _ptr(ws), ws.numel(), _stream()),
                      "hs_loss")
        return stats, (d_out if d_out is not None else d_out_f64)


def _check_pair(a, b):
    """loss.py:35-45.  Two float32 arrays stay float32 (exact in the FP64 kernel);
    anything else is read as float64, as the reference's np.asarray(.., float64)."""
    a = np.asarray(a)
    b = np.asarray(b)
    dt = np.float32 if a.dtype == np.float32 and b.dtype == np.float32 else np.float64
    a = np.ascontiguousarray(a, dtype=dt)
    b = np.ascontiguousarray(b, dtype=dt)
    if a.shape != b.shape:
        raise errors.ShapeMismatch(f"{a.shape} vs {b.shape}")
    if a.ndim not in (2, 3):
        raise errors.ShapeMismatch("expected HxW or HxWxC images")
    return a, b


def _run(rendered, target, lambda_ssim):
    a, b = _check_pair(rendered, target)
    if not 0.0 <= lambda_ssim <= 1.0:
        raise ValueError("lambda_ssim must lie in [0, 1]")
    if lambda_ssim != 0.0 and min(a.shape[0], a.shape[1]) < SSIM_WINDOW:
        raise errors.ImageTooSmall(f"needs at least {SSIM_WINDOW} pixels on each side")
    dev = torch.device("cuda", torch.cuda.current_device())
    x = torch.from_numpy(a).to(dev)
    y = torch.from_numpy(b).to(dev)
    d64 = torch.empty(x.shape, dtype=torch.float64, device=dev)
    stats, _ = DeviceLoss(lambda_ssim)(x, y, d_out=None, d_out_f64=d64)
    return stats.cpu().numpy(), d64.cpu().numpy()


def ssim_with_grad(a, b):
    """Mean SSIM of a against b and d(mean SSIM)/da (loss.py:48-79)."""
    stats, d = _run(a, b, 1.0)
    if d.ndim == 2:  # the reference returns (H,W,1) for 2-D images (loss.py:40-42, 55)
        d = d[..., None]
    # lambda 1: gradient = 0 * d_l1 - s_grad, exactly -s_grad
    return float(stats[2]), -d


def ssim(a, b):
    """Mean SSIM in [-1, 1]; exactly 1.0 for identical images (loss.py:82-85)."""
    value, _ = ssim_with_grad(a, b)
    return value


def compute_loss(rendered, target, lambda_ssim=0.2):
    """Loss scalar plus its exact gradient w.r.t. the rendered image (loss.py:88-106)."""
    stats, d = _run(rendered, target, lambda_ssim)
    return float(stats[0]), d
