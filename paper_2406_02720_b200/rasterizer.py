"""Drop-in replacement for ``halfsplat.rasterizer`` running on the B200.

Same functions, argument meaning, return types and exceptions as the reference
module (rasterizer.py:43-642): host numpy in, host numpy out.  Every call goes
through the device pipeline in ``device.py`` (libhalfsplat_b200.so); host
buffers are copied to HBM on entry and results copied back on exit, so this is
the end-to-end path a reference caller gets by switching imports.

float64 reference scenes are uploaded as float64 (the FP64 preprocess then sees
exactly the reference's inputs); float32 scenes stay float32.  The blend runs in
FP32; see DESIGN.md for the parity contract.

Outputs have the reference's dtypes by default: float64 images and gradients,
int32 terminal indices, int64 touch counts (rasterizer.py:357-361, 400;
GradientSet.zeros 85-97).  `set_output_dtype(np.float32)` (or HS_HOST_FLOAT=float32)
is an explicit opt-in that returns the images as the FP32 the blend computes and
the gradients in the scene's own dtype, halving the bytes that cross PCIe.
"""

import ctypes
import os
import weakref
from dataclasses import dataclass

import numpy as np
import torch

from . import device as _dev
from .errors import EmptyScene, ImageTooLarge, MismatchedForward  # noqa: F401  (re-export)
from .geometry import CameraModel, Scene

TILE = 16
RADIUS_SIGMAS = 3.5
MAX_PIXELS = 2**31


@dataclass
class ScreenSplat:
    """One primitive projected into one view (rasterizer.py:43-56)."""

    prim_index: int
    mu_hat: np.ndarray
    conic: np.ndarray
    whiten2d: np.ndarray
    n_ray: np.ndarray
    alpha1: float
    alpha2: float
    rgb: np.ndarray
    depth: float
    tile_span: tuple  # (tx0, tx1, ty0, ty1), inclusive


@dataclass
class RenderOutput:
    """Forward-pass result (rasterizer.py:59-69)."""

    color: np.ndarray
    alpha: np.ndarray
    depth: np.ndarray
    per_pixel_terminal_index: np.ndarray
    camera: object = None
    transmittance: np.ndarray = None
    frame: object = None
    radii: np.ndarray = None


@dataclass
class GradientSet:
    """Per-primitive gradients, index-aligned with the scene (rasterizer.py:72-105)."""

    d_mu: np.ndarray
    d_log_scale: np.ndarray
    d_rotation: np.ndarray
    d_sh: np.ndarray
    d_normal: np.ndarray
    d_raw_opacity_a: np.ndarray
    d_raw_opacity_b: np.ndarray
    pos_grad_norm: np.ndarray
    touch_count: np.ndarray

    NAMES = ("d_mu", "d_log_scale", "d_rotation", "d_sh", "d_normal", "d_raw_opacity_a",
             "d_raw_opacity_b", "pos_grad_norm", "touch_count")

    @classmethod
    def zeros(cls, n, sh_k):
        return cls(d_mu=np.zeros((n, 3)), d_log_scale=np.zeros((n, 3)),
                   d_rotation=np.zeros((n, 4)), d_sh=np.zeros((n, sh_k, 3)),
                   d_normal=np.zeros((n, 3)), d_raw_opacity_a=np.zeros(n),
                   d_raw_opacity_b=np.zeros(n), pos_grad_norm=np.zeros(n),
                   touch_count=np.zeros(n, dtype=np.int64))

    def add(self, other):
        for name in self.NAMES:
            getattr(self, name).__iadd__(getattr(other, name))
        return self


class FrameGeometry:
    """Binned view (rasterizer.py:108-147).  The device frame does the work; the
    reference's integer arrays and packed columns are materialised on first
    access (they are parity observables, not needed to render)."""

    def __init__(self, dframe, dscene, kernel):
        self._device = dframe
        self._scene = dscene
        self.kernel = kernel
        self.n_total = dframe.n_total
        self.tiles_x = dframe.tiles_x
        self.tiles_y = dframe.tiles_y
        self._export = None

    def _exported(self):
        if self._export is None:
            self._export = self._device.export()
        return self._export

    @property
    def valid(self):
        return self._exported()["valid"]

    @property
    def packed(self):
        return self._exported()["packed"].astype(np.float64)

    @property
    def mode(self):
        return self._exported()["mode"]

    @property
    def pair_splat(self):
        return self._exported()["pair_splat"]

    @property
    def tile_starts(self):
        return self._exported()["tile_starts"]

    @property
    def tile_rect(self):
        return self._exported()["tile_rect"]

    @property
    def radii(self):
        return self._exported()["radii"]


def _n(scene):
    return int(scene.mu.shape[0])


# Host dtype of the floating-point outputs: the reference's float64 unless the
# caller opts into float32 (module docstring).
_OUTPUT_DTYPE = [np.float32 if os.environ.get("HS_HOST_FLOAT") == "float32" else np.float64]


def set_output_dtype(dtype):
    """np.float64 (default, the reference's dtypes) or np.float32 (opt-in: images
    as computed in FP32, gradients in the scene's dtype).  Returns the previous one."""
    dtype = np.dtype(dtype).type
    if dtype not in (np.float32, np.float64):
        raise ValueError("output dtype must be float32 or float64")
    prev, _OUTPUT_DTYPE[0] = _OUTPUT_DTYPE[0], dtype
    return prev


def output_dtype():
    return _OUTPUT_DTYPE[0]


def _host_float_dtype(t):
    """torch dtype a floating device tensor is returned in."""
    if _OUTPUT_DTYPE[0] is np.float64:
        return torch.float64
    return t.dtype


def _to_host(tensors):
    """D2H through pinned staging buffers (one sync for the whole batch).  Float
    tensors are widened on the device when float64 is requested, so the host
    gets the reference's dtype without a host-side conversion pass."""
    staged = []
    for t in tensors:
        if t.is_floating_point() and t.dtype != _host_float_dtype(t):
            t = t.to(_host_float_dtype(t))
        h = torch.empty(t.shape, dtype=t.dtype, pin_memory=True)
        h.copy_(t, non_blocking=True)
        staged.append(h)
    torch.cuda.current_stream().synchronize()
    return [h.numpy() for h in staged]


def resolve_threads(threads):
    """Accepted for signature compatibility (rasterizer.py:150-156); the GPU ignores it."""
    return 1 if threads is None else max(1, int(threads))


class _WorkspacePool:
    """Device workspaces recycled across calls.  A FrameGeometry owns one until it
    is garbage collected, so a frame kept for a later render_backward is never
    overwritten, while a plain render -> render_backward loop reuses the same
    buffers every iteration (no cudaMalloc/cudaFree in steady state)."""

    def __init__(self, keep=2):
        self.keep = keep
        self.free = {}

    def acquire(self, device):
        lst = self.free.setdefault(str(device), [])
        return lst.pop() if lst else _dev.Workspace(device)

    def release(self, device, ws):
        lst = self.free.setdefault(str(device), [])
        if len(lst) < self.keep:
            lst.append(ws)


_POOL = _WorkspacePool()


def prepare(scene, cam, kernel="half"):
    """Project a scene into one view; returns FrameGeometry (rasterizer.py:159)."""
    dscene = Scene.from_any(scene)
    ws = _POOL.acquire(dscene.device)
    dframe = _dev.prepare(dscene, cam, kernel, ws=ws)
    fg = FrameGeometry(dframe, dscene, kernel)
    fg._ws = ws
    fg._ws_gen = [0]  # renders issued into this workspace
    weakref.finalize(fg, _POOL.release, dscene.device, ws)
    return fg


def render(scene, cam, kernel="half", threads=None, frame=None):
    """Render one view (rasterizer.py:351).  Deterministic for any launch config."""
    resolve_threads(threads)
    cam = CameraModel.from_any(cam)
    if frame is None:
        frame = prepare(scene, cam, kernel)
    dscene = frame._scene
    dout = _dev.render(dscene, cam, kernel, frame=frame._device, ws=frame._ws)
    frame._ws_gen[0] += 1
    color, alpha, depth, trans, term, radii = _to_host(
        [dout.color, dout.alpha, dout.depth, dout.transmittance, dout.terminal, dout.radii])
    if frame._device.resolve():
        # the view was binned with P on the device and overflowed its workspace's pair
        # capacity; resolve() re-binned it with a larger one: blend it again
        dout = _dev.render(dscene, cam, kernel, frame=frame._device, ws=frame._ws)
        color, alpha, depth, trans, term, radii = _to_host(
            [dout.color, dout.alpha, dout.depth, dout.transmittance, dout.terminal, dout.radii])
    out = RenderOutput(color=color, alpha=alpha, depth=depth, per_pixel_terminal_index=term,
                       camera=cam, transmittance=trans, frame=frame, radii=radii)
    out._device_out = dout
    out._gen = frame._ws_gen[0]
    out._host_scene = scene
    return out


def render_backward(scene, cam, out, d_color, threads=None):
    """Gradients of sum(d_color * rendered color) for every parameter (rasterizer.py:386)."""
    resolve_threads(threads)
    cam = CameraModel.from_any(cam)
    frame = out.frame
    if frame is None or frame.n_total != _n(scene):
        raise MismatchedForward("forward bookkeeping does not match the scene")
    d_color = np.asarray(d_color)
    if d_color.shape != (cam.height, cam.width, 3):
        raise MismatchedForward(f"cotangent shape {d_color.shape} != {(cam.height, cam.width, 3)}")
    if np.shape(out.per_pixel_terminal_index) != (cam.height, cam.width):
        raise MismatchedForward("terminal-index shape mismatch")
    dout = getattr(out, "_device_out", None)
    if dout is not None and getattr(out, "_gen", None) != frame._ws_gen[0]:
        dout = None  # the frame was rendered again since: its device buffers moved on
    dscene = frame._scene if getattr(out, "_host_scene", None) is scene else Scene.from_any(scene)
    if dout is None:
        # a RenderOutput assembled by the caller: upload its bookkeeping
        dev = dscene.device
        dout = _dev.DeviceRenderOutput(
            color=None, alpha=None, depth=None,
            transmittance=torch.as_tensor(np.asarray(out.transmittance, np.float32), device=dev),
            terminal=torch.as_tensor(np.asarray(out.per_pixel_terminal_index, np.int32),
                                     device=dev),
            radii=frame._device.radii, frame=frame._device, camera=cam)
    dc = _upload_f32(d_color, dscene.device)
    return GradientSet(*_backward_to_host(dscene, cam, dout, dc))


def _upload_f32(a, device):
    """Host array -> device float32.  The conversion runs on the host into a pinned
    staging buffer (torch's threaded copy, ~0.3 ms for a 1080p f64 cotangent) and
    the upload is one async DMA at the pinned rate: a pageable float64 upload moves
    twice the bytes at a third of the rate (B200 box: 19 vs 55 GB/s).  Rounding is
    the same round-to-nearest as converting on the device."""
    src = a if isinstance(a, torch.Tensor) else torch.as_tensor(np.ascontiguousarray(a))
    if src.dtype == torch.float32 and src.is_pinned():
        return src.to(device, non_blocking=True)
    stage = torch.empty(src.shape, dtype=torch.float32, pin_memory=True)
    dst = torch.empty(src.shape, dtype=torch.float32, device=device)
    # in row chunks, so the DMA of one chunk overlaps the conversion of the next
    rows = src.shape[0] if src.dim() else 1
    step = max(1, -(-rows // UPLOAD_CHUNKS))
    for r in range(0, rows, step):
        stage[r:r + step].copy_(src[r:r + step])
        dst[r:r + step].copy_(stage[r:r + step], non_blocking=True)
    return dst


# row chunks of the host-side conversion + upload in _upload_f32
UPLOAD_CHUNKS = 4


# K7 runs in this many primitive buckets on the drop-in path, so the D2H of each
# bucket's gradient rows overlaps the next bucket's K7.
D2H_BUCKETS = 4


def _backward_to_host(dscene, cam, dout, dc):
    """render_backward with the gradient download overlapped with K7: after each
    primitive bucket a side stream copies that bucket's rows of every field into
    pinned host arrays (touch counts widened to int64 on the device first, and the
    float fields to float64 when the reference's dtype is requested)."""
    n = len(dscene)
    dev = dscene.device
    grads = _dev.DeviceGradientSet.empty_like_scene(dscene)
    touch64 = torch.empty(n, dtype=torch.int64, device=dev)
    src = [getattr(grads, name) for name in GradientSet.NAMES[:-1]]
    fields = [t if t.dtype == _host_float_dtype(t) else
              torch.empty(t.shape, dtype=_host_float_dtype(t), device=dev) for t in src]
    widen = [(a, b) for a, b in zip(src, fields) if a is not b]
    fields.append(touch64)
    host = [torch.empty(t.shape, dtype=t.dtype, pin_memory=True) for t in fields]
    compute = torch.cuda.current_stream(dev)
    copy = _copy_stream(dev)
    nb = max(1, min(D2H_BUCKETS, n))
    # bucket starts on the 128-primitive K7 CTA grid (hs_preprocess_bwd_range)
    edges = [min(n, (n * i // nb + 127) // 128 * 128) for i in range(nb)] + [n]
    buckets = [(edges[i], edges[i + 1]) for i in range(nb) if edges[i + 1] > edges[i]]

    def on_bucket(b, e):
        touch64[b:e].copy_(grads.touch_count[b:e])
        for a, w in widen:
            w[b:e].copy_(a[b:e])
        ev = torch.cuda.Event()
        ev.record(compute)
        copy.wait_event(ev)
        with torch.cuda.stream(copy):
            for h, t in zip(host, fields):
                h[b:e].copy_(t[b:e], non_blocking=True)

    _dev.render_backward(dscene, cam, dout, dc, grads=grads, buckets=buckets,
                         on_bucket=on_bucket)
    copy.synchronize()  # before the device buffers go back to the allocator
    return [h.numpy() for h in host]


_COPY_STREAMS = {}


def _copy_stream(dev):
    key = torch.device(dev).index
    if key is None:
        key = torch.cuda.current_device()
    if key not in _COPY_STREAMS:
        _COPY_STREAMS[key] = torch.cuda.Stream(device=key)
    return _COPY_STREAMS[key]


def screen_splats(scene, cam, kernel="half"):
    """Per-primitive projected splats for one view (rasterizer.py:578-603)."""
    cam = CameraModel.from_any(cam)
    frame = prepare(scene, cam, kernel)
    ex = frame._exported()
    dscene = frame._scene
    vals = torch.empty((len(dscene), 20), dtype=torch.float64, device=dscene.device)
    lib = _dev._native.load()
    _dev._native.check(lib.hs_screen_splats(
        ctypes.byref(_dev.scene_struct(dscene)), ctypes.byref(_dev.camera_struct(cam)),
        0 if kernel == "half" else 1, _dev._ptr(vals), _dev._stream()), "hs_screen_splats")
    vals = vals.cpu().numpy()
    out = []
    for i, prim in enumerate(ex["valid"]):
        v = vals[prim]
        out.append(ScreenSplat(
            prim_index=int(prim), mu_hat=v[0:2].copy(),
            conic=np.array([[v[2], v[3]], [v[3], v[4]]]),
            whiten2d=np.array([[v[5], 0.0], [v[6], v[7]]]), n_ray=v[8:11].copy(),
            alpha1=float(v[11]), alpha2=float(v[12]), rgb=v[13:16].copy(), depth=float(v[16]),
            tile_span=tuple(int(x) for x in ex["tile_rect"][i])))
    return out


def render_depth_normalmap(out, alpha_threshold=0.5):
    """Per-pixel normals from screen-space depth differences (rasterizer.py:606-642).

    Post-processing of a rendered depth map, evaluated with torch ops on the
    render's device."""
    cam = out.camera
    dev = torch.device("cuda") if torch.cuda.is_available() else torch.device("cpu")
    depth = torch.as_tensor(np.asarray(out.depth, dtype=np.float64), device=dev)
    alpha = torch.as_tensor(np.asarray(out.alpha, dtype=np.float64), device=dev)
    h, w = depth.shape
    ys, xs = torch.meshgrid(torch.arange(h, device=dev, dtype=torch.float64),
                            torch.arange(w, device=dev, dtype=torch.float64), indexing="ij")
    pts = torch.stack([depth * (xs + 0.5 - cam.cx) / cam.fx,
                       depth * (ys + 0.5 - cam.cy) / cam.fy, depth], dim=-1)
    valid = alpha >= alpha_threshold
    normals = torch.zeros((h, w, 3), dtype=torch.float64, device=dev)
    if h >= 3 and w >= 3:
        dx = pts[1:-1, 2:] - pts[1:-1, :-2]
        dy = pts[2:, 1:-1] - pts[:-2, 1:-1]
        ok = (valid[1:-1, 1:-1] & valid[1:-1, 2:] & valid[1:-1, :-2] & valid[2:, 1:-1]
              & valid[:-2, 1:-1])
        cross = torch.linalg.cross(dx, dy, dim=-1)
        norm = torch.linalg.norm(cross, dim=-1)
        ok &= norm > 1e-12
        safe = torch.where(norm > 1e-12, norm, torch.ones_like(norm))
        cross = torch.where(ok[..., None], cross / safe[..., None], torch.zeros_like(cross))
        flip = cross[..., 2] > 0
        cross = torch.where(flip[..., None], -cross, cross)
        normals[1:-1, 1:-1] = cross
    return normals.cpu().numpy()
