"""K1/K7 scene staging: float scenes with whole 16-B SH rows stage each CTA's
primitives with bulk copies (cp.async.bulk on an mbarrier), everything else with
per-thread cp.async.  The two paths must be indistinguishable: the same scene
with every field 4 bytes off 16-B alignment (all CTAs on the cp.async path) gives
bit-identical frames, images and gradients, for one view, for accumulation and for
the multi-view passes."""

import numpy as np
import pytest
import torch

from paper_2406_02720_b200 import device, multiview, scenes
from paper_2406_02720_b200.geometry import CameraModel, Scene

pytestmark = pytest.mark.gpu


def _misaligned(t):
    """The same values in a buffer whose first element sits 4 bytes past 16-B
    alignment (contiguous, so Scene keeps it as is)."""
    flat = torch.empty(t.numel() + 1, dtype=t.dtype, device=t.device)
    out = flat[1:].view(t.shape)
    out.copy_(t)
    assert out.data_ptr() % 16 != 0 and out.is_contiguous()
    return out


def _scenes(sa):
    sc = Scene(*(getattr(sa, f) for f in sa.FIELDS), sh_degree=sa.sh_degree,
               background_color=sa.background_color, device="cuda", dtype=torch.float32)
    fields = [_misaligned(getattr(sc, f)) for f in sa.FIELDS]
    mis = Scene(*fields, sh_degree=sa.sh_degree, background_color=sa.background_color,
                device="cuda", dtype=torch.float32)
    for f in sa.FIELDS:
        assert getattr(mis, f).data_ptr() % 16 != 0, f
    return sc, mis


def _grads_equal(a, b):
    for name in device.DeviceGradientSet.NAMES:
        assert torch.equal(getattr(a, name), getattr(b, name)), name


# n: whole CTAs only (1024), a tail that is a multiple of 4 primitives (1000: its
# CTA also bulk-copies), a tail that is not (1001: cp.async for that CTA)
@pytest.mark.parametrize("n", [1024, 1000, 1001])
@pytest.mark.parametrize("deg", [1, 3])
def test_bulk_and_cp_async_staging_agree(cuda, n, deg):
    sa = scenes.frustum(n, deg, 96, 64, seed=21 + n + deg)
    cam = CameraModel(**sa.cameras[0])
    sc, mis = _scenes(sa)
    d = torch.as_tensor(scenes.cotangent(cam.height, cam.width), dtype=torch.float32,
                        device="cuda")
    outs, grads = [], []
    for s in (sc, mis):
        out = device.render(s, cam)
        g = device.render_backward(s, cam, out, d)
        device.render_backward(s, cam, out, d, grads=g, accumulate=True)  # K7 mode 1
        outs.append(out)
        grads.append(g)
    a, b = outs
    assert a.frame.num_pairs > 0
    ea, eb = a.frame.export(), b.frame.export()
    for k in ea:
        assert np.array_equal(np.asarray(ea[k]), np.asarray(eb[k])), k
    for name in ("color", "alpha", "depth", "transmittance", "terminal", "radii"):
        assert torch.equal(getattr(a, name), getattr(b, name)), name
    _grads_equal(*grads)


def test_bulk_and_cp_async_staging_agree_views(cuda):
    """The multi-view K1 and K7 (ViewBatch) on both staging paths."""
    sa = scenes.ball(1536, 3, 64, 48, views=3, seed=9)
    cams = [CameraModel(**c) for c in sa.cameras]
    ds = [torch.as_tensor(scenes.cotangent(c.height, c.width, seed=3 + v), dtype=torch.float32,
                          device="cuda") for v, c in enumerate(cams)]
    res = []
    for s in _scenes(sa):
        g = device.DeviceGradientSet.empty_like_scene(s)
        multiview.ViewBatch(s, len(cams)).run(s, cams, ds, list(range(len(cams))), g)
        res.append(g)
    _grads_equal(*res)
