"""The multi-view geometry backward (hs_merge_rows + hs_preprocess_bwd_views,
multiview.ViewBatch): one pass over the scene for a batch of views must give the
same gradients, bit for bit, as K7 per view accumulating in view order
(GradientSet.add, rasterizer.py:100-105)."""

import numpy as np
import pytest
import torch

from paper_2406_02720_b200 import device, errors, multiview, scenes
from paper_2406_02720_b200.geometry import CameraModel, Scene

pytestmark = pytest.mark.gpu


def _setup(n, deg, views, dtype, seed=5, w=96, h=80):
    sa = scenes.ball(n, deg, w, h, views=views, seed=seed)
    sc = Scene(*(getattr(sa, f) for f in sa.FIELDS), sh_degree=sa.sh_degree,
               background_color=sa.background_color, device="cuda", dtype=dtype)
    cams = [CameraModel(**c) for c in sa.cameras]
    dcs = [torch.as_tensor(scenes.cotangent(h, w, seed=10 + v), dtype=torch.float32,
                           device="cuda") for v in range(views)]
    return sc, cams, dcs


def test_prepare_views_equals_prepare(cuda):
    """One K1 pass for several views (hs_preprocess_fwd_views): every frame's
    integers, packed columns and radii equal prepare()'s, bit for bit."""
    sc, cams, _ = _setup(4000, 3, 5, torch.float32, seed=12)
    wss = [device.Workspace("cuda") for _ in range(5)]
    frames = device.prepare_views(sc, cams, workspaces=wss)
    for v, fr in enumerate(frames):
        ref = device.prepare(sc, cams[v])
        got, exp = fr.export(), ref.export()
        for k in exp:
            assert np.array_equal(np.asarray(got[k]), np.asarray(exp[k])), (v, k)
        assert torch.equal(fr.radii, ref.radii), v
    # K1 alone, then each frame ranked and binned on its own stream
    streams = [torch.cuda.Stream() for _ in range(5)]
    frames = device.prepare_views(sc, cams, workspaces=wss, bin=False)
    ready = torch.cuda.Event()
    ready.record()
    binned = []
    for v, fr in enumerate(frames):
        streams[v].wait_event(ready)
        with torch.cuda.stream(streams[v]):
            binned.append(device.bin_frame(fr, wss[v]))
    for st in streams:
        torch.cuda.current_stream().wait_stream(st)
    for v, fr in enumerate(binned):
        got, exp = fr.export(), device.prepare(sc, cams[v]).export()
        for k in exp:
            assert np.array_equal(np.asarray(got[k]), np.asarray(exp[k])), (v, k)
    with pytest.raises(ValueError):
        device.prepare_views(sc, cams[:2], workspaces=[wss[0], wss[0]])


def _per_view(sc, cams, dcs, ids, kernel="half"):
    rast = device.Rasterizer("cuda", kernel=kernel)
    g = device.DeviceGradientSet.empty_flat(sc)
    for j, v in enumerate(ids):
        out = rast.render(sc, cams[v])
        rast.render_backward(sc, cams[v], out, dcs[v], grads=g, accumulate=j > 0)
    return g


def _same(a, b, tiny=0.0):
    # equal values (a 0 + (-0) sum may differ in the sign of zero only); `tiny`:
    # float atomics flush subnormal addends to zero
    if not a.is_floating_point():
        return torch.equal(a, b)
    bad = (a.double() - b.double()).abs() > tiny
    if bad.any():
        print("mismatches", int(bad.sum()), "of", a.numel(), "max |diff|",
              float((a.double() - b.double()).abs().max()))
    return not bool(bad.any())


@pytest.mark.parametrize("dtype", [torch.float32, torch.float64])
@pytest.mark.parametrize("deg", [0, 3])
def test_view_batch_equals_per_view_k7(cuda, dtype, deg):
    sc, cams, dcs = _setup(4000, deg, 4, dtype)
    ids = [0, 1, 2, 3]
    ref = _per_view(sc, cams, dcs, ids)
    vb = multiview.ViewBatch(sc, len(ids))
    got = multiview.batch_gradients(sc, cams, dcs, ids, batch=vb)
    for name in device.DeviceGradientSet.NAMES:
        assert _same(getattr(ref, name), getattr(got, name)), name
    assert int(got.touch_count.max()) <= 4 and int(got.touch_count.sum()) > 0


def test_view_batch_more_views_than_one_launch(cuda):
    """11 views: two launches (8 + 3), the second adding into the first's output."""
    sc, cams, dcs = _setup(3000, 2, 11, torch.float32, seed=6, w=64, h=48)
    ids = list(range(11))
    ref = _per_view(sc, cams, dcs, ids)
    got = multiview.batch_gradients(sc, cams, dcs, ids, batch=multiview.ViewBatch(sc, 11))
    for name in device.DeviceGradientSet.NAMES:
        assert _same(getattr(ref, name), getattr(got, name)), name


@pytest.mark.parametrize("shared_k1", [True, False])
def test_view_batch_full_kernel_and_subset(cuda, shared_k1):
    sc, cams, dcs = _setup(3000, 1, 5, torch.float32, seed=7)
    ids = [4, 1, 3]
    ref = _per_view(sc, cams, dcs, ids, kernel="full")
    vb = multiview.ViewBatch(sc, 5, rast=device.Rasterizer("cuda", kernel="full"),
                             shared_k1=shared_k1)
    got = multiview.batch_gradients(sc, cams, dcs, ids, batch=vb)
    for name in device.DeviceGradientSet.NAMES:
        assert _same(getattr(ref, name), getattr(got, name)), name


def test_view_batch_buckets_and_reduction_stores(cuda):
    """Primitive buckets (each launch over [b, e)) and device-atomic reduction stores
    into zeroed buffers both give the single-launch result (the atomics up to
    flushed subnormals)."""
    sc, cams, dcs = _setup(5000, 3, 3, torch.float32, seed=8)
    ids = [0, 1, 2]
    vb = multiview.ViewBatch(sc, 3)
    one = vb.run(sc, cams, dcs, ids, device.DeviceGradientSet.empty_flat(sc))
    one = {k: getattr(one, k).clone() for k in device.DeviceGradientSet.NAMES}
    calls = []
    bk = vb.run(sc, cams, dcs, ids, device.DeviceGradientSet.empty_flat(sc),
                buckets=multiview.GradientAllReduce.bucket_ranges(len(sc), buckets=3),
                on_bucket=lambda b, e: calls.append((b, e)))
    assert len(calls) == 3 and calls[-1][1] == len(sc)
    red = device.DeviceGradientSet.empty_flat(sc)
    red.flat.zero_()
    red.touch_count.zero_()
    ptrs = {k: getattr(red, k).data_ptr() for k in device.DeviceGradientSet.NAMES}
    ptrs["mode"] = 2
    vb.run(sc, cams, dcs, ids, red, reduce_ptrs=ptrs)
    torch.cuda.synchronize()
    for name in device.DeviceGradientSet.NAMES:
        assert _same(one[name], getattr(bk, name)), name
        assert _same(one[name], getattr(red, name), 2 * torch.finfo(torch.float32).tiny), name


def test_view_batch_rejects_bad_rows(cuda):
    sc, cams, dcs = _setup(1000, 0, 2, torch.float32, seed=9)
    bad = [torch.zeros((len(sc), 8), device="cuda")] * 2
    with pytest.raises(errors.MismatchedForward):
        device.geometry_backward_views(sc, cams, bad)
    with pytest.raises(ValueError):
        device.geometry_backward_views(sc, cams, bad[:1])


def test_view_batch_repeated_steps_on_streams(cuda):
    """Steady state: the same ViewBatch run step after step (the views' workspaces
    then bin asynchronously, each on its stream) keeps giving the per-view result,
    also for a different subset of views and after the scene changes."""
    sc, cams, dcs = _setup(4000, 2, 6, torch.float32, seed=14)
    vb = multiview.ViewBatch(sc, 6)
    assert len(vb.streams) == 6
    ids = [0, 2, 3, 5]
    ref = _per_view(sc, cams, dcs, ids)
    for _ in range(3):
        got = multiview.batch_gradients(sc, cams, dcs, ids, batch=vb)
        torch.cuda.synchronize()
        for name in device.DeviceGradientSet.NAMES:
            assert _same(getattr(ref, name), getattr(got, name)), name
    ids2 = [5, 1, 4]
    ref2 = _per_view(sc, cams, dcs, ids2)
    got2 = multiview.batch_gradients(sc, cams, dcs, ids2, batch=vb)
    for name in device.DeviceGradientSet.NAMES:
        assert _same(getattr(ref2, name), getattr(got2, name)), name
    with torch.no_grad():
        sc.mu.mul_(1.01)  # a new scene state: the pair counts change
    ref3 = _per_view(sc, cams, dcs, ids)
    got3 = multiview.batch_gradients(sc, cams, dcs, ids, batch=vb)
    for name in device.DeviceGradientSet.NAMES:
        assert _same(getattr(ref3, name), getattr(got3, name)), name
