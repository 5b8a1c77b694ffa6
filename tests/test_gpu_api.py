"""GPU behaviour of the public surfaces: the drop-in `rasterizer` module (numpy
in/out), the blend-core plugin (Seam 1), the device API, and the reference's
bit-identity properties evaluated on the GPU path."""

import numpy as np
import pytest
import torch

from conftest import load_golden
from parity import assert_grads, assert_images
from test_oracle_properties import identity_camera, look_at, make_scene, tie
from paper_2406_02720_b200 import backend, device, errors, multiview, scenes
from paper_2406_02720_b200 import rasterizer as R
from paper_2406_02720_b200.geometry import CameraModel, Scene

pytestmark = pytest.mark.gpu


def dev_scene(sa, dtype=torch.float64):
    return Scene(*(getattr(sa, f) for f in sa.FIELDS), sh_degree=sa.sh_degree,
                 background_color=sa.background_color, device="cuda", dtype=dtype)


def test_dropin_render_matches_oracle(cuda):
    from oracle import oracle as O
    rng = np.random.default_rng(3)
    sa = make_scene(rng, 20, sh_degree=2)
    cam = look_at([0.4, -0.3, -0.6], [0, 0, 3.0], 96, 72)
    out = R.render(sa, cam)
    ref = O.render(sa, cam)
    assert_images({"color": out.color, "alpha": out.alpha, "depth": out.depth,
                   "transmittance": out.transmittance, "terminal": out.per_pixel_terminal_index},
                  {"color": ref.color, "alpha": ref.alpha, "depth": ref.depth,
                   "transmittance": ref.transmittance, "terminal": ref.per_pixel_terminal_index})
    d_color = rng.uniform(-1, 1, (72, 96, 3))
    g = R.render_backward(sa, cam, out, d_color)
    rg = O.render_backward(sa, cam, ref, d_color)
    assert_grads({k: getattr(g, k) for k in rg if k != "touch_count"},
                 {k: v for k, v in rg.items() if k != "touch_count"})
    assert np.array_equal(g.touch_count, rg["touch_count"])
    fg = out.frame
    assert np.array_equal(fg.pair_splat, ref.frame.pair_splat)
    assert np.array_equal(fg.tile_starts, ref.frame.tile_starts)


def test_dropin_output_dtypes_match_reference(cuda):
    """Seam 2 returns the reference's dtypes by default (the dtypes of its own arrays in
    the golden fixture: float64 images and gradients, int32 terminal, int64 touch
    counts); float32 is an explicit opt-in that keeps gradients in the scene's dtype."""
    gold = load_golden("mini")
    sa = scenes.frustum(300, 2, 64, 48, seed=3)
    s64 = sa.as_float64()
    cam = CameraModel(**sa.cameras[0])
    images = ("color", "alpha", "depth", "transmittance")
    out = R.render(s64, cam)
    g = R.render_backward(s64, cam, out, gold["d_color"])
    for k in images:
        assert getattr(out, k).dtype == gold[k].dtype == np.float64, k
    assert out.per_pixel_terminal_index.dtype == gold["terminal"].dtype == np.int32
    for k in R.GradientSet.NAMES:
        assert getattr(g, k).dtype == gold[k].dtype, k
    assert_images({k: getattr(out, k) for k in images} |
                  {"terminal": out.per_pixel_terminal_index},
                  {k: gold[k] for k in images + ("terminal",)})
    assert_grads({k: getattr(g, k) for k in R.GradientSet.NAMES[:-1]},
                 {k: gold[k] for k in R.GradientSet.NAMES[:-1]})
    # float32 scene, default: still float64 out (widened on the device, same values)
    out32 = R.render(sa, cam)
    g32 = R.render_backward(sa, cam, out32, gold["d_color"])
    assert out32.color.dtype == np.float64 and g32.d_mu.dtype == np.float64
    prev = R.set_output_dtype(np.float32)
    try:
        o = R.render(s64, cam)
        gg = R.render_backward(s64, cam, o, gold["d_color"])
        assert o.color.dtype == np.float32 and o.per_pixel_terminal_index.dtype == np.int32
        assert gg.d_mu.dtype == np.float64 and gg.touch_count.dtype == np.int64  # scene's dtype
        assert np.array_equal(gg.d_mu, g.d_mu)  # FP64 K7: nothing rounded
        assert np.array_equal(o.color.astype(np.float64), out.color)
        o = R.render(sa, cam)
        gg = R.render_backward(sa, cam, o, gold["d_color"])
        assert o.color.dtype == np.float32 and gg.d_mu.dtype == np.float32
        assert np.array_equal(gg.d_mu.astype(np.float64), g32.d_mu)
    finally:
        R.set_output_dtype(prev)
    assert R.output_dtype() is np.float64


def test_dropin_errors(cuda):
    rng = np.random.default_rng(0)
    sa = make_scene(rng, 3)
    empty = scenes.SceneArrays(**{f: getattr(sa, f)[:0] for f in sa.FIELDS},
                               sh_degree=sa.sh_degree)
    with pytest.raises(errors.EmptyScene):
        R.render(empty, identity_camera())
    with pytest.raises(ValueError):
        R.render(sa, identity_camera(), kernel="quarter")
    cam = identity_camera(32, 32)
    out = R.render(sa, cam)
    with pytest.raises(errors.MismatchedForward):
        R.render_backward(sa, cam, out, np.zeros((16, 16, 3)))
    bigger = make_scene(rng, 5)
    with pytest.raises(errors.MismatchedForward):
        R.render_backward(bigger, cam, out, np.zeros((32, 32, 3)))


def test_image_too_large(cuda):
    rng = np.random.default_rng(0)
    sa = dev_scene(make_scene(rng, 3))
    cam = CameraModel(np.eye(4), 10.0, 10.0, 10.0, 10.0, 65536, 32769)
    with pytest.raises(errors.ImageTooLarge):
        device.render(sa, cam)


def test_half_full_bit_identical_on_gpu(cuda):
    for seed in range(5):
        sa = tie(make_scene(np.random.default_rng(seed), 6))
        cam = look_at([0.3, -0.2, -0.5], [0, 0, 3.0])
        a = device.render(dev_scene(sa), cam, "half")
        b = device.render(dev_scene(sa), cam, "full")
        assert torch.equal(a.color, b.color) and torch.equal(a.depth, b.depth)
        assert torch.equal(a.alpha, b.alpha)


def test_odd_symmetry_bit_identical_on_gpu(cuda):
    for seed in range(5):
        sa = make_scene(np.random.default_rng(100 + seed), 6)
        fl = scenes.SceneArrays(**{f: getattr(sa, f).copy() for f in sa.FIELDS},
                                sh_degree=sa.sh_degree, background_color=sa.background_color)
        fl.normal = -fl.normal
        fl.raw_opacity_a, fl.raw_opacity_b = sa.raw_opacity_b.copy(), sa.raw_opacity_a.copy()
        cam = look_at([0.2, 0.1, -0.6], [0, 0, 3.0])
        a = device.render(dev_scene(sa), cam)
        b = device.render(dev_scene(fl), cam)
        assert torch.equal(a.color, b.color)


def test_run_to_run_determinism(cuda):
    """Launch-config / scheduling invariance: the persistent tile queue hands tiles
    to warps in a different order each run; outputs and gradients are bitwise equal."""
    sa = scenes.frustum(30_000, 3, 640, 360, seed=5)
    sc = dev_scene(sa, torch.float32)
    cam = CameraModel(**sa.cameras[0])
    dc = torch.as_tensor(scenes.cotangent(360, 640), dtype=torch.float32)
    res = []
    for _ in range(3):
        out = device.render(sc, cam)
        g = device.render_backward(sc, cam, out, dc)
        res.append((out.color.clone(), out.terminal.clone(), g.d_mu.clone(), g.d_sh.clone(),
                    g.d_normal.clone()))
    for r in res[1:]:
        for a, b in zip(res[0], r):
            assert torch.equal(a, b)


def test_zero_cotangent_and_tied_normal_on_gpu(cuda):
    rng = np.random.default_rng(1)
    sa = make_scene(rng, 6)
    cam = identity_camera(32, 32)
    sc = dev_scene(sa)
    out = device.render(sc, cam)
    g = device.render_backward(sc, cam, out, torch.zeros((32, 32, 3)))
    for k in device.DeviceGradientSet.NAMES[:-2]:
        assert not getattr(g, k).any(), k
    st = dev_scene(tie(sa))
    out = device.render(st, cam)
    g = device.render_backward(st, cam, out, torch.as_tensor(rng.uniform(-1, 1, (32, 32, 3))))
    assert g.d_normal.abs().max().item() == 0.0
    assert g.d_raw_opacity_a.abs().max().item() > 0.0


def test_culled_touch_count_on_gpu(cuda):
    rng = np.random.default_rng(2)
    sa = make_scene(rng, 5)
    sa.mu[0, 2] = -5.0
    cam = identity_camera(32, 32)
    out = R.render(sa, cam)
    g = R.render_backward(sa, cam, out, rng.uniform(-1, 1, (32, 32, 3)))
    assert g.touch_count[0] == 0 and g.pos_grad_norm[0] == 0.0
    assert (g.touch_count[1:] == 1).all()
    assert out.radii[0] == 0 and (out.radii[1:] > 0).all()


@pytest.mark.parametrize("chunks", [1, 3])
def test_seam1_blend_plugin_vs_oracle(cuda, chunks):
    """cuda_blend.forward_tiles/backward_tiles on the reference's packed splats
    (golden c1/ball_small), honouring [tile_lo, tile_hi) and += on pair rows."""
    from oracle import oracle as O
    assert backend.get_backend().__name__.endswith("cuda_blend")
    blend = backend.get_backend()
    for name in ("ball_small", "ties"):
        gold = load_golden(name)
        tx, ty = int(gold["tiles_x"]), int(gold["tiles_y"])
        h, w = gold["color"].shape[:2]
        bg = np.array(scenes.BACKGROUND)
        color = np.zeros((h, w, 3)); alpha = np.zeros((h, w)); depth = np.zeros((h, w))
        trans = np.ones((h, w)); term = np.zeros((h, w), np.int32)
        n_tiles = tx * ty
        bounds = np.linspace(0, n_tiles, chunks + 1).astype(int)
        args = (gold["packed"], gold["mode"], gold["pair_splat"], gold["tile_starts"], h, w, tx, bg)
        for lo, hi in zip(bounds[:-1], bounds[1:]):
            blend.forward_tiles(*args, color, alpha, depth, trans, term, int(lo), int(hi))
        assert_images({"color": color, "alpha": alpha, "depth": depth, "transmittance": trans,
                       "terminal": term}, gold)
        pg = np.zeros((gold["pair_splat"].shape[0], 12))
        for lo, hi in zip(bounds[:-1], bounds[1:]):
            blend.backward_tiles(*args, gold["d_color"], gold["transmittance"], gold["terminal"],
                                 pg, int(lo), int(hi))
        ref = np.zeros_like(pg)
        O.backward_tiles(*args, gold["d_color"], gold["transmittance"], gold["terminal"], ref, 0,
                         n_tiles)
        rel = np.linalg.norm(pg - ref, axis=0) / np.maximum(np.linalg.norm(ref, axis=0), 1e-30)
        assert rel.max() < 1e-3, rel


def test_seam1_threaded_chunks_vs_oracle(cuda):
    """The reference's dispatch (rasterizer.py:373-378, 412-417): 8 threads call the
    plugin concurrently on disjoint tile chunks of one frame.  The first call blends
    the frame once and the rest copy their tiles out of the kept result; images and
    pair rows equal the oracle's, and an in-place change of an input array (same
    pointers) is detected and recomputed."""
    from concurrent.futures import ThreadPoolExecutor
    from oracle import oracle as O
    blend = backend.get_backend()
    gold = load_golden("ball_small")
    tx, ty = int(gold["tiles_x"]), int(gold["tiles_y"])
    h, w = gold["color"].shape[:2]
    bg = np.array(scenes.BACKGROUND)
    n_tiles = tx * ty
    bounds = np.linspace(0, n_tiles, 9).astype(int)
    spans = list(zip(bounds[:-1].tolist(), bounds[1:].tolist()))
    packed = gold["packed"].copy()
    args = (packed, gold["mode"], gold["pair_splat"], gold["tile_starts"], h, w, tx, bg)

    def forward():
        out = [np.zeros((h, w, 3)), np.zeros((h, w)), np.zeros((h, w)), np.ones((h, w)),
               np.zeros((h, w), np.int32)]
        with ThreadPoolExecutor(max_workers=8) as pool:
            list(pool.map(lambda sp: blend.forward_tiles(*args, *out, *sp), spans))
        return dict(zip(("color", "alpha", "depth", "transmittance", "terminal"), out))

    def oracle_forward():
        out = [np.zeros((h, w, 3)), np.zeros((h, w)), np.zeros((h, w)), np.ones((h, w)),
               np.zeros((h, w), np.int32)]
        O.forward_tiles(*args, *out, 0, n_tiles)
        return dict(zip(("color", "alpha", "depth", "transmittance", "terminal"), out))

    for _ in range(2):  # the second frame is a cache hit for every chunk
        assert_images(forward(), gold)
    pg = np.zeros((gold["pair_splat"].shape[0], 12))
    with ThreadPoolExecutor(max_workers=8) as pool:
        list(pool.map(lambda sp: blend.backward_tiles(*args, gold["d_color"],
                                                      gold["transmittance"], gold["terminal"],
                                                      pg, *sp), spans))
    ref = np.zeros_like(pg)
    O.backward_tiles(*args, gold["d_color"], gold["transmittance"], gold["terminal"], ref, 0,
                     n_tiles)
    rel = np.linalg.norm(pg - ref, axis=0) / np.maximum(np.linalg.norm(ref, axis=0), 1e-30)
    assert rel.max() < 1e-3, rel
    # same buffers, new values: the colour columns change in place
    packed[:, 9:12] *= 0.5
    got = forward()
    assert_images(got, oracle_forward())
    from paper_2406_02720_b200 import _native
    _native.load().hs_seam1_cache_clear()


def test_seam1_rejects_bad_arrays(cuda):
    gold = load_golden("mini")
    h, w = gold["color"].shape[:2]
    blend = backend.get_backend()
    with pytest.raises(ValueError):
        blend.forward_tiles(gold["packed"].astype(np.float32), gold["mode"], gold["pair_splat"],
                            gold["tile_starts"], h, w, int(gold["tiles_x"]),
                            np.zeros(3), np.zeros((h, w, 3)), np.zeros((h, w)), np.zeros((h, w)),
                            np.zeros((h, w)), np.zeros((h, w), np.int32), 0, 1)


def test_multiview_accumulation_equals_sum(cuda):
    sa = scenes.ball(5000, 2, 96, 96, views=4, seed=4)
    sc = dev_scene(sa, torch.float32)
    cams = [CameraModel(**c) for c in sa.cameras]
    dcs = [torch.as_tensor(scenes.cotangent(96, 96, seed=v), dtype=torch.float32) for v in range(4)]
    batch = multiview.batch_gradients(sc, cams, dcs, [0, 1, 2, 3])
    total = torch.zeros_like(batch.flat)
    for v in range(4):
        g = device.DeviceGradientSet.empty_flat(sc)
        out = device.render(sc, cams[v])
        device.render_backward(sc, cams[v], out, dcs[v], grads=g)
        total += g.flat
    torch.testing.assert_close(batch.flat, total, rtol=1e-6, atol=1e-7)
    assert batch.touch_count.max().item() <= 4


def test_torch_autograd_matches_oracle(cuda):
    """rasterize_half_gaussians: loss.backward() gives the oracle's GradientSet."""
    from oracle import oracle as O
    from paper_2406_02720_b200.torch_api import (HalfGaussianRasterizationSettings,
                                                 HalfGaussianRasterizer)
    sa = scenes.frustum(3000, 2, 160, 120, seed=12)
    cam = sa.cameras[0]
    settings = HalfGaussianRasterizationSettings(
        image_height=cam["height"], image_width=cam["width"], world_to_cam=cam["world_to_cam"],
        fx=cam["fx"], fy=cam["fy"], cx=cam["cx"], cy=cam["cy"], sh_degree=sa.sh_degree,
        background=tuple(sa.background_color))
    params = {f: torch.tensor(getattr(sa, f), device="cuda", requires_grad=True)
              for f in sa.FIELDS}
    rast = HalfGaussianRasterizer(settings)
    color, radii = rast(params["mu"], params["normal"], params["raw_opacity_a"],
                        params["raw_opacity_b"], params["log_scale"], params["rotation"],
                        params["sh_coeffs"])
    d_color = scenes.cotangent(cam["height"], cam["width"], seed=3)
    loss = (color * torch.as_tensor(d_color, dtype=torch.float32, device="cuda")).sum()
    loss.backward()
    s64 = sa.as_float64()
    ref = O.render(s64, CameraModel(**cam))
    rg = O.render_backward(s64, CameraModel(**cam), ref, d_color)
    assert abs(loss.item() - float((ref.color * d_color).sum())) < 1e-3 * abs(loss.item()) + 1e-2
    got = {"d_mu": params["mu"].grad, "d_log_scale": params["log_scale"].grad,
           "d_rotation": params["rotation"].grad, "d_sh": params["sh_coeffs"].grad,
           "d_normal": params["normal"].grad, "d_raw_opacity_a": params["raw_opacity_a"].grad,
           "d_raw_opacity_b": params["raw_opacity_b"].grad}
    assert_grads({k: v.double().cpu().numpy() for k, v in got.items()},
                 {k: rg[k] for k in got}, groups=tuple(got))
    assert (radii.cpu().numpy() > 0).sum() == ref.frame.valid.shape[0]


def test_reduction_store_modes_match_accumulate(cuda):
    """hs_grads.accumulate = 2 (device atomics into zeroed buffers) gives bit for bit
    the gradients of the read-modify-write accumulation over the same two views,
    up to subnormals (float atomics flush them); the multicast mode 3 differs only
    in the store instruction."""
    from paper_2406_02720_b200 import device
    from paper_2406_02720_b200.geometry import CameraModel, Scene
    sa = scenes.ball(4000, 2, 96, 72, views=4, seed=3)
    scene = Scene(*(getattr(sa, f) for f in sa.FIELDS), sh_degree=sa.sh_degree,
                  background_color=sa.background_color, device="cuda", dtype=torch.float32)
    cams = [CameraModel(**c) for c in sa.cameras]
    dcs = [torch.as_tensor(scenes.cotangent(c.height, c.width, seed=i), dtype=torch.float32,
                           device="cuda") for i, c in enumerate(cams)]
    ref = device.DeviceGradientSet.empty_flat(scene)
    red = device.DeviceGradientSet.empty_flat(scene)
    red.flat.zero_()
    red.touch_count.zero_()
    ptrs = {name: getattr(red, name).data_ptr() for name in device.DeviceGradientSet.NAMES}
    ptrs["mode"] = 2
    rast = device.Rasterizer("cuda")
    for j, v in enumerate((0, 2)):
        out = rast.render(scene, cams[v])
        rast.render_backward(scene, cams[v], out, dcs[v], grads=ref, accumulate=j > 0)
        out = rast.render(scene, cams[v])
        rast.render_backward(scene, cams[v], out, dcs[v], grads=red, reduce_ptrs=ptrs)
    torch.cuda.synchronize()
    for name in device.DeviceGradientSet.NAMES:
        assert _same_up_to_subnormals(getattr(ref, name), getattr(red, name)), name


def _same_up_to_subnormals(a, b):
    """Float atomics flush subnormal operands and results to zero, so values may
    differ by subnormal amounts (< 2 * FLT_MIN) and by nothing else."""
    if not a.is_floating_point():
        return torch.equal(a, b)
    return bool(((a.double() - b.double()).abs() <= 2 * torch.finfo(a.dtype).tiny).all())


def test_fused_gradient_reduce_single_rank(cuda):
    """FusedGradientReduce over a one-rank NCCL group (symmetric memory; without an
    NVSwitch it runs the same protocol with device atomics): equals batch_gradients."""
    import torch.distributed as dist
    from paper_2406_02720_b200 import device, multiview
    from paper_2406_02720_b200.geometry import CameraModel, Scene
    if not dist.is_initialized():
        dist.init_process_group("nccl", init_method="tcp://127.0.0.1:29517", rank=0,
                                world_size=1, device_id=torch.device("cuda", 0))
    try:
        sa = scenes.ball(3000, 1, 80, 64, views=3, seed=8)
        scene = Scene(*(getattr(sa, f) for f in sa.FIELDS), sh_degree=sa.sh_degree,
                      background_color=sa.background_color, device="cuda", dtype=torch.float32)
        cams = [CameraModel(**c) for c in sa.cameras]
        dcs = [torch.as_tensor(scenes.cotangent(c.height, c.width, seed=i), dtype=torch.float32,
                               device="cuda") for i, c in enumerate(cams)]
        ref = multiview.batch_gradients(scene, cams, dcs, [0, 1, 2])
        fused = multiview.FusedGradientReduce(scene)
        got = multiview.batch_gradients(scene, cams, dcs, [0, 1, 2], fused=fused)
        torch.cuda.synchronize()
        for name in device.DeviceGradientSet.NAMES:
            assert _same_up_to_subnormals(getattr(ref, name), getattr(got, name)), name
        # the same reduction stores from the multi-view K7 (views on their streams)
        got = multiview.batch_gradients(scene, cams, dcs, [0, 1, 2], fused=fused,
                                        batch=multiview.ViewBatch(scene, 3))
        torch.cuda.synchronize()
        for name in device.DeviceGradientSet.NAMES:
            assert _same_up_to_subnormals(getattr(ref, name), getattr(got, name)), name
    finally:
        dist.destroy_process_group()


def test_bucketed_k7_and_allreduce_single_rank(cuda):
    """K7 over primitive buckets (hs_preprocess_bwd_range) with each bucket's NCCL
    all-reduce issued right after its launch (one-rank NCCL group: the exchange is
    the identity): bit-identical to one K7 launch, for a fresh and an accumulating
    view."""
    import torch.distributed as dist
    from paper_2406_02720_b200 import device, multiview
    from paper_2406_02720_b200.geometry import CameraModel, Scene
    if not dist.is_initialized():
        dist.init_process_group("nccl", init_method="tcp://127.0.0.1:29519", rank=0,
                                world_size=1, device_id=torch.device("cuda", 0))
    try:
        sa = scenes.ball(5000, 3, 96, 72, views=4, seed=12)
        scene = Scene(*(getattr(sa, f) for f in sa.FIELDS), sh_degree=sa.sh_degree,
                      background_color=sa.background_color, device="cuda", dtype=torch.float32)
        cams = [CameraModel(**c) for c in sa.cameras]
        dcs = [torch.as_tensor(scenes.cotangent(c.height, c.width, seed=i), dtype=torch.float32,
                               device="cuda") for i, c in enumerate(cams)]
        ref = device.DeviceGradientSet.empty_flat(scene)
        got = device.DeviceGradientSet.empty_flat(scene)
        red = multiview.GradientAllReduce(got)
        buckets = multiview.GradientAllReduce.bucket_ranges(len(scene), buckets=3)
        rast = device.Rasterizer("cuda")
        for j, v in enumerate((1, 3)):
            out = rast.render(scene, cams[v])
            rast.render_backward(scene, cams[v], out, dcs[v], grads=ref, accumulate=j > 0)
            out = rast.render(scene, cams[v])
            last = j == 1
            rast.render_backward(scene, cams[v], out, dcs[v], grads=got, accumulate=j > 0,
                                 buckets=buckets, on_bucket=red.start_range if last else None)
        red.finish()
        torch.cuda.synchronize()
        for name in device.DeviceGradientSet.NAMES:
            assert torch.equal(getattr(ref, name), getattr(got, name)), name
    finally:
        dist.destroy_process_group()


def test_seam1_large_thin_splats_vs_oracle(cuda):
    """Seam 1 on reference-packed splats with radii up to ~1000 px: pack_records stores
    them in the stable conic form (kFlagNoWin) and the blend core matches the oracle."""
    from oracle import oracle as O
    from paper_2406_02720_b200.geometry import CameraModel
    blend = backend.get_backend()
    rng = np.random.default_rng(4)
    sa = scenes.frustum(60, 1, 640, 480, seed=6, sig_lo=1.0, sig_hi=2.0)
    ls = sa.log_scale.astype(np.float64)
    ls[:, 0] += np.log(rng.uniform(60.0, 150.0, len(ls)))
    sa.log_scale = ls.astype(np.float32)
    s64 = sa.as_float64()
    cam = CameraModel(**sa.cameras[0])
    fr = O.prepare(s64, cam)
    h, w, tx, ty = cam.height, cam.width, fr.tiles_x, fr.tiles_y
    bg = np.array(scenes.BACKGROUND)
    args = (fr.packed, fr.mode, fr.pair_splat, fr.tile_starts, h, w, tx, bg)
    out = [np.zeros((h, w, 3)), np.zeros((h, w)), np.zeros((h, w)), np.ones((h, w)),
           np.zeros((h, w), np.int32)]
    ref = [np.zeros((h, w, 3)), np.zeros((h, w)), np.zeros((h, w)), np.ones((h, w)),
           np.zeros((h, w), np.int32)]
    blend.forward_tiles(*args, *out, 0, tx * ty)
    O.forward_tiles(*args, *ref, 0, tx * ty)
    keys = ("color", "alpha", "depth", "transmittance", "terminal")
    assert_images(dict(zip(keys, out)), dict(zip(keys, ref)))
    d_color = scenes.cotangent(h, w, seed=3)
    pg = np.zeros((fr.pair_splat.shape[0], 12))
    pr = np.zeros_like(pg)
    blend.backward_tiles(*args, d_color, ref[3], ref[4], pg, 0, tx * ty)
    O.backward_tiles(*args, d_color, ref[3], ref[4], pr, 0, tx * ty)
    rel = np.linalg.norm(pg - pr, axis=0) / np.maximum(np.linalg.norm(pr, axis=0), 1e-30)
    assert rel.max() < 1e-3, rel
