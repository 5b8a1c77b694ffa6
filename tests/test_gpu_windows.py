"""Strip windows of the blend kernels (hs_blend.cu strip_window): a splat is not
evaluated on the 16x4-pixel strips of a tile where its Gaussian is below 2^-27,
which FP32 makes equivalent to evaluating it (T(1 - w) rounds to T).  These tests
check that the windows are conservative against the exact per-strip maximum of
the Gaussian (safety threshold 2^-25), that they do skip work, and that images
and gradients on a scene full of skipped strips match the FP64 oracle."""

import ctypes

import numpy as np
import pytest
import torch

from parity import assert_grads, assert_images, GRAD_GROUPS
from paper_2406_02720_b200 import _native, device, scenes
from paper_2406_02720_b200.geometry import CameraModel, Scene

pytestmark = pytest.mark.gpu


def _scene():
    # small anisotropic splats: many straddle tile borders with strips they never reach
    return scenes.frustum(6000, 1, 256, 192, seed=21, sig_lo=0.3, sig_hi=3.0)


def _strip_gmax(packed, pair_splat, tile_starts, tiles_x):
    """Exact max of the Gaussian over each 16x4 strip for every (tile, pair): (P, 4)."""
    t = np.repeat(np.arange(len(tile_starts) - 1), np.diff(tile_starts))
    p = packed[pair_splat].astype(np.float64)
    off = np.arange(16) + 0.5
    dx = (t % tiles_x)[:, None] * 16 + off[None, :] - p[:, 0:1]
    dy = (t // tiles_x)[:, None] * 16 + off[None, :] - p[:, 1:2]
    a, b, c = (p[:, k, None, None] for k in (2, 3, 4))
    pw = -0.5 * (a * dx[:, None, :] ** 2 + c * dy[:, :, None] ** 2) - b * dx[:, None, :] * dy[:, :, None]
    return np.exp(pw).reshape(len(p), 4, 64).max(axis=2)


def test_windows_conservative_and_effective(cuda):
    sa = _scene()
    cam = CameraModel(**sa.cameras[0])
    sc = Scene(*(getattr(sa, f) for f in sa.FIELDS), sh_degree=sa.sh_degree,
               background_color=sa.background_color, device="cuda", dtype=torch.float32)
    fr = device.prepare(sc, cam)
    hist = torch.zeros(4, dtype=torch.int64, device="cuda")
    st = _native.load().hs_blend_window_stats(
        ctypes.byref(fr.st), ctypes.c_void_p(hist.data_ptr()),
        ctypes.c_void_p(torch.cuda.current_stream().cuda_stream))
    _native.check(st, "hs_blend_window_stats")
    none, lower, upper, full = (int(v) for v in hist.cpu())
    ex = fr.export()
    g = _strip_gmax(ex["packed"], ex["pair_splat"], ex["tile_starts"], fr.tiles_x)
    need = g >= 2.0 ** -25          # strips that must be evaluated
    may_none = ~need.any(1)
    may_lower = ~need[:, 2:].any(1)  # nothing needed in strips 2-3
    may_upper = ~need[:, :2].any(1)
    assert none + lower + upper + full == len(g)
    assert none <= may_none.sum()
    assert none + lower <= may_lower.sum()
    assert none + upper <= may_upper.sum()
    # and effective: everything a 2^-30 criterion skips is skipped (the kernel's bound
    # sits at 2^-27, a factor 8 inside)
    strict = g >= 2.0 ** -30
    assert none >= (~strict.any(1)).sum() > 0
    assert none + lower >= (~strict[:, 2:].any(1)).sum()
    assert none + upper >= (~strict[:, :2].any(1)).sum()
    assert lower > 0 and upper > 0


def test_windowed_scene_matches_oracle(cuda):
    from oracle import oracle as O
    sa = _scene()
    cam = CameraModel(**sa.cameras[0])
    d_color = scenes.cotangent(cam.height, cam.width, seed=2)
    s64 = sa.as_float64()
    ref = O.render(s64, cam)
    ref_g = O.render_backward(s64, cam, ref, d_color)
    sc = Scene(*(getattr(sa, f) for f in sa.FIELDS), sh_degree=sa.sh_degree,
               background_color=sa.background_color, device="cuda", dtype=torch.float32)
    out = device.render(sc, cam)
    got = {"color": out.color.cpu().numpy(), "alpha": out.alpha.cpu().numpy(),
           "depth": out.depth.cpu().numpy(), "transmittance": out.transmittance.cpu().numpy(),
           "terminal": out.terminal.cpu().numpy()}
    assert_images(got, {"color": ref.color, "alpha": ref.alpha, "depth": ref.depth,
                        "transmittance": ref.transmittance,
                        "terminal": ref.per_pixel_terminal_index})
    g = device.render_backward(sc, cam, out, torch.as_tensor(d_color, dtype=torch.float32))
    assert_grads({k: getattr(g, k).double().cpu().numpy() for k in GRAD_GROUPS},
                 {k: ref_g[k] for k in GRAD_GROUPS})


def test_occluded_view_matches_oracle(cuda):
    """Mean tile list above 1000 pairs: K6 takes its occluded instantiation (windows on
    the partially-active path, masked by the halves that still hold an active pixel)."""
    from oracle import oracle as O
    sa = scenes.frustum(6000, 1, 64, 48, seed=8, sig_lo=6.0, sig_hi=24.0)
    cam = CameraModel(**sa.cameras[0])
    d_color = scenes.cotangent(cam.height, cam.width, seed=5)
    s64 = sa.as_float64()
    ref = O.render(s64, cam)
    ref_g = O.render_backward(s64, cam, ref, d_color)
    assert ref.frame.pair_splat.shape[0] > 1000 * (len(ref.frame.tile_starts) - 1)
    assert (ref.per_pixel_terminal_index < np.diff(ref.frame.tile_starts).max()).mean() > 0.5
    sc = Scene(*(getattr(sa, f) for f in sa.FIELDS), sh_degree=sa.sh_degree,
               background_color=sa.background_color, device="cuda", dtype=torch.float32)
    out = device.render(sc, cam)
    got = {"color": out.color.cpu().numpy(), "alpha": out.alpha.cpu().numpy(),
           "depth": out.depth.cpu().numpy(), "transmittance": out.transmittance.cpu().numpy(),
           "terminal": out.terminal.cpu().numpy()}
    assert_images(got, {"color": ref.color, "alpha": ref.alpha, "depth": ref.depth,
                        "transmittance": ref.transmittance,
                        "terminal": ref.per_pixel_terminal_index})
    g = device.render_backward(sc, cam, out, torch.as_tensor(d_color, dtype=torch.float32))
    assert_grads({k: getattr(g, k).double().cpu().numpy() for k in GRAD_GROUPS},
                 {k: ref_g[k] for k in GRAD_GROUPS})


def test_large_thin_splats_stable_conic(cuda):
    """Splats with a radius above 256 px carry the cancellation-free conic form, take the
    generic blend path and no strip windows; a scene of long, thin, large splats matches
    the oracle (images, gradients and the exported packed conic)."""
    from oracle import oracle as O
    rng = np.random.default_rng(4)
    sa = scenes.frustum(60, 1, 640, 480, seed=6, sig_lo=1.0, sig_hi=2.0)
    # stretch every splat along one axis to 60-150x its width: radii up to ~1000 px.
    # Before the stable conic form (hs_common.cuh kFlagNoWin) alpha was 1.7e-4 off here.
    ls = sa.log_scale.astype(np.float64)
    ls[:, 0] += np.log(rng.uniform(60.0, 150.0, len(ls)))
    sa.log_scale = ls.astype(np.float32)
    cam = CameraModel(**sa.cameras[0])
    sc = Scene(*(getattr(sa, f) for f in sa.FIELDS), sh_degree=sa.sh_degree,
               background_color=sa.background_color, device="cuda", dtype=torch.float32)
    out = device.render(sc, cam)
    assert int(out.radii.max()) > 256
    d_color = scenes.cotangent(cam.height, cam.width, seed=3)
    s64 = sa.as_float64()
    ref = O.render(s64, cam)
    ref_g = O.render_backward(s64, cam, ref, d_color)
    got = {"color": out.color.cpu().numpy(), "alpha": out.alpha.cpu().numpy(),
           "depth": out.depth.cpu().numpy(), "transmittance": out.transmittance.cpu().numpy(),
           "terminal": out.terminal.cpu().numpy()}
    assert_images(got, {"color": ref.color, "alpha": ref.alpha, "depth": ref.depth,
                        "transmittance": ref.transmittance,
                        "terminal": ref.per_pixel_terminal_index})
    g = device.render_backward(sc, cam, out, torch.as_tensor(d_color, dtype=torch.float32))
    assert_grads({k: getattr(g, k).double().cpu().numpy() for k in GRAD_GROUPS},
                 {k: ref_g[k] for k in GRAD_GROUPS})
    # the export reconstructs (a, b, c) from the stable form
    ex = out.frame.export()
    np.testing.assert_allclose(ex["packed"][:, 2:5], ref.frame.packed[:, 2:5], rtol=2e-6,
                               atol=1e-30)


@pytest.mark.parametrize("sub", ["1", "2", "4"])
def test_forward_sub_tiles_vs_oracle(cuda, sub, monkeypatch):
    """K5 in 16x16 tiles, 16x8 or 16x4 sub-tiles (HS_SUBTILE forces the split the
    frame size would otherwise pick): every split matches the oracle, terminal
    counts agree exactly across splits and images to well below the contract (the
    strip windows of a sub-tile skip only FP32-invisible work)."""
    from oracle import oracle as O
    from parity import assert_images
    from paper_2406_02720_b200 import device, scenes
    from paper_2406_02720_b200.geometry import CameraModel, Scene
    sa = scenes.frustum(20_000, 2, 320, 200, seed=17, sig_lo=0.5, sig_hi=8.0)
    cam = CameraModel(**sa.cameras[0])
    sc = Scene(*(getattr(sa, f) for f in sa.FIELDS), sh_degree=sa.sh_degree,
               background_color=sa.background_color, device="cuda", dtype=torch.float32)
    monkeypatch.setenv("HS_SUBTILE", "1")
    base = device.render(sc, cam)
    monkeypatch.setenv("HS_SUBTILE", sub)
    out = device.render(sc, cam)
    assert torch.equal(out.terminal, base.terminal)
    assert (out.color - base.color).abs().max().item() < 1e-6
    ref = O.render(sa.as_float64(), cam)
    assert_images({"color": out.color.cpu().numpy(), "alpha": out.alpha.cpu().numpy(),
                   "depth": out.depth.cpu().numpy(),
                   "transmittance": out.transmittance.cpu().numpy(),
                   "terminal": out.terminal.cpu().numpy()},
                  {"color": ref.color, "alpha": ref.alpha, "depth": ref.depth,
                   "transmittance": ref.transmittance, "terminal": ref.per_pixel_terminal_index})
