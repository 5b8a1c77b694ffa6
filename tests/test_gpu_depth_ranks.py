"""Depth ranks (hs_binning.cu run_depth_sort_hi): a stable sort on the upper 32
bits of the f64 depth (as 24-bit offsets from the frame's smallest) plus a
per-run fixup, with a full 64-bit re-sort when a run is too long for the fixup
or the depths span too wide a range for 24 bits.  The pair order must stay exactly np.lexsort's
(tile, depth, index) order in all three regimes: short runs, runs just under
the fixup limit, and runs far over it (the fallback)."""

import numpy as np
import pytest
import torch

from paper_2406_02720_b200 import device, scenes
from paper_2406_02720_b200.geometry import CameraModel, Scene

pytestmark = pytest.mark.gpu


def _with_depths(n, z, seed=3):
    """A frustum scene (float64) whose depths are replaced by `z` (x, y rescaled)."""
    sa = scenes.frustum(n, 1, 160, 120, seed=seed, sig_lo=1.0, sig_hi=5.0).as_float64()
    mu = sa.mu.copy()
    mu[:, :2] *= (z / mu[:, 2])[:, None]
    mu[:, 2] = z
    sa.mu = mu
    return sa


def _check(sa):
    from oracle import oracle as O
    cam = CameraModel(**sa.cameras[0])
    sc = Scene(*(getattr(sa, f) for f in sa.FIELDS), sh_degree=sa.sh_degree,
               background_color=sa.background_color, device="cuda", dtype=torch.float64)
    frame = device.prepare(sc, cam)
    ex = frame.export()
    ref = O.prepare(sa, cam)
    assert np.array_equal(ex["tile_starts"], ref.tile_starts)
    assert np.array_equal(ex["pair_splat"], ref.pair_splat)
    return frame


def test_short_runs_in_upper_bits():
    # depths 2^-40 apart: dozens of splats share the upper 32 bits in shuffled order
    rng = np.random.default_rng(1)
    n = 3000
    z = 4.0 + rng.integers(0, 200, n) * 2.0 ** -40 + rng.integers(0, 100, n) * 1e-5
    _check(_with_depths(n, z))


def test_runs_just_under_the_fixup_limit():
    rng = np.random.default_rng(2)
    n = 6000
    # three buckets of 2000 (limit 2048), descending low bits against the index order
    z = 3.0 + (np.arange(n) // 2000) * 0.25 + (n - np.arange(n)) * 2.0 ** -44
    z = z[rng.permutation(n)]
    _check(_with_depths(n, z))


def test_long_runs_take_the_full_sort():
    rng = np.random.default_rng(3)
    n = 4000
    # one bucket of 2500 distinct depths (over the limit: the full sort) plus 1500
    # exactly equal ones (ranked by index)
    z = np.concatenate([4.0 + rng.permutation(2500) * 2.0 ** -42, np.full(1500, 5.0)])
    _check(_with_depths(n, z[rng.permutation(n)]))


def test_depth_range_wider_than_24_bits_takes_the_full_sort():
    # visible depths from 0.02 to 5000: the upper words span more than 2^24, so the
    # 24-bit key overflows and the ranks come from the 64-bit sort
    rng = np.random.default_rng(4)
    n = 3000
    z = np.exp(rng.uniform(np.log(0.02), np.log(5000.0), n))
    sa = _with_depths(n, z)
    sa.cameras[0]["near_clip"] = 0.01
    assert _check(sa).st.depth_sort_full == 1


def test_depth_range_just_inside_24_bits():
    # upper words from 2.0 to just under 2^(2+16): the widest range the 24-bit keys hold
    rng = np.random.default_rng(5)
    n = 3000
    z = 2.0 * 2.0 ** rng.uniform(0.0, 15.99, n)
    assert _check(_with_depths(n, z)).st.depth_sort_full == 0


def test_workspace_reuse_across_pair_counts():
    """One Rasterizer (persistent workspace) over scenes whose pair count grows and
    shrinks: hs_read_pairs_and_bin bins in place when the workspace fits and asks for
    a larger one otherwise; every render equals a fresh one bit for bit."""
    rast = device.Rasterizer("cuda", slots=1)
    for n, seed in ((500, 1), (4000, 2), (800, 3), (6000, 4)):
        sa = scenes.frustum(n, 1, 96, 64, seed=seed, sig_lo=1.0, sig_hi=6.0)
        cam = CameraModel(**sa.cameras[0])
        sc = Scene(*(getattr(sa, f) for f in sa.FIELDS), sh_degree=sa.sh_degree,
                   background_color=sa.background_color, device="cuda", dtype=torch.float32)
        a = rast.render(sc, cam)
        ca, ta = a.color.clone(), a.terminal.clone()
        pa = a.frame.export()["pair_splat"]
        b = device.render(sc, cam)
        assert torch.equal(ca, b.color) and torch.equal(ta, b.terminal)
        assert np.array_equal(pa, b.frame.export()["pair_splat"])


# ---- binning with P on the device (hs_bin_async) ------------------------------

def _dev_scene(sa, dtype=torch.float32):
    return Scene(*(getattr(sa, f) for f in sa.FIELDS), sh_degree=sa.sh_degree,
                 background_color=sa.background_color, device="cuda", dtype=dtype)


def _assert_matches_oracle(out, sa, cam):
    from oracle import oracle as O
    ref = O.prepare(sa.as_float64(), cam)
    ex = out.frame.export()
    assert np.array_equal(ex["pair_splat"], ref.pair_splat)
    assert np.array_equal(ex["tile_starts"], ref.tile_starts)


def test_async_binning_equals_sync_and_oracle():
    """A Rasterizer bins its first view after reading P, later views with P left on
    the device: every view's pair order and tile ranges equal the oracle's, and the
    async render equals a synchronous one bit for bit."""
    rast = device.Rasterizer("cuda", slots=1)
    for sa in (scenes.frustum(6000, 2, 320, 240, seed=5, sig_lo=0.5, sig_hi=8.0),
               scenes.frustum(3000, 1, 200, 150, seed=6, clustered=True, dup=0.2),
               scenes.ball(5000, 3, 256, 192, views=4, seed=7)):
        sc = _dev_scene(sa)
        cam = CameraModel(**sa.cameras[0])
        for rep in range(3):
            out = rast.render(sc, cam)
            if rep > 0:
                assert out.frame.pending  # binned with P left on the device
            ref = device.render(sc, cam)
            assert torch.equal(out.color, ref.color) and torch.equal(out.terminal, ref.terminal)
            _assert_matches_oracle(out, sa, cam)


def test_async_binning_overflow_is_detected_and_rebinned():
    """A view whose P exceeds the workspace's capacity: nothing is binned (empty
    tile lists, no out-of-bounds work); resolve() re-bins it so a second blend is
    exact, and a view nobody resolved is reported by the next prepare."""
    small = scenes.frustum(300, 1, 640, 480, seed=1, sig_lo=0.5, sig_hi=1.0)
    big = scenes.frustum(30000, 1, 640, 480, seed=2, sig_lo=4.0, sig_hi=20.0)
    s_small, s_big = _dev_scene(small), _dev_scene(big)
    cam = CameraModel(**small.cameras[0])
    ref = device.render(s_big, cam)
    assert ref.frame.num_pairs > device._capacity_for(device.render(s_small, cam).frame.num_pairs)

    rast = device.Rasterizer("cuda", slots=1)
    rast.render(s_small, cam)
    out = rast.render(s_big, cam)  # async, over capacity
    assert out.frame.pending
    torch.cuda.synchronize()
    assert int(out.terminal.max()) == 0  # empty tile lists: background only
    assert out.frame.resolve() is True  # re-binned synchronously with a larger workspace
    again = device.render(s_big, cam, frame=out.frame)
    assert torch.equal(again.color, ref.color) and torch.equal(again.terminal, ref.terminal)
    _assert_matches_oracle(again, big, cam)

    rast = device.Rasterizer("cuda", slots=1)
    rast.render(s_small, cam)
    rast.render(s_big, cam)  # overflows; nobody resolves it
    with pytest.raises(device.BinningOverflow):
        rast.render(s_small, cam)
    out = rast.render(s_big, cam)  # the capacity was reset: P is read, then binned
    assert torch.equal(out.color, ref.color)


def test_async_binning_depth_fallback():
    """A view whose depth runs overflow the fixup while binned asynchronously: the
    status carries the depth flag, resolve() re-ranks with the full sort, and the
    workspace ranks later views with the full sort from then on."""
    rng = np.random.default_rng(3)
    n = 4000
    z = np.concatenate([4.0 + rng.permutation(2500) * 2.0 ** -42, np.full(1500, 5.0)])
    long_runs = _with_depths(n, z[rng.permutation(n)])
    short = _with_depths(n, 3.0 + rng.uniform(0, 1, n))
    rast = device.Rasterizer("cuda", slots=1)
    cam = CameraModel(**short.cameras[0])
    rast.render(_dev_scene(short, torch.float64), cam)
    out = rast.render(_dev_scene(long_runs, torch.float64), cam)
    assert out.frame.pending
    _assert_matches_oracle(out, long_runs, cam)  # export() resolves: full sort, re-bin
    assert rast.slots[0].depth_sort_full == 1
    out = rast.render(_dev_scene(long_runs, torch.float64), cam)
    assert out.frame.pending and out.frame.st.depth_sort_full == 1
    _assert_matches_oracle(out, long_runs, cam)
