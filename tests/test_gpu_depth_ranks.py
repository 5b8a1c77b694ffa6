"""Depth ranks (hs_binning.cu run_depth_sort_hi): a stable sort on the upper 32
bits of the f64 depth plus a per-run fixup, with a full 64-bit re-sort when a
run is too long for the fixup.  The pair order must stay exactly np.lexsort's
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
    ex = device.prepare(sc, cam).export()
    ref = O.prepare(sa, cam)
    assert np.array_equal(ex["tile_starts"], ref.tile_starts)
    assert np.array_equal(ex["pair_splat"], ref.pair_splat)


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
