"""Density control on the device (csrc/hs_densify.cu, trainer.py mirror)
against the reference's densify_and_prune / reset_opacity
(tests/golden/densify.npz, trainer.py:229-350).

Contract: with the reference's split offsets (a numpy Generator passed as
`rng`), a float64 scene densifies BIT-IDENTICALLY -- the new rows, their order,
the re-aligned Adam moments, the report, and reset_opacity -- except that a
split child's or clone's position may differ by <= 2 ulp where CUDA's exp()
and numpy's differ by an ulp (as in K1).  float32 scenes
match within float32 rounding.  Without a Generator the split offsets come from
the device Philox stream: same rows except the children's positions, which are
checked statistically."""

import numpy as np
import pytest
import torch

import adam_cases as A
from conftest import load_golden

pytestmark = pytest.mark.gpu


def _setup(c, dtype):
    from paper_2406_02720_b200 import trainer as T
    from paper_2406_02720_b200.geometry import Scene
    scene = Scene(*(c["params"][f] for f in A.FIELDS), sh_degree=c["deg"], device="cuda",
                  dtype=dtype)
    gs, ms, cnt = c["stats"]
    stats = T.DensifyStats(torch.as_tensor(gs, device="cuda"), torch.as_tensor(ms, device="cuda"),
                           torch.as_tensor(cnt, device="cuda"))
    opt = T.AdamState(scene)
    for k, f in enumerate(A.FIELDS):
        opt._m[k].copy_(torch.as_tensor(c["m"][f]))
        opt._v[k].copy_(torch.as_tensor(c["v"][f]))
    for g in T.GROUPS:
        opt.t[g] = 7
    cfg = T.TrainConfig(total_iters=100, densify_until=50, max_primitives=c["max_primitives"])
    return scene, stats, opt, cfg


@pytest.mark.parametrize("dtype", [torch.float64, torch.float32])
def test_densify_matches_reference(cuda, dtype):
    from paper_2406_02720_b200 import trainer as T
    gold = load_golden("densify")
    for name in gold["cases"]:
        c = A.densify_case(gold, name)
        scene, stats, opt, cfg = _setup(c, dtype)
        new, new_stats, report = T.densify_and_prune(scene, stats, cfg, opt,
                                                     np.random.default_rng(c["seed"]),
                                                     c["extent"])
        torch.cuda.synchronize()
        assert report == c["report"], name
        assert len(new) == c["out"]["mu"].shape[0]
        assert int(new_stats.count.sum()) == 0 and len(new_stats.grad_sum) == len(new)
        for k, f in enumerate(A.FIELDS):
            got = getattr(new, f).cpu().numpy().astype(np.float64)
            gm = opt._m[k].cpu().numpy().astype(np.float64)
            gv = opt._v[k].cpu().numpy().astype(np.float64)
            if dtype == torch.float64 and f == "mu":
                ulps = np.abs(got - c["out"][f]) / np.spacing(np.abs(c["out"][f]))
                assert ulps.max() <= 2, (name, f, ulps.max())
            elif dtype == torch.float64:
                assert np.array_equal(got, c["out"][f]), (name, f)
            else:
                np.testing.assert_allclose(got, c["out"][f], rtol=1e-6, atol=1e-6,
                                           err_msg=f"{name} {f}")
            assert np.array_equal(gm, c["out_m"][f]), (name, f)
            assert np.array_equal(gv, c["out_v"][f]), (name, f)
        assert all(opt.t[g] == 7 for g in T.GROUPS)
        T.reset_opacity(new, opt, 0.01)
        torch.cuda.synchronize()
        got = np.stack([new.raw_opacity_a.cpu().numpy(), new.raw_opacity_b.cpu().numpy()], 1)
        if dtype == torch.float64:
            assert np.array_equal(got, c["reset"]), name
        else:
            np.testing.assert_allclose(got, c["reset"], rtol=1e-6, atol=1e-6)
        assert float(opt._m[5].abs().sum() + opt._v[6].abs().sum()) == 0.0
        assert opt.t["opacity_a"] == 0 and opt.t["opacity_b"] == 0 and opt.t["mu"] == 7


def test_densify_device_rng(cuda):
    """Philox split offsets: every row but the children's positions as with the
    reference's draws; the children's offsets in the parent frame look like
    N(0, 1) and differ between seeds."""
    from paper_2406_02720_b200 import trainer as T
    gold = load_golden("densify")
    c = A.densify_case(gold, "unlimited")
    outs = []
    for seed in (1, 2):
        scene, stats, opt, cfg = _setup(c, torch.float64)
        new, _, report = T.densify_and_prune(scene, stats, cfg, opt, seed, c["extent"])
        assert report == c["report"]
        outs.append({f: getattr(new, f).cpu().numpy() for f in A.FIELDS})
    nk = c["out"]["mu"].shape[0] - 2 * report["split"]
    for f in A.FIELDS:
        if f != "mu":
            assert np.array_equal(outs[0][f], c["out"][f]), f
    assert np.array_equal(outs[0]["mu"][:nk], c["out"]["mu"][:nk])
    assert not np.array_equal(outs[0]["mu"][nk:], outs[1]["mu"][nk:])
    # whiten the children's offsets: R^T (mu_child - mu_parent) / scale ~ N(0, 1)
    from oracle import oracle as O
    ks = report["split"]
    parent_rows = []
    p = c["params"]
    # parents are the split candidates in index order (unlimited budget)
    avg = np.where(c["stats"][2] > 0, c["stats"][0] / np.maximum(c["stats"][2], 1), 0.0)
    a1, a2 = O._sigmoid(p["raw_opacity_a"]), O._sigmoid(p["raw_opacity_b"])
    mx = np.exp(p["log_scale"]).max(axis=1)
    prune = (np.maximum(a1, a2) < 0.005) | (mx > 0.1 * c["extent"])
    parent_rows = np.nonzero((avg >= 2e-4) & ~prune & (mx > 0.01 * c["extent"]))[0]
    assert parent_rows.size == ks
    rot = O._quat_to_rot(p["rotation"][parent_rows])
    z = []
    for d in range(2):
        delta = outs[0]["mu"][nk + d * ks: nk + (d + 1) * ks] - p["mu"][parent_rows]
        local = np.einsum("nba,nb->na", rot, delta) / np.exp(p["log_scale"][parent_rows])
        z.append(local)
    z = np.concatenate(z).ravel()
    assert abs(z.mean()) < 0.15 and 0.8 < z.std() < 1.2, (z.mean(), z.std())


def test_densify_stats_update(cuda):
    from paper_2406_02720_b200 import device
    from paper_2406_02720_b200 import trainer as T
    from paper_2406_02720_b200.geometry import Scene
    rng = np.random.default_rng(3)
    n = 1000
    scene = Scene(rng.normal(size=(n, 3)), rng.normal(size=(n, 3)), rng.normal(size=(n, 4)),
                  rng.normal(size=(n, 4, 3)), rng.normal(size=(n, 3)), rng.normal(size=n),
                  rng.normal(size=n), sh_degree=1, device="cuda", dtype=torch.float32)
    g = device.DeviceGradientSet.empty_like_scene(scene)
    stats = T.DensifyStats.zeros(n)
    ref = [np.zeros(n), np.zeros((n, 3)), np.zeros(n, np.int64)]
    for _ in range(3):
        pg = rng.random(n).astype(np.float32)
        dm = rng.normal(size=(n, 3)).astype(np.float32)
        tc = rng.integers(0, 3, n).astype(np.int32)
        g.pos_grad_norm.copy_(torch.as_tensor(pg))
        g.d_mu.copy_(torch.as_tensor(dm))
        g.touch_count.copy_(torch.as_tensor(tc))
        stats.update(g)
        ref[0] += pg
        ref[1] += dm
        ref[2] += tc
    torch.cuda.synchronize()
    assert np.array_equal(stats.grad_sum.cpu().numpy(), ref[0])
    assert np.array_equal(stats.mu_grad_sum.cpu().numpy(), ref[1])
    assert np.array_equal(stats.count.cpu().numpy(), ref[2])
