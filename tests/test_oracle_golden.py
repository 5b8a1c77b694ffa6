"""Pin the CPU oracle against outputs of the reference itself (tests/golden/,
produced by tests/golden/make_golden.py from /root/reference).  CPU only."""

import hashlib
import os

import numpy as np
import pytest

from conftest import load_golden
from oracle import oracle as O
from paper_2406_02720_b200 import scenes

FULL = {
    "c1": (lambda: scenes.make_config("c1"), "half"),
    "mini": (lambda: scenes.frustum(300, 2, 64, 48, seed=3), "half"),
    "mini_full": (lambda: scenes.frustum(300, 2, 64, 48, seed=3), "full"),
    "ball_small": (lambda: scenes.ball(3000, 3, 96, 72, views=4, seed=9), "half"),
    "ties": (lambda: scenes.frustum(2000, 1, 96, 80, seed=5, clustered=True, dup=0.3), "half"),
}
INTS = {"valid": np.int64, "mode": np.int8, "tile_rect": np.int32, "pair_splat": np.int32,
        "tile_starts": np.int64}
GRADS = ("d_mu", "d_log_scale", "d_rotation", "d_sh", "d_normal", "d_raw_opacity_a",
         "d_raw_opacity_b", "pos_grad_norm")


class Cam:
    def __init__(self, kw):
        for k, v in kw.items():
            setattr(self, k, v)
        self.near_clip = 0.01


def test_erf_matches_reference_bitwise():
    gold = load_golden("erf")
    got = np.array([O.erf(z) for z in gold["z"]])
    assert np.array_equal(got, gold["erf"])
    # exactly odd (kernels.py:136-147 relies on it)
    assert all(O.erf(-z) == -O.erf(z) for z in gold["z"][:500])


@pytest.mark.parametrize("name", list(FULL))
def test_oracle_full_fixture(name):
    gold = load_golden(name)
    gen, kernel = FULL[name]
    sa = gen().as_float64()
    cam = Cam(sa.cameras[int(gold["cam_idx"])])
    out = O.render(sa, cam, kernel=kernel, threads=4)
    f = out.frame
    for k, dt in INTS.items():
        assert np.array_equal(np.asarray(getattr(f, k), dtype=dt), gold[k]), k
    assert np.array_equal(f.radii, gold["radii"]), "radii"
    # packed: only libm-vs-numpy `exp` ulps separate the two
    np.testing.assert_allclose(f.packed, gold["packed"], rtol=1e-9, atol=1e-12)
    for k in ("color", "alpha", "depth", "transmittance"):
        np.testing.assert_allclose(getattr(out, k), gold[k], rtol=0, atol=1e-11)
    assert np.array_equal(out.per_pixel_terminal_index, gold["terminal"])
    if "d_color" in gold:
        g = O.render_backward(sa, cam, out, gold["d_color"], threads=4)
        for k in GRADS:
            den = max(np.linalg.norm(gold[k]), 1e-300)
            assert np.linalg.norm(g[k] - gold[k]) / den < 1e-9, k
        assert np.array_equal(g["touch_count"], gold["touch_count"])


def _sha(a, dt):
    return hashlib.sha256(np.ascontiguousarray(a, dtype=dt).tobytes()).hexdigest()


def test_oracle_c2_summary():
    """Full c2 (100k, SH3, 800x800): integer hashes, sampled pixels, gradients."""
    gold = load_golden("c2")
    sa = scenes.make_config("c2").as_float64()
    cam = Cam(sa.cameras[0])
    out = O.render(sa, cam)
    f = out.frame
    for k, dt in INTS.items():
        assert _sha(getattr(f, k), dt) == str(gold[f"sha_{k}"]), k
    assert _sha(f.radii, np.int32) == str(gold["sha_radii"]), "radii"
    px = gold["px_index"]
    np.testing.assert_allclose(out.color.reshape(-1, 3)[px], gold["px_color"], atol=1e-11)
    assert np.array_equal(out.per_pixel_terminal_index.reshape(-1)[px], gold["px_terminal"])
    assert _sha(out.per_pixel_terminal_index, np.int32) == str(gold["terminal_sha"])
    g = O.render_backward(sa, cam, out, scenes.cotangent(cam.height, cam.width))
    rows = gold["grad_rows"]
    for k in GRADS:
        assert abs(np.linalg.norm(g[k]) - float(gold[f"norm_{k}"])) <= 1e-9 * float(gold[f"norm_{k}"])
        ref = gold[f"sample_{k}"]
        assert np.linalg.norm(g[k][rows] - ref) <= 1e-9 * max(np.linalg.norm(ref), 1e-300), k


def test_oracle_c3_binning_hashes():
    """Headline config c3 (1M, 1080p): the oracle's FrameGeometry integers hash
    to the reference's; counts match SURVEY.md 8(d)."""
    gold = load_golden("c3")
    sa = scenes.make_config("c3").as_float64()
    f = O.prepare(sa, Cam(sa.cameras[0]))
    assert f.valid.shape[0] == int(gold["M"]) == 846_464
    assert f.pair_splat.shape[0] == int(gold["P"]) == 3_384_553
    for k, dt in INTS.items():
        assert _sha(getattr(f, k), dt) == str(gold[f"sha_{k}"]), k


@pytest.mark.slow
@pytest.mark.skipif(not os.environ.get("HS_SLOW"), reason="set HS_SLOW=1 (minutes, ~10 GB)")
@pytest.mark.parametrize("name,cfg", [("c5", "c5"), ("c4v0", "c4")])
def test_oracle_large_binning_hashes(name, cfg):
    gold = load_golden(name)
    sa = scenes.make_config(cfg).as_float64()
    f = O.prepare(sa, Cam(sa.cameras[0]))
    for k, dt in INTS.items():
        assert _sha(getattr(f, k), dt) == str(gold[f"sha_{k}"]), k


def test_loss_oracle_matches_reference():
    """compute_loss / ssim_with_grad (loss.py:48-106): the oracle's gradients
    are bit-identical to the reference's; the scalars differ only by the
    summation order of the means (numpy pairwise vs sequential)."""
    gold = load_golden("loss")
    for c in gold["cases"]:
        a, b, lam = gold[f"{c}_a"], gold[f"{c}_b"], float(gold[f"{c}_lambda"])
        loss, grad = O.compute_loss(a, b, lam)
        assert grad.shape == gold[f"{c}_grad"].shape, c
        assert np.array_equal(grad, gold[f"{c}_grad"]), c
        assert loss == pytest.approx(float(gold[f"{c}_loss"]), rel=1e-12, abs=1e-15), c
        if lam > 0:
            s, sg = O.ssim_with_grad(a, b)
            assert sg.shape == gold[f"{c}_ssim_grad"].shape, c
            assert np.array_equal(sg, gold[f"{c}_ssim_grad"]), c
            assert s == pytest.approx(float(gold[f"{c}_ssim"]), rel=1e-12), c
    s, _ = O.ssim_with_grad(gold["same_l02_a"], gold["same_l02_a"])
    assert s == 1.0


def test_loss_oracle_float64_inputs():
    """The oracle on float64 / uint8 inputs float32 cannot hold (loss64.npz)."""
    gold = load_golden("loss64")
    for c in gold["cases"]:
        a, b, lam = gold[f"{c}_a"], gold[f"{c}_b"], float(gold[f"{c}_lambda"])
        loss, grad = O.compute_loss(a, b, lam)
        assert np.array_equal(grad, gold[f"{c}_grad"]), c
        assert loss == pytest.approx(float(gold[f"{c}_loss"]), rel=1e-12, abs=1e-15), c


def test_adam_oracle_matches_reference():
    """OracleAdam (trainer.py:192-224 restated) steps the reference's scenes
    bit-identically, including frozen groups, the 'full' tie, zero-gradient
    rows and the normal renormalisation."""
    import adam_cases as A
    from paper_2406_02720_b200 import trainer as T
    gold = load_golden("adam")
    for name in gold["cases"]:
        deg, kw, params, steps, t_ref = A.case(gold, name)
        cfg = A.config(kw)
        opt = O.OracleAdam(params)
        for it, (iteration, grads, after) in enumerate(steps):
            lrs = T.learning_rates(cfg, iteration, A.SPATIAL_SCALE)
            enabled = T.active_groups(cfg)
            lrs = {g: (lr if g in enabled else 0.0) for g, lr in lrs.items()}
            opt.step(params, grads, lrs, cfg.kernel == "full")
            for f in A.FIELDS:
                assert np.array_equal(params[f], after[f]), (name, it, f)
        assert [opt.t[g] for g in O.ADAM_GROUPS] == list(t_ref), name


def test_densify_oracle_matches_reference():
    """densify_and_prune / reset_opacity restated in numpy reproduce the
    reference's new scenes, re-aligned moments and reports bit for bit."""
    import adam_cases as A
    gold = load_golden("densify")
    for name in gold["cases"]:
        c = A.densify_case(gold, name)
        cfg = dict(A.DENSIFY_CFG, max_primitives=c["max_primitives"])
        new, nm, nv, report = O.densify_and_prune(
            {f: a.copy() for f, a in c["params"].items()}, *c["stats"], c["m"], c["v"], cfg,
            c["extent"], np.random.default_rng(c["seed"]))
        assert report == c["report"], name
        for f in A.FIELDS:
            assert np.array_equal(new[f], c["out"][f]), (name, f)
            assert np.array_equal(nm[f], c["out_m"][f]), (name, f)
            assert np.array_equal(nv[f], c["out_v"][f]), (name, f)
        O.reset_opacity(new, 0.01)
        assert np.array_equal(np.stack([new["raw_opacity_a"], new["raw_opacity_b"]], 1),
                              c["reset"]), name
