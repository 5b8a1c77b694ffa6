"""The reference's own rasterizer properties (tests/test_rasterizer.py of the
reference) checked on the CPU oracle, so the checker itself is held to the
reference's semantics: bit-identical half==full for tied opacities, odd symmetry,
permutation and thread-count invariance, finite-difference gradients."""

import numpy as np
import pytest

from oracle import oracle as O
from paper_2406_02720_b200 import scenes
from paper_2406_02720_b200.geometry import CameraModel


def logit(p):
    return np.log(p) - np.log1p(-p)


def make_scene(rng, n=8, sh_degree=1, spread=0.5, z_lo=2.0, z_hi=4.0,
               background=(0.1, 0.15, 0.2), min_depth_gap=0.02):
    """Same recipe as the reference's make_scene (tests/test_rasterizer.py:17-40)."""
    while True:
        depths = np.sort(rng.uniform(z_lo, z_hi, n))
        if n == 1 or np.diff(depths).min() > min_depth_gap:
            break
    k = (sh_degree + 1) ** 2
    mu, ls, rot, sh, nrm, ra, rb = [], [], [], [], [], [], []
    for i in range(n):
        mu.append([rng.uniform(-spread, spread), rng.uniform(-spread, spread), depths[i]])
        ls.append(rng.uniform(np.log(0.05), np.log(0.25), 3))
        rot.append(rng.normal(size=4))
        sh.append(np.concatenate([rng.uniform(-0.8, 0.8, (1, 3)),
                                  rng.uniform(-0.2, 0.2, (k - 1, 3))]))
        v = rng.normal(size=3)
        nrm.append(v / np.linalg.norm(v))
        ra.append(logit(rng.uniform(0.15, 0.85)))
        rb.append(logit(rng.uniform(0.15, 0.85)))
    return scenes.SceneArrays(mu=np.array(mu), log_scale=np.array(ls), rotation=np.array(rot),
                              sh_coeffs=np.array(sh), normal=np.array(nrm),
                              raw_opacity_a=np.array(ra), raw_opacity_b=np.array(rb),
                              sh_degree=sh_degree, background_color=np.array(background))


def identity_camera(w=64, h=64, f=60.0):
    return CameraModel(np.eye(4), f, f, w / 2.0, h / 2.0, w, h)


def look_at(pos, target, w=64, h=64, f=60.0):
    return CameraModel.look_at(pos, target, w, h, f)


def tie(sa):
    out = scenes.SceneArrays(**{f: getattr(sa, f).copy() for f in sa.FIELDS},
                             sh_degree=sa.sh_degree, background_color=sa.background_color)
    out.raw_opacity_b = out.raw_opacity_a.copy()
    return out


def test_full_gaussian_equivalence_bit_identical():
    for seed in range(5):
        sa = tie(make_scene(np.random.default_rng(seed), 6))
        cam = look_at([0.3, -0.2, -0.5], [0, 0, 3.0])
        a = O.render(sa, cam, kernel="half")
        b = O.render(sa, cam, kernel="full")
        assert np.array_equal(a.color, b.color) and np.array_equal(a.depth, b.depth)


def test_odd_symmetry_bit_identical():
    for seed in range(5):
        sa = make_scene(np.random.default_rng(100 + seed), 6)
        fl = scenes.SceneArrays(**{f: getattr(sa, f).copy() for f in sa.FIELDS},
                                sh_degree=sa.sh_degree, background_color=sa.background_color)
        fl.normal = -fl.normal
        fl.raw_opacity_a, fl.raw_opacity_b = sa.raw_opacity_b.copy(), sa.raw_opacity_a.copy()
        cam = look_at([0.2, 0.1, -0.6], [0, 0, 3.0])
        assert np.array_equal(O.render(sa, cam).color, O.render(fl, cam).color)


def test_permutation_and_thread_invariance(rng):
    sa = make_scene(rng, 12)
    cam = identity_camera(80, 48)
    perm = rng.permutation(12)
    sp = scenes.SceneArrays(**{f: getattr(sa, f)[perm] for f in sa.FIELDS},
                            sh_degree=sa.sh_degree, background_color=sa.background_color)
    a = O.render(sa, cam, threads=1)
    assert np.array_equal(a.color, O.render(sp, cam, threads=1).color)
    assert np.array_equal(a.color, O.render(sa, cam, threads=4).color)


def test_transmittance_telescoping_and_background(rng):
    sa = make_scene(rng, 10)
    out = O.render(sa, identity_camera())
    assert np.abs(out.alpha + out.transmittance - 1.0).max() < 1e-6
    sa.raw_opacity_a[:] = -50.0
    sa.raw_opacity_b[:] = -50.0
    out = O.render(sa, identity_camera())
    assert np.allclose(out.color, sa.background_color, atol=1e-12)


def test_zero_cotangent_and_tied_normal_grad(rng):
    sa = make_scene(rng, 6)
    cam = identity_camera(32, 32)
    out = O.render(sa, cam)
    g = O.render_backward(sa, cam, out, np.zeros((32, 32, 3)))
    assert not any(g[k].any() for k in g if k not in ("touch_count",))
    st = tie(sa)
    out = O.render(st, cam)
    g = O.render_backward(st, cam, out, rng.uniform(-1, 1, (32, 32, 3)))
    assert np.abs(g["d_normal"]).max() == 0.0
    assert np.abs(g["d_raw_opacity_a"]).max() > 0.0


def test_gradients_match_finite_differences():
    """tests/test_rasterizer.py:220-226: every parameter group within 1e-3 of FD."""
    rng = np.random.default_rng(42)
    sa = make_scene(rng, 4, sh_degree=1, spread=0.4)
    cam = look_at([0.1, -0.2, -0.3], [0, 0, 3.0], 24, 24, 30.0)
    d_color = rng.uniform(-1.0, 1.0, (24, 24, 3))
    out = O.render(sa, cam, threads=1)
    g = O.render_backward(sa, cam, out, d_color, threads=1)
    names = {"mu": "d_mu", "log_scale": "d_log_scale", "rotation": "d_rotation",
             "sh_coeffs": "d_sh", "normal": "d_normal", "raw_opacity_a": "d_raw_opacity_a",
             "raw_opacity_b": "d_raw_opacity_b"}
    for field, gname in names.items():
        arr = getattr(sa, field)
        flat = arr.reshape(-1)
        an = g[gname].reshape(-1)
        for j in range(flat.shape[0]):
            h = 1e-4 * max(abs(flat[j]), 1.0)
            orig = flat[j]
            flat[j] = orig + h
            lp = float(np.sum(O.render(sa, cam, threads=1).color * d_color))
            flat[j] = orig - h
            lm = float(np.sum(O.render(sa, cam, threads=1).color * d_color))
            flat[j] = orig
            fd = (lp - lm) / (2 * h)
            rel = abs(an[j] - fd) / max(abs(an[j]), abs(fd), 1e-6)
            assert rel <= 1e-3, (field, j, an[j], fd)


def test_culled_bookkeeping(rng):
    sa = make_scene(rng, 5)
    sa.mu[0, 2] = -5.0
    cam = identity_camera(32, 32)
    out = O.render(sa, cam)
    g = O.render_backward(sa, cam, out, rng.uniform(-1, 1, (32, 32, 3)))
    assert g["touch_count"][0] == 0 and g["pos_grad_norm"][0] == 0.0
    assert (g["touch_count"][1:] == 1).all()


@pytest.mark.parametrize("lo,hi", [(0, 7), (7, 30), (30, 48)])
def test_blend_core_tile_ranges(lo, hi):
    """forward_tiles/backward_tiles write only tiles [lo, hi) (Seam 1 contract)."""
    sa = scenes.frustum(400, 1, 96, 128, seed=8).as_float64()
    cam = CameraModel(**sa.cameras[0])
    full = O.render(sa, cam)
    f = full.frame
    h, w = cam.height, cam.width
    color = np.full((h, w, 3), -1.0)
    alpha, depth, trans = (np.full((h, w), -1.0) for _ in range(3))
    term = np.full((h, w), -7, np.int32)
    O.forward_tiles(f.packed, f.mode, f.pair_splat, f.tile_starts, h, w, f.tiles_x,
                    np.asarray(sa.background_color), color, alpha, depth, trans, term, lo, hi)
    mask = np.zeros((h, w), bool)
    for t in range(lo, hi):
        ty, tx = divmod(t, f.tiles_x)
        mask[ty * 16:(ty + 1) * 16, tx * 16:(tx + 1) * 16] = True
    assert np.array_equal(color[mask], full.color[mask])
    assert (term[~mask] == -7).all()
