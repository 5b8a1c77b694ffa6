"""screen_splats (rasterizer.py:578-603) and the reference's closed-form single
splat test (tests/test_rasterizer.py:59-80) on the GPU path."""

import numpy as np
import pytest

from test_oracle_properties import identity_camera, make_scene
from paper_2406_02720_b200 import rasterizer as R
from paper_2406_02720_b200 import scenes

pytestmark = pytest.mark.gpu


def logit(p):
    return float(np.log(p) - np.log1p(-p))


def paired_response(conic, mu_hat, n_ray, a1, a2, whiten2d, pixel):
    """kernels.py:185-197 (closed form of the half-Gaussian pair at one pixel)."""
    from oracle import oracle as O
    d = np.asarray(pixel, dtype=np.float64) - mu_hat
    g = np.exp(-0.5 * (d @ conic @ d))
    u = whiten2d @ d
    m = n_ray[0] * u[0] + n_ray[1] * u[1]
    n3 = abs(n_ray[2])
    e = float(np.sign(m)) if n3 < 1e-6 else O.erf(m / (np.sqrt(2.0) * n3))
    w = 0.5 * ((a1 + a2) + (a1 - a2) * e) * g
    return float(np.clip(w, 0.0, 0.99))


def test_single_centered_splat_matches_closed_form(cuda):
    sa = scenes.SceneArrays(
        mu=np.array([[0.0, 0.0, 2.0]]), log_scale=np.log([[0.3, 0.3, 0.3]]),
        rotation=np.array([[1.0, 0.0, 0.0, 0.0]]), sh_coeffs=np.array([[[1.0, -0.5, -0.5]]]),
        normal=np.array([[0.0, 0.0, 1.0]]), raw_opacity_a=np.array([logit(0.99)]),
        raw_opacity_b=np.array([logit(0.99)]), sh_degree=0,
        background_color=np.zeros(3))
    cam = identity_camera(64, 64, 60.0)
    out = R.render(sa, cam)
    splat = R.screen_splats(sa, cam)[0]
    w = paired_response(splat.conic, splat.mu_hat, splat.n_ray, splat.alpha1, splat.alpha2,
                        splat.whiten2d, [32.5, 32.5])
    # FP32 blend vs the FP64 closed form
    np.testing.assert_allclose(out.color[32, 32], splat.rgb * w, atol=2e-6)
    assert abs(out.alpha[32, 32] - w) < 2e-6 and out.alpha[32, 32] > 0.9


def test_screen_splats_fields_match_oracle_packed(cuda):
    from oracle import oracle as O
    rng = np.random.default_rng(5)
    sa = make_scene(rng, 30, sh_degree=2)
    cam = identity_camera(80, 64)
    ss = R.screen_splats(sa, cam)
    f = O.prepare(sa, cam)
    assert [s.prim_index for s in ss] == list(f.valid)
    for s, row in zip(ss, f.packed):
        np.testing.assert_allclose(s.mu_hat, row[0:2], rtol=1e-12)
        np.testing.assert_allclose([s.conic[0, 0], s.conic[0, 1], s.conic[1, 1]], row[2:5],
                                   rtol=1e-9)
        np.testing.assert_allclose(s.rgb, row[9:12], rtol=1e-12, atol=1e-15)
        assert abs(s.depth - row[12]) < 1e-12
        assert abs(np.linalg.norm(s.n_ray) - 1.0) < 1e-12
        assert 0.0 < s.alpha1 < 1.0 and 0.0 < s.alpha2 < 1.0
        c1 = 0.5 * (s.alpha1 + s.alpha2)
        assert abs(c1 - row[7]) < 1e-12
