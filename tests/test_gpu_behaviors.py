"""Behavioural properties the reference's own rasterizer tests check
(tests/test_rasterizer.py of the reference), run against the GPU path through the
drop-in API: background-only renders, culling, permutation invariance,
telescoping transmittance, and the depth-normal-map post-process."""

import numpy as np
import pytest

pytestmark = pytest.mark.gpu


class _Scene:
    FIELDS = ("mu", "log_scale", "rotation", "sh_coeffs", "normal", "raw_opacity_a",
              "raw_opacity_b")

    def __init__(self, **kw):
        for k, v in kw.items():
            setattr(self, k, v)

    def take(self, idx):
        return _Scene(**{f: getattr(self, f)[idx].copy() for f in self.FIELDS},
                      sh_degree=self.sh_degree, background_color=self.background_color)


def _logit(p):
    return np.log(p) - np.log1p(-p)


def _scene(rng, n=8, deg=1, spread=0.5, bg=(0.1, 0.15, 0.2)):
    """Random scene with depths at least 0.02 apart (a stable blend order)."""
    while True:
        z = np.sort(rng.uniform(2.0, 4.0, n))
        if n == 1 or np.diff(z).min() > 0.02:
            break
    k = (deg + 1) ** 2
    nrm = rng.normal(size=(n, 3))
    return _Scene(mu=np.column_stack([rng.uniform(-spread, spread, (n, 2)), z]),
                  log_scale=rng.uniform(np.log(0.05), np.log(0.25), (n, 3)),
                  rotation=rng.normal(size=(n, 4)),
                  sh_coeffs=np.concatenate([rng.uniform(-0.8, 0.8, (n, 1, 3)),
                                            rng.uniform(-0.2, 0.2, (n, k - 1, 3))], axis=1),
                  normal=nrm / np.linalg.norm(nrm, axis=1, keepdims=True),
                  raw_opacity_a=_logit(rng.uniform(0.15, 0.85, n)),
                  raw_opacity_b=_logit(rng.uniform(0.15, 0.85, n)),
                  sh_degree=deg, background_color=np.array(bg))


def _cam(w=64, h=64, f=60.0):
    from paper_2406_02720_b200.geometry import CameraModel
    return CameraModel(world_to_cam=np.eye(4), fx=f, fy=f, cx=w / 2, cy=h / 2, width=w,
                       height=h)


def test_zero_opacity_renders_background(cuda):
    from paper_2406_02720_b200 import rasterizer as R
    sc = _scene(np.random.default_rng(0), 4)
    sc.raw_opacity_a[:] = -50.0
    sc.raw_opacity_b[:] = -50.0
    out = R.render(sc, _cam())
    assert np.array_equal(out.color, np.broadcast_to(sc.background_color.astype(np.float32),
                                                     out.color.shape))
    assert np.all(out.alpha == 0.0)


def test_behind_camera_culled(cuda):
    from paper_2406_02720_b200 import rasterizer as R
    sc = _scene(np.random.default_rng(1), 3)
    sc.mu[:, 2] = -1.0
    out = R.render(sc, _cam())
    assert np.allclose(out.color, sc.background_color, atol=1e-7)
    assert np.all(out.radii == 0)


def test_transmittance_telescoping(cuda):
    from paper_2406_02720_b200 import rasterizer as R
    out = R.render(_scene(np.random.default_rng(2), 10), _cam())
    assert np.abs(out.alpha + out.transmittance - 1.0).max() < 1e-6


def test_permutation_invariance_bitwise(cuda):
    """Reordering the primitives reorders nothing on screen: images bit-identical,
    gradients permuted bit-identically (the blend order is depth, then index)."""
    from paper_2406_02720_b200 import rasterizer as R
    rng = np.random.default_rng(3)
    sc = _scene(rng, 8)
    perm = rng.permutation(8)
    cam = _cam(80, 48)
    d_color = rng.uniform(-1, 1, (48, 80, 3))
    a, b = R.render(sc, cam), R.render(sc.take(perm), cam)
    assert np.array_equal(a.color, b.color) and np.array_equal(a.depth, b.depth)
    ga = R.render_backward(sc, cam, a, d_color)
    gb = R.render_backward(sc.take(perm), cam, b, d_color)
    for name in ("d_mu", "d_log_scale", "d_rotation", "d_sh", "d_normal", "d_raw_opacity_a",
                 "d_raw_opacity_b", "touch_count"):
        assert np.array_equal(getattr(ga, name)[perm], getattr(gb, name)), name


def test_depth_normalmap_planes_and_mask(cuda):
    """render_depth_normalmap (rasterizer.py:606-642) on analytic plane depths."""
    from paper_2406_02720_b200 import rasterizer as R

    class Out:
        pass

    wh = 48
    cam = _cam(wh, wh, 40.0)
    ys, xs = np.mgrid[0:wh, 0:wh]
    dirs = np.stack([(xs + 0.5 - cam.cx) / cam.fx, (ys + 0.5 - cam.cy) / cam.fy,
                     np.ones((wh, wh))], axis=-1)
    for n, tol in (([0.0, 0.0, 1.0], 0.02), ([np.sqrt(0.5), 0.0, np.sqrt(0.5)], 0.05)):
        n = np.asarray(n)
        o = Out()
        o.depth, o.alpha, o.camera = (n[2] * 2.0) / (dirs @ n), np.ones((wh, wh)), cam
        normals = R.render_depth_normalmap(o)
        inner = normals[14:-14, 14:-14]
        if n[0] == 0.0:
            assert np.abs(inner - np.array([0.0, 0.0, -1.0])).max() < tol
        else:
            assert np.abs(np.abs(inner[..., 2]) - np.cos(np.pi / 4)).max() < tol
    sc = _scene(np.random.default_rng(4), 2)
    sc.raw_opacity_a[:] = -50
    sc.raw_opacity_b[:] = -50
    assert not R.render_depth_normalmap(R.render(sc, _cam(32, 32))).any()


@pytest.mark.parametrize("wh", [(1, 1), (15, 17), (33, 2)])
def test_tiny_and_ragged_images_vs_oracle(cuda, wh):
    """Images smaller than a tile and ragged edges: same integers, images and
    gradients as the oracle."""
    from oracle import oracle as O
    from paper_2406_02720_b200 import rasterizer as R
    w, h = wh
    sc = _scene(np.random.default_rng(7), 12, spread=0.2)
    cam = _cam(w, h, 20.0)
    ref = O.render(sc, cam)
    out = R.render(sc, cam)
    np.testing.assert_allclose(out.color, ref.color, atol=1e-5)
    assert np.array_equal(out.per_pixel_terminal_index, ref.per_pixel_terminal_index)
    d = np.random.default_rng(1).uniform(-1, 1, (h, w, 3))
    g = R.render_backward(sc, cam, out, d)
    rg = O.render_backward(sc, cam, ref, d)
    for name in ("d_mu", "d_log_scale", "d_rotation", "d_sh", "d_normal", "d_raw_opacity_a",
                 "d_raw_opacity_b"):
        a, b = getattr(g, name), rg[name]
        assert np.linalg.norm(a - b) <= 1e-3 * max(np.linalg.norm(b), 1e-12), name


def test_everything_culled(cuda):
    """No pair at all (P = 0): background image, zero gradients, zero touch counts."""
    from paper_2406_02720_b200 import rasterizer as R
    sc = _scene(np.random.default_rng(8), 5)
    sc.mu[:, 0] += 100.0  # far off screen
    cam = _cam(40, 24)
    out = R.render(sc, cam)
    assert np.allclose(out.color, sc.background_color, atol=1e-7)
    g = R.render_backward(sc, cam, out, np.ones((24, 40, 3)))
    assert not g.d_mu.any() and not g.d_sh.any() and not g.touch_count.any()
