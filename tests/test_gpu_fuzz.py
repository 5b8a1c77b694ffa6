"""Randomised parity sweep: many small scenes with randomly drawn generator
parameters (size, SH degree, opacity and scale ranges, clustered/duplicated
depths, extreme splitting normals, camera pose, kernel, dtype), each against
the FP64 oracle under the parity contract of tests/parity.py.  Seeded, so a
failure reproduces (96 scenes, ~10 s on a B200)."""

import numpy as np
import pytest
import torch

from parity import assert_grads, assert_images
from test_gpu_parity import run_gpu

from paper_2406_02720_b200 import scenes

pytestmark = pytest.mark.gpu

INT_KEYS = ("valid", "tile_rect", "mode", "pair_splat", "tile_starts")


def _draw(seed):
    rng = np.random.default_rng(1000 + seed)
    w = int(rng.integers(16, 200))
    h = int(rng.integers(16, 160))
    n = int(rng.integers(50, 3000))
    sh = int(rng.integers(0, 4))
    kind = rng.choice(["frustum", "ball"])
    if kind == "frustum":
        sa = scenes.frustum(n, sh, w, h, seed=seed, sig_lo=float(rng.uniform(0.3, 2.0)),
                            sig_hi=float(rng.uniform(2.5, 20.0)),
                            clustered=bool(rng.random() < 0.3),
                            dup=float(rng.choice([0.0, 0.2])))
        cam_idx = 0
    else:
        sa = scenes.ball(n, sh, w, h, views=4, seed=seed)
        cam_idx = int(rng.integers(0, 4))
    # opacities from nearly transparent to nearly opaque (exercises termination and
    # the 0.99 clamp), and a share of near-edge-on splitting normals (steep / sign)
    lo, hi = sorted(rng.uniform(0.01, 0.999, 2))
    p = rng.uniform(lo, hi, (2, len(sa.mu)))
    sa.raw_opacity_a[:] = np.log(p[0]) - np.log1p(-p[0])
    sa.raw_opacity_b[:] = np.log(p[1]) - np.log1p(-p[1])
    if rng.random() < 0.5:
        w2c = np.asarray(sa.cameras[cam_idx]["world_to_cam"], dtype=np.float64)
        m = sa.mu.astype(np.float64) + w2c[:3, :3].T @ w2c[:3, 3]  # mu - camera centre
        ray = m / np.linalg.norm(m, axis=1, keepdims=True)
        perp = np.cross(ray, rng.normal(size=ray.shape))
        perp /= np.linalg.norm(perp, axis=1, keepdims=True)
        pick = rng.random(len(m)) < 0.3
        tilt = 10.0 ** rng.uniform(-7, -1, len(m))
        nrm = np.where(pick[:, None], perp + tilt[:, None] * ray, sa.normal)
        sa.normal[:] = (nrm / np.linalg.norm(nrm, axis=1, keepdims=True)).astype(np.float32)
    kernel = "full" if rng.random() < 0.2 else "half"
    dtype = torch.float64 if rng.random() < 0.3 else torch.float32
    return sa, cam_idx, kernel, dtype


@pytest.mark.parametrize("seed", range(96))
def test_random_scene_vs_oracle(cuda, seed):
    from oracle import oracle as O
    from paper_2406_02720_b200.geometry import CameraModel
    sa, cam_idx, kernel, dtype = _draw(seed)
    s64 = sa.as_float64()
    cam = CameraModel(**sa.cameras[cam_idx])
    d_color = np.random.default_rng(seed).uniform(-1, 1, (cam.height, cam.width, 3))
    ref_out = O.render(s64, cam, kernel=kernel)
    ref_g = O.render_backward(s64, cam, ref_out, d_color)
    got = run_gpu(sa, cam_idx, kernel, dtype, d_color)
    f = ref_out.frame
    for k in INT_KEYS:
        assert np.array_equal(np.asarray(got[k]), np.asarray(getattr(f, k))), (seed, k)
    ref = {"color": ref_out.color, "alpha": ref_out.alpha, "depth": ref_out.depth,
           "transmittance": ref_out.transmittance,
           "terminal": ref_out.per_pixel_terminal_index}
    assert_images(got, ref)
    assert_grads(got, ref_g)
