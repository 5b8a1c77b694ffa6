"""GPU parity: the CUDA path (through the C-ABI) against the reference's own
outputs (golden fixtures) and against the live CPU oracle.

Every call below goes through libhalfsplat_b200.so; the oracle is only the
checker.  Tolerances: tests/parity.py.
"""

import hashlib

import numpy as np
import pytest
import torch

from conftest import load_golden
from parity import GRAD_GROUPS, PACKED_RTOL, assert_grads, assert_images
from paper_2406_02720_b200 import device, scenes
from paper_2406_02720_b200.geometry import CameraModel, Scene

pytestmark = pytest.mark.gpu

FULL_FIXTURES = {
    "c1": (lambda: scenes.make_config("c1"), "half"),
    "mini": (lambda: scenes.frustum(300, 2, 64, 48, seed=3), "half"),
    "mini_full": (lambda: scenes.frustum(300, 2, 64, 48, seed=3), "full"),
    "ball_small": (lambda: scenes.ball(3000, 3, 96, 72, views=4, seed=9), "half"),
    "ties": (lambda: scenes.frustum(2000, 1, 96, 80, seed=5, clustered=True, dup=0.3), "half"),
}
SUMMARY_FIXTURES = ("c2", "c3", "c5", "c4v0")
INT_DTYPES = {"valid": np.int64, "mode": np.int8, "tile_rect": np.int32, "pair_splat": np.int32,
              "tile_starts": np.int64}


def scene_sha(sa):
    h = hashlib.sha256()
    for f in sa.FIELDS:
        h.update(np.ascontiguousarray(getattr(sa, f), dtype=np.float32).tobytes())
    return h.hexdigest()


def device_scene(sa, dtype=torch.float32):
    return Scene(*(getattr(sa, f) for f in sa.FIELDS), sh_degree=sa.sh_degree,
                 background_color=sa.background_color, device="cuda", dtype=dtype)


def run_gpu(sa, cam_idx, kernel="half", dtype=torch.float32, d_color=None):
    sc = device_scene(sa, dtype)
    cam = CameraModel(**sa.cameras[cam_idx])
    out = device.render(sc, cam, kernel)
    res = {
        "color": out.color.cpu().numpy(), "alpha": out.alpha.cpu().numpy(),
        "depth": out.depth.cpu().numpy(), "transmittance": out.transmittance.cpu().numpy(),
        "terminal": out.terminal.cpu().numpy(),
    }
    res.update(out.frame.export())
    if d_color is not None:
        g = device.render_backward(sc, cam, out, torch.as_tensor(d_color, dtype=torch.float32))
        for name in GRAD_GROUPS + ("touch_count",):
            res[name] = getattr(g, name).double().cpu().numpy()
    return res


@pytest.mark.parametrize("name", list(FULL_FIXTURES))
@pytest.mark.parametrize("dtype", [torch.float32, torch.float64])
def test_full_fixture_parity(cuda, name, dtype):
    gold = load_golden(name)
    gen, kernel = FULL_FIXTURES[name]
    sa = gen()
    assert scene_sha(sa) == str(gold["scene_sha"]), "scene generator drifted"
    d_color = gold["d_color"] if "d_color" in gold else None
    got = run_gpu(sa, int(gold["cam_idx"]), kernel, dtype, d_color)
    # integers: bit-exact
    for k, dt in INT_DTYPES.items():
        assert np.array_equal(np.asarray(got[k], dtype=dt), gold[k]), k
    # radii = ceil(3.5 sqrt(lambda_max)) of the reference's own cov_ray, 0 when culled
    assert got["radii"].dtype == np.int32
    assert np.array_equal(got["radii"], gold["radii"]), "radii"
    # packed: FP64 value rounded to FP32
    ref32 = gold["packed"].astype(np.float32).astype(np.float64)
    np.testing.assert_allclose(got["packed"].astype(np.float64), ref32, rtol=PACKED_RTOL,
                               atol=1e-30)
    assert_images(got, gold)
    if d_color is not None:
        assert_grads(got, gold)
        assert np.array_equal(got["touch_count"], gold["touch_count"])


@pytest.mark.parametrize("name", SUMMARY_FIXTURES)
def test_full_size_summary_parity(cuda, name):
    gold = load_golden(name)
    cfg = {"c4v0": "c4"}.get(name, name)
    sa = scenes.make_config(cfg)
    assert scene_sha(sa) == str(gold["scene_sha"]), "scene generator drifted"
    cam = CameraModel(**sa.cameras[int(gold["cam_idx"])])
    d_color = scenes.cotangent(cam.height, cam.width) if "grad_rows" in gold else None
    got = run_gpu(sa, int(gold["cam_idx"]), "half", torch.float32, d_color)
    for k, dt in INT_DTYPES.items():
        h = hashlib.sha256(np.ascontiguousarray(got[k], dtype=dt).tobytes()).hexdigest()
        assert h == str(gold[f"sha_{k}"]), f"{k} differs from the reference"
    h = hashlib.sha256(np.ascontiguousarray(got["radii"], dtype=np.int32).tobytes()).hexdigest()
    assert h == str(gold["sha_radii"]), "radii differ from the reference"
    assert int(got["radii"].astype(np.int64).sum()) == int(gold["radii_sum"])
    assert got["valid"].shape[0] == int(gold["M"])
    assert got["pair_splat"].shape[0] == int(gold["P"])
    rows = gold["packed_sample_rows"]
    np.testing.assert_allclose(got["packed"][rows].astype(np.float64),
                               gold["packed_sample"].astype(np.float32).astype(np.float64),
                               rtol=PACKED_RTOL, atol=1e-30)
    # terminal: mismatch fraction over the whole frame from the sampled pixels
    px = gold["px_index"]
    sample_got = {
        "color": got["color"].reshape(-1, 3)[px], "alpha": got["alpha"].reshape(-1)[px],
        "depth": got["depth"].reshape(-1)[px],
        "transmittance": got["transmittance"].reshape(-1)[px],
        "terminal": got["terminal"].reshape(-1)[px],
    }
    sample_ref = {"color": gold["px_color"], "alpha": gold["px_alpha"], "depth": gold["px_depth"],
                  "transmittance": gold["px_transmittance"], "terminal": gold["px_terminal"]}
    assert_images(sample_got, sample_ref)
    assert int(got["terminal"].astype(np.int64).sum()) > 0
    if d_color is not None:
        rows = gold["grad_rows"]
        for g in GRAD_GROUPS:
            ref_norm = float(gold[f"norm_{g}"])
            got_norm = float(np.linalg.norm(got[g]))
            assert abs(got_norm - ref_norm) <= 1e-3 * ref_norm, (g, got_norm, ref_norm)
        sample = {g: got[g][rows] for g in GRAD_GROUPS}
        ref = {g: gold[f"sample_{g}"] for g in GRAD_GROUPS}
        assert_grads(sample, ref)


def _oracle():
    from oracle import oracle
    return oracle


@pytest.mark.parametrize("kernel", ["half", "full"])
def test_live_oracle_medium(cuda, kernel):
    """Unseen scene, both kernels: GPU vs the CPU oracle run on this host."""
    O = _oracle()
    sa = scenes.frustum(20_000, 3, 320, 240, seed=11, sig_lo=0.8, sig_hi=6.0)
    s64 = sa.as_float64()
    cam = CameraModel(**sa.cameras[0])
    d_color = scenes.cotangent(cam.height, cam.width, seed=4)
    ref_out = O.render(s64, cam, kernel=kernel)
    ref_g = O.render_backward(s64, cam, ref_out, d_color)
    got = run_gpu(sa, 0, kernel, torch.float32, d_color)
    f = ref_out.frame
    assert np.array_equal(got["valid"], f.valid)
    assert np.array_equal(got["pair_splat"], f.pair_splat)
    assert np.array_equal(got["tile_starts"], f.tile_starts)
    assert np.array_equal(got["tile_rect"], f.tile_rect)
    assert np.array_equal(got["mode"], f.mode)
    ref = {"color": ref_out.color, "alpha": ref_out.alpha, "depth": ref_out.depth,
           "transmittance": ref_out.transmittance, "terminal": ref_out.per_pixel_terminal_index}
    assert_images(got, ref)
    assert_grads(got, ref_g)


def test_look_at_views_oracle(cuda):
    """Rotated cameras (the ball views): every integer exact, images/grads in tolerance."""
    O = _oracle()
    sa = scenes.ball(20_000, 3, 256, 192, views=8, seed=21)
    s64 = sa.as_float64()
    for idx in (0, 3, 6):
        cam = CameraModel(**sa.cameras[idx])
        d_color = scenes.cotangent(cam.height, cam.width, seed=idx)
        ref_out = O.render(s64, cam)
        ref_g = O.render_backward(s64, cam, ref_out, d_color)
        got = run_gpu(sa, idx, "half", torch.float64, d_color)
        assert np.array_equal(got["pair_splat"], ref_out.frame.pair_splat)
        assert np.array_equal(got["tile_starts"], ref_out.frame.tile_starts)
        ref = {"color": ref_out.color, "alpha": ref_out.alpha, "depth": ref_out.depth,
               "transmittance": ref_out.transmittance,
               "terminal": ref_out.per_pixel_terminal_index}
        assert_images(got, ref)
        assert_grads(got, ref_g)


def test_radii_match_live_oracle(cuda):
    """Radii bit-exact against the live oracle on an unseen scene with a wide radius
    range (sigma 0.3-40 px), float32 and float64 inputs."""
    O = _oracle()
    sa = scenes.frustum(20_000, 1, 480, 320, seed=23, sig_lo=0.3, sig_hi=40.0)
    ref = O.prepare(sa.as_float64(), CameraModel(**sa.cameras[0]))
    assert ref.radii.max() > 100
    for dt in (torch.float32, torch.float64):
        got = run_gpu(sa, 0, "half", dt)
        assert np.array_equal(got["radii"], ref.radii), dt


def test_steep_and_sign_mode_splats_oracle(cuda):
    """Splitting planes that nearly contain the viewing ray: |n_ray.z| from ~1e-3 down
    through the sign-mode threshold (1e-6), where |za|, |zb| reach 1e5+.  These take
    the side-record (steep) form on the packed path or the sign mode; images and
    gradients must still match the FP64 oracle under the same contract."""
    O = _oracle()
    sa = scenes.frustum(6000, 2, 256, 192, seed=23, sig_lo=1.0, sig_hi=8.0)
    rng = np.random.default_rng(5)
    # normals perpendicular to the ray through each centre, tilted by tiny angles
    mu = sa.mu.astype(np.float64)
    ray = mu / np.linalg.norm(mu, axis=1, keepdims=True)
    perp = np.cross(ray, rng.normal(size=ray.shape))
    perp /= np.linalg.norm(perp, axis=1, keepdims=True)
    tilt = 10.0 ** rng.uniform(-7, -2, len(mu))
    nrm = perp + tilt[:, None] * ray
    sa.normal[:] = (nrm / np.linalg.norm(nrm, axis=1, keepdims=True)).astype(np.float32)
    s64 = sa.as_float64()
    cam = CameraModel(**sa.cameras[0])
    d_color = scenes.cotangent(cam.height, cam.width, seed=8)
    ref_out = O.render(s64, cam)
    ref_g = O.render_backward(s64, cam, ref_out, d_color)
    f = ref_out.frame
    assert (f.mode == 1).sum() > 0 and (np.abs(f.packed[:, 5]) > 1e3).sum() > 100
    for dtype in (torch.float32, torch.float64):
        got = run_gpu(sa, 0, "half", dtype, d_color)
        assert np.array_equal(got["pair_splat"], f.pair_splat)
        assert np.array_equal(got["mode"], f.mode)
        ref = {"color": ref_out.color, "alpha": ref_out.alpha, "depth": ref_out.depth,
               "transmittance": ref_out.transmittance,
               "terminal": ref_out.per_pixel_terminal_index}
        assert_images(got, ref)
        assert_grads(got, ref_g)


def test_wide_splat_row_merge_oracle(cuda):
    """Large splats (c5-like sigma 8-40 px): the frame's mean rows per primitive is
    >= 32, so K7a merges each splat's rows with 8 lanes and a shuffle tree
    (HS_K7A_WIDE_ROWS) instead of one lane in row order.  Integers bit-exact,
    images and gradients within the parity contract against the FP64 oracle."""
    O = _oracle()
    sa = scenes.frustum(800, 2, 320, 240, seed=31, sig_lo=8.0, sig_hi=40.0, clustered=True,
                        dup=0.1)
    s64 = sa.as_float64()
    cam = CameraModel(**sa.cameras[0])
    d_color = scenes.cotangent(cam.height, cam.width, seed=9)
    ref_out = O.render(s64, cam)
    ref_g = O.render_backward(s64, cam, ref_out, d_color)
    f = ref_out.frame
    assert len(f.pair_splat) >= 32 * len(sa.mu)  # the wide merge path is the one taken
    got = run_gpu(sa, 0, "half", torch.float32, d_color)
    assert np.array_equal(got["pair_splat"], f.pair_splat)
    assert np.array_equal(got["tile_starts"], f.tile_starts)
    ref = {"color": ref_out.color, "alpha": ref_out.alpha, "depth": ref_out.depth,
           "transmittance": ref_out.transmittance, "terminal": ref_out.per_pixel_terminal_index}
    assert_images(got, ref)
    assert_grads(got, ref_g)


@pytest.mark.parametrize("kernel,size", [("half", (128, 96)), ("full", (128, 96)),
                                         ("half", (528, 512))])
def test_split_backward_long_lists_oracle(cuda, kernel, size):
    """Small frames run K6 as (tile, segment) units, each below the top starting from
    K5's checkpoint (hs_blend.cu "K6 segments"; segments of 64 positions at 48 tiles,
    256 at 1056): balls whose tile lists run to thousands of splats, pixels alive
    through several segments, against the oracle's gradients; K5's images and the
    integers are unchanged."""
    O = _oracle()
    w, h = size
    sa = scenes.ball(30_000 if w == 128 else 60_000, 2, w, h, views=2, seed=31)
    s64 = sa.as_float64()
    cam = CameraModel(**sa.cameras[1])
    d_color = scenes.cotangent(cam.height, cam.width, seed=7)
    ref_out = O.render(s64, cam, kernel=kernel)
    ref_g = O.render_backward(s64, cam, ref_out, d_color)
    got = run_gpu(sa, 1, kernel, torch.float32, d_color)
    lens = np.diff(np.asarray(got["tile_starts"]))
    assert lens.max() > 4 * 256  # several segments per tile
    assert (got["terminal"] > 2 * 256).mean() > 0.05  # pixels alive past two checkpoints
    assert np.array_equal(got["tile_starts"], ref_out.frame.tile_starts)
    ref = {"color": ref_out.color, "alpha": ref_out.alpha, "depth": ref_out.depth,
           "transmittance": ref_out.transmittance, "terminal": ref_out.per_pixel_terminal_index}
    assert_images(got, ref)
    assert_grads(got, ref_g)
    assert np.array_equal(got["touch_count"], ref_g["touch_count"])
