"""Device optimizer step (csrc/hs_adam.cu, trainer.py mirror) against the
reference's trainer.step (tests/golden/adam.npz) and the oracle.

Contract: a float64 scene steps BIT-IDENTICALLY to the reference (same
statement order, -fmad=false, IEEE division and sqrt), for every mode, the
'full' opacity tie, frozen groups and zero-gradient rows; a float32 scene
within float32 rounding of the float64 result (atol 2e-6, rtol 1e-6)."""

import numpy as np
import pytest
import torch

import adam_cases as A
from conftest import load_golden

pytestmark = pytest.mark.gpu


def _device_scene(params, deg, dtype):
    from paper_2406_02720_b200.geometry import Scene
    return Scene(*(params[f] for f in A.FIELDS), sh_degree=deg, device="cuda", dtype=dtype)


def _device_grads(scene, grads):
    from paper_2406_02720_b200.device import DeviceGradientSet
    g = DeviceGradientSet.empty_like_scene(scene)
    for name in A.GRADS:
        getattr(g, name).copy_(torch.as_tensor(grads[name]))
    g.pos_grad_norm.zero_()
    g.touch_count.zero_()
    return g


@pytest.mark.parametrize("dtype", [torch.float64, torch.float32])
def test_adam_step_matches_reference(cuda, dtype):
    from paper_2406_02720_b200 import trainer as T
    gold = load_golden("adam")
    for name in gold["cases"]:
        deg, kw, params, steps, t_ref = A.case(gold, name)
        cfg = A.config(kw)
        scene = _device_scene(params, deg, dtype)
        state = T.AdamState(scene)
        for it, (iteration, grads, after) in enumerate(steps):
            T.adam_step(scene, _device_grads(scene, grads), cfg, state, iteration,
                        A.SPATIAL_SCALE)
            torch.cuda.synchronize()
            for f in A.FIELDS:
                got = getattr(scene, f).cpu().numpy().astype(np.float64)
                if dtype == torch.float64:
                    assert np.array_equal(got, after[f]), (name, it, f)
                else:
                    np.testing.assert_allclose(got, after[f], rtol=1e-6, atol=2e-6,
                                               err_msg=f"{name} step {it} {f}")
        assert [state.t[g] for g in T.GROUPS] == list(t_ref), name


def test_train_step_end_to_end(cuda):
    """render -> hs_loss -> backward -> hs_adam_step on a small float64 scene:
    the loss equals the oracle's compute_loss of the GPU image, the Adam update
    equals OracleAdam applied to the GPU's own gradients (bit-exact), and 30
    steps towards a target reduce the loss."""
    from oracle import oracle as O
    from paper_2406_02720_b200 import device, scenes
    from paper_2406_02720_b200 import trainer as T
    from paper_2406_02720_b200.geometry import CameraModel, Scene
    sa = scenes.frustum(1500, 2, 96, 64, seed=4)
    cam = CameraModel(**sa.cameras[0])
    scene = Scene(*(getattr(sa, f) for f in sa.FIELDS), sh_degree=sa.sh_degree,
                  background_color=sa.background_color, device="cuda", dtype=torch.float64)
    # target: the same scene with shifted colours
    tsc = Scene(*(getattr(sa, f) for f in sa.FIELDS), sh_degree=sa.sh_degree,
                background_color=sa.background_color, device="cuda", dtype=torch.float64)
    tsc.sh_coeffs[:, 0, :] += 0.3
    target = device.render(tsc, cam).color.clone()
    cfg = T.TrainConfig(total_iters=100, densify_until=50)
    state = T.AdamState(scene)
    trainer = T.StepRunner(scene, cfg)
    before = {f: getattr(scene, f).cpu().numpy().copy() for f in A.FIELDS}
    loss0, grads, out = trainer.step(scene, (cam, target), state, iteration=0)
    ref_loss, _ = O.compute_loss(out.color.cpu().numpy(), target.cpu().numpy(), 0.2)
    assert loss0 == pytest.approx(ref_loss, rel=1e-12)
    opt = O.OracleAdam(before)
    g = {name: getattr(grads, name).cpu().numpy() for name in A.GRADS}
    lrs = T.learning_rates(cfg, 0, 1.0)
    opt.step(before, g, lrs, False)
    for f in A.FIELDS:
        assert np.array_equal(getattr(scene, f).cpu().numpy(), before[f]), f
    losses = [loss0]
    for it in range(1, 30):
        loss, _, _ = trainer.step(scene, (cam, target), state, iteration=it)
        losses.append(loss)
    assert losses[-1] < 0.8 * losses[0], losses


def test_trainer_run_matches_reference(cuda, tmp_path):
    """Trainer.run (trainer.py:365-449) against the reference's own 40-iteration run
    (tests/golden/train.npz): same view order and split draws from the seeded
    Generator, so the density-control events and primitive counts must match
    exactly; loss / PSNR follow within 2e-3 relative (the GPU blends in FP32,
    the reference in FP64) and the mean opacity disparity within 1e-4."""
    import csv
    from paper_2406_02720_b200 import trainer as T
    from paper_2406_02720_b200.geometry import CameraModel, Scene
    gold = load_golden("train")
    deg = int(gold["deg"])
    f = A.split(gold["scene"], A.FIELDS, deg)
    scene = Scene(*(f[k] for k in A.FIELDS), sh_degree=deg, background_color=gold["background"],
                  device="cuda", dtype=torch.float64)
    fx, fy, cx, cy, w, h = gold["cam"]
    views = [(f"v{v}", CameraModel(world_to_cam=gold[f"w2c{v}"], fx=fx, fy=fy, cx=cx, cy=cy,
                                   width=int(w), height=int(h)), gold[f"target{v}"])
             for v in range(3)]
    cfg = T.TrainConfig(total_iters=40, densify_until=35, densify_interval=10,
                        opacity_reset_start=30, opacity_reset_interval=30,
                        opacity_reset_until=35, densify_grad_threshold=2e-5, seed=3,
                        prune_extent_factor=5.0, percent_dense=0.02)
    tr = T.Trainer(scene, views, cfg, metrics_path=str(tmp_path / "m.csv"))
    tr.run()
    fields = [str(x) for x in gold["fields"]]
    ref = gold["rows"]
    got = np.array([[float(r[k]) for k in fields] for r in tr.metrics_rows])
    exact = [fields.index(k) for k in ("iteration", "num_primitives", "cloned", "split",
                                       "pruned", "opacity_reset")]
    assert np.array_equal(got[:, exact], ref[:, exact])
    for k in ("loss", "psnr"):
        c = fields.index(k)
        np.testing.assert_allclose(got[:, c], ref[:, c], rtol=2e-3, atol=1e-6, err_msg=k)
    # Adam's first steps are lr * sign(g): a near-zero opacity gradient whose FP32 sign
    # differs moves one primitive by 2 lr, i.e. the mean disparity by ~1e-4 / N
    c = fields.index("opacity_disparity")
    np.testing.assert_allclose(got[:, c], ref[:, c], rtol=0, atol=1e-4, err_msg="disparity")
    with open(tmp_path / "m.csv") as fh:
        assert [r["num_primitives"] for r in csv.DictReader(fh)] == \
            [str(int(x)) for x in ref[:, fields.index("num_primitives")]]


def test_metrics_psnr_and_disparity(cuda):
    from oracle import oracle as O
    from paper_2406_02720_b200 import metrics
    from paper_2406_02720_b200 import trainer as T
    from paper_2406_02720_b200.geometry import Scene
    rng = np.random.default_rng(2)
    a = rng.random((40, 50, 3)).astype(np.float32)
    b = a + np.float32(0.1)
    assert metrics.psnr(a, a) == np.inf
    assert metrics.psnr(a, b) == pytest.approx(20.0, rel=1e-6)
    mse = np.mean((a.astype(np.float64) - b) ** 2)
    assert metrics.psnr(a, b) == pytest.approx(10 * np.log10(1 / mse), rel=1e-12)
    n = 3000
    sc = Scene(rng.normal(size=(n, 3)), rng.normal(size=(n, 3)), rng.normal(size=(n, 4)),
               rng.normal(size=(n, 1, 3)), rng.normal(size=(n, 3)), rng.normal(0, 3, n),
               rng.normal(0, 3, n), sh_degree=0, device="cuda", dtype=torch.float64)
    p = sc.numpy()
    ref = np.abs(O._sigmoid(p["raw_opacity_a"]) - O._sigmoid(p["raw_opacity_b"])).mean()
    assert T.opacity_disparity(sc) == pytest.approx(ref, rel=1e-12)
