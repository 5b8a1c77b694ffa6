"""GPU loss (csrc/hs_loss.cu) against the reference's compute_loss /
ssim_with_grad (tests/golden/loss.npz, loss.py:48-106) and the oracle.

Tolerances (FP64 arithmetic in the reference's order, FP32 image inputs that
the fixtures already hold exactly): loss and mean SSIM within 1e-12 relative
(only the reduction order differs); float64 gradients within 1e-12 of the
largest gradient entry or of 1/n, whichever is larger (FMA contraction and the
reciprocal forms differ from numpy by a few ulp);
the float32 cotangent within float32 rounding (1e-6 relative to the largest
entry).  Errors mirror the reference: ShapeMismatch, ImageTooSmall, ValueError."""

import numpy as np
import pytest

from conftest import load_golden

pytestmark = pytest.mark.gpu


def _grad_close(got, ref, rel):
    # scale: the largest entry, but at least the natural gradient unit 1/n (for
    # identical images the reference's SSIM gradient is pure rounding noise)
    scale = max(np.abs(ref).max(), 1.0 / ref.size)
    return np.abs(got - ref).max() <= rel * scale


def test_loss_matches_reference_golden(cuda):
    from paper_2406_02720_b200 import loss as L
    gold = load_golden("loss")
    for c in gold["cases"]:
        a, b, lam = gold[f"{c}_a"], gold[f"{c}_b"], float(gold[f"{c}_lambda"])
        val, grad = L.compute_loss(a, b, lam)
        ref = gold[f"{c}_grad"]
        assert grad.shape == ref.shape and grad.dtype == np.float64, c
        assert val == pytest.approx(float(gold[f"{c}_loss"]), rel=1e-12, abs=1e-15), c
        assert _grad_close(grad, ref, 1e-12), c
        if lam > 0:
            s, sg = L.ssim_with_grad(a, b)
            assert s == pytest.approx(float(gold[f"{c}_ssim"]), rel=1e-12), c
            assert sg.shape == gold[f"{c}_ssim_grad"].shape, c
            assert _grad_close(sg, gold[f"{c}_ssim_grad"], 1e-12), c
    same = gold["same_l02_a"]
    assert L.ssim(same, same) == pytest.approx(1.0, abs=1e-15)


def test_device_loss_cotangent_1080p_vs_oracle(cuda):
    """Full-size (1920x1080x3) image pair as the training step sees it: the
    float32 cotangent and the device loss against the oracle."""
    import torch
    from oracle import oracle as O
    from paper_2406_02720_b200 import loss as L
    rng = np.random.default_rng(5)
    h, w = 1080, 1920
    # smooth-ish target plus a perturbed render, float32-exact
    base = rng.random((h // 8, w // 8, 3)).astype(np.float32)
    tgt = np.repeat(np.repeat(base, 8, axis=0), 8, axis=1)
    ren = np.clip(tgt + rng.normal(0, 0.05, tgt.shape), 0, 1).astype(np.float32)
    ref_loss, ref_grad = O.compute_loss(ren, tgt, 0.2)
    dl = L.DeviceLoss(0.2)
    x = torch.from_numpy(ren).to(cuda)
    y = torch.from_numpy(tgt).to(cuda)
    stats, d = dl(x, y)
    torch.cuda.synchronize()
    assert d.dtype == torch.float32 and tuple(d.shape) == (h, w, 3)
    assert float(stats[0]) == pytest.approx(ref_loss, rel=1e-12)
    assert _grad_close(d.cpu().numpy().astype(np.float64), ref_grad, 1e-6)
    # repeated calls reuse the workspace and are deterministic
    stats2, d2 = dl(x, y)
    assert torch.equal(stats, stats2) and torch.equal(d, d2)


def test_loss_errors_mirror_reference(cuda):
    from paper_2406_02720_b200 import errors
    from paper_2406_02720_b200 import loss as L
    a = np.zeros((16, 16, 3), np.float32)
    with pytest.raises(errors.ShapeMismatch):
        L.compute_loss(a, np.zeros((16, 17, 3), np.float32))
    with pytest.raises(errors.ShapeMismatch):
        L.compute_loss(np.zeros(5), np.zeros(5))
    with pytest.raises(ValueError):
        L.compute_loss(a, a, lambda_ssim=1.5)
    with pytest.raises(errors.ImageTooSmall):
        L.compute_loss(np.zeros((10, 30, 3)), np.zeros((10, 30, 3)), 0.2)
    # lambda 0 skips SSIM and accepts small images (loss.py:97-99)
    val, g = L.compute_loss(np.ones((4, 5)), np.zeros((4, 5)), 0.0)
    assert val == 1.0 and g.shape == (4, 5) and np.all(g == 1.0 / 20)


def test_loss_many_channels_vs_oracle(cuda):
    """C = 6 and 9: a full 4-channel group plus a tail group (separate launches)."""
    from oracle import oracle as O
    from paper_2406_02720_b200 import loss as L
    rng = np.random.default_rng(11)
    for c in (6, 9):
        a = rng.random((29, 45, c)).astype(np.float32)
        b = rng.random((29, 45, c)).astype(np.float32)
        ref_loss, ref_grad = O.compute_loss(a, b, 0.3)
        val, grad = L.compute_loss(a, b, 0.3)
        assert val == pytest.approx(ref_loss, rel=1e-12)
        assert _grad_close(grad, ref_grad, 1e-12)


@pytest.mark.parametrize("seed", range(16))
def test_loss_random_shapes_vs_oracle(cuda, seed):
    """Random sizes (ragged against the 32x16 tiles), channel counts, lambdas and
    exact ties against the C oracle (itself bit-identical to the reference)."""
    from oracle import oracle as O
    from paper_2406_02720_b200 import loss as L
    rng = np.random.default_rng(seed)
    h, w = int(rng.integers(11, 90)), int(rng.integers(11, 120))
    c = int(rng.choice([1, 2, 3, 4, 5]))
    lam = float(rng.choice([0.0, 1.0, rng.uniform(0, 1)]))
    a = rng.random((h, w, c)).astype(np.float32)
    b = np.clip(a + rng.normal(0, 0.2, a.shape), 0, 1).astype(np.float32)
    ties = rng.random(a.shape) < 0.1
    b[ties] = a[ties]
    if c == 1 and rng.random() < 0.5:
        a, b = a[..., 0], b[..., 0]
    ref_loss, ref_grad = O.compute_loss(a, b, lam)
    val, grad = L.compute_loss(a, b, lam)
    assert grad.shape == ref_grad.shape
    assert val == pytest.approx(ref_loss, rel=1e-12, abs=1e-15)
    assert _grad_close(grad, ref_grad, 1e-12)


def test_loss_float64_inputs_match_reference(cuda):
    """Float64 renders and uint8 targets are read unrounded (hs_loss_f64): a uint8/255
    target, differences below float32 resolution (sign(diff) stays +-1, so the L1
    cotangent keeps its 1/n per pixel) and a 2-D pair, against the reference's own
    compute_loss / ssim_with_grad / psnr (tests/golden/loss64.npz)."""
    from paper_2406_02720_b200 import loss as L
    from paper_2406_02720_b200 import metrics as M
    gold = load_golden("loss64")
    for c in gold["cases"]:
        a, b, lam = gold[f"{c}_a"], gold[f"{c}_b"], float(gold[f"{c}_lambda"])
        val, grad = L.compute_loss(a, b, lam)
        ref = gold[f"{c}_grad"]
        assert grad.shape == ref.shape and grad.dtype == np.float64, c
        assert val == pytest.approx(float(gold[f"{c}_loss"]), rel=1e-12, abs=1e-15), c
        assert _grad_close(grad, ref, 1e-12), c
        # the L1 part's sign pattern is exact (no float32 ties)
        assert np.array_equal(np.sign(grad) != 0, np.sign(ref) != 0) or lam > 0, c
        assert M.psnr(a, b) == pytest.approx(float(gold[f"{c}_psnr"]), rel=1e-12), c
        if lam > 0:
            s, sg = L.ssim_with_grad(a, b)
            assert s == pytest.approx(float(gold[f"{c}_ssim"]), rel=1e-12), c
            assert _grad_close(sg, gold[f"{c}_ssim_grad"], 1e-12), c


def test_device_loss_float64_tensors(cuda):
    """DeviceLoss on float64 CUDA tensors takes the float64 kernel too."""
    import torch
    from paper_2406_02720_b200 import loss as L
    gold = load_golden("loss64")
    a, b = gold["tiny_diff_l02_a"], gold["tiny_diff_l02_b"]
    stats, d = L.DeviceLoss(0.2)(torch.from_numpy(a).to(cuda), torch.from_numpy(b).to(cuda),
                                 d_out_f64=torch.empty(a.shape, dtype=torch.float64, device=cuda))
    assert float(stats[0]) == pytest.approx(float(gold["tiny_diff_l02_loss"]), rel=1e-12)
    assert _grad_close(d.cpu().numpy(), gold["tiny_diff_l02_grad"], 1e-12)
