"""The FP32 erf of the blend kernels (csrc/hs_common.cuh:erf32), emulated
bit-faithfully in numpy float32 (fmaf = one rounding): accuracy against the
reference's fast_erf (golden) and exact oddness."""

import os
import re

import numpy as np
import pytest

from conftest import REPO, load_golden

HEADER = os.path.join(REPO, "paper_2406_02720_b200", "csrc", "hs_common.cuh")


def coefficients():
    body = open(HEADER).read().split("float erf32(float z)")[1].split("}")[0]
    first = float(re.search(r"float r = ([-+0-9.e]+)f;", body).group(1))
    rest = [float(x) for x in re.findall(r"fmaf\(r, a, ([-+0-9.e]+)f\)", body)]
    return [first] + rest  # highest order first


def fmaf(a, b, c):
    return (a.astype(np.float64) * b + c).astype(np.float32)


def erf32(z):
    z = np.asarray(z, dtype=np.float32)
    a = np.minimum(np.abs(z), np.float32(3.92))
    cs = coefficients()
    r = np.full_like(a, np.float32(cs[0]))
    for c in cs[1:]:
        r = fmaf(r, a, np.float32(c))
    r = (r * a).astype(np.float32)
    e = (np.float32(1.0) - np.exp2(r.astype(np.float64)).astype(np.float32)).astype(np.float32)
    return np.copysign(e, z)


def test_coefficients_parse():
    assert len(coefficients()) == 6


def test_erf32_accuracy_vs_reference_erf():
    gold = load_golden("erf")
    z = gold["z"].astype(np.float32)
    got = erf32(z).astype(np.float64)
    # reference polynomial is within 5e-9 of erf; the FP32 one within ~3.3e-7
    assert np.abs(got - gold["erf"]).max() < 4e-7


def test_erf32_is_exactly_odd():
    z = np.linspace(-5, 5, 20001, dtype=np.float32)
    assert np.array_equal(erf32(-z), -erf32(z))
    assert erf32(np.float32(0.0)) == 0.0


@pytest.mark.gpu
def test_device_erf32_on_mufu(cuda):
    """The device erf itself (MUFU.EX2, not an exact exp2): within 4e-7 of the
    reference's fast_erf on its golden points, and bitwise odd."""
    import torch
    from paper_2406_02720_b200 import _native
    lib = _native.load()
    gold = load_golden("erf")
    z = np.concatenate([gold["z"].astype(np.float32),
                        np.linspace(-6, 6, 200001, dtype=np.float32)])
    zt = torch.as_tensor(z, device="cuda")
    outs = []
    for arg in (zt, -zt):
        o = torch.empty_like(arg)
        _native.check(lib.hs_probe_erf32(arg.data_ptr(), o.data_ptr(), arg.numel(), None),
                      "probe_erf32")
        outs.append(o.cpu().numpy())
    pos, neg = outs
    ng = gold["z"].shape[0]
    assert np.abs(pos[:ng].astype(np.float64) - gold["erf"]).max() < 4e-7
    assert np.array_equal(neg, -pos)
    # the emulation above agrees with the hardware to a few ulps of 1.0f
    assert np.abs(pos - erf32(z)).max() <= 2.0 ** -21
