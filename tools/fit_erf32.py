"""Fit the FP32 erf used by the blend kernels (csrc/hs_common.cuh:erf32).

erf(x) = 1 - 2**Q(x) for x >= 0 with Q(x) = x * R(x), R of degree 5, fitted
to log2(erfc(x)) on [0, 3.92] by iteratively reweighted least squares
(Lawson) with weight erfc(x)*ln2 (i.e. minimising the absolute error of erf).
Prints the coefficients (lowest order first) and the max abs error of an
FP32 Horner evaluation against scipy's erf.  Build-time tool only.
"""
import math

import numpy as np
from scipy.special import erf, erfc

X_MAX = 3.92


def fit(deg, lo=0.0, hi=X_MAX, iters=60):
    xs = (np.cos(np.linspace(0, np.pi, 4000)) * 0.5 + 0.5) * (hi - lo) + lo
    f = np.log2(erfc(xs))
    w = erfc(xs) * math.log(2)
    v = np.stack([xs ** (k + 1) for k in range(deg)], 1)
    wt = np.ones_like(xs)
    for _ in range(iters):
        c, *_ = np.linalg.lstsq(v * (w * wt)[:, None], f * w * wt, rcond=None)
        err = np.abs((v @ c - f) * w)
        wt = wt * (err / err.max()) ** 0.5 + 1e-12
        wt /= wt.max()
    return c


def eval_f32(c, x):
    x = np.minimum(np.abs(x).astype(np.float32), np.float32(X_MAX))
    acc = np.full_like(x, np.float32(c[-1]))
    for k in range(len(c) - 2, -1, -1):
        acc = (acc.astype(np.float64) * x + np.float32(c[k])).astype(np.float32)
    q = (acc.astype(np.float64) * x).astype(np.float32)
    return (np.float32(1) - np.exp2(q.astype(np.float64)).astype(np.float32))


if __name__ == "__main__":
    coeffs = fit(6).astype(np.float32)
    xs = np.linspace(0, 6, 200001)
    err = np.abs(eval_f32(coeffs, xs).astype(np.float64) - erf(xs)).max()
    for v in coeffs:
        print("%.9ef" % v)
    print("max abs error", err)
