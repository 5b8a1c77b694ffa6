"""Image-quality metrics on the GPU (drop-in for metrics.py's psnr / ssim).

`psnr` takes the MSE from the same `hs_loss` pass that computes the training loss
(lambda 0: L1 and MSE only); `ssim` is loss.ssim.  float32 pairs are read as float32,
anything else as float64 (metrics.py:15-16).
"""

import math

import numpy as np

from .loss import _run, ssim  # noqa: F401  (shared implementation, re-exported)


def psnr(a, b):
    """10 log10(1 / MSE) over all channels; inf for identical images (metrics.py:13-22)."""
    stats, _ = _run(a, b, 0.0)
    mse = float(stats[3])
    if mse == 0.0:
        return math.inf
    return float(10.0 * np.log10(1.0 / mse))
