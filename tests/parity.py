"""Parity contract between the FP32 GPU blend and the FP64 reference/oracle.

Stated once here and used by every GPU parity test:

  integers   valid, tile_rect, mode, pair_splat, tile_starts, radii: bit-exact
  packed     each column equals the FP64 value rounded to FP32 (rtol 2e-6; the
             FP64 preprocess differs from numpy only by libm `exp` ulps)
  images     max |delta| <= 1e-4 over pixels whose `terminal` matches, and the
             terminal-mismatch fraction <= 1e-3 of pixels; the all-pixel max is
             reported (a terminal flip moves a pixel by up to ~w*T/(1-w))
  gradients  per parameter group ||g - g_ref|| / ||g_ref|| <= 1e-3 (norm-wise;
             elementwise relative error is meaningless under cancellation)
"""

import numpy as np

PIXEL_ATOL = 1e-4
TERMINAL_MISMATCH_FRAC = 1e-3
GRAD_REL = 1e-3
PACKED_RTOL = 2e-6

GRAD_GROUPS = ("d_mu", "d_log_scale", "d_rotation", "d_sh", "d_normal", "d_raw_opacity_a",
               "d_raw_opacity_b", "pos_grad_norm")


def image_report(got, ref):
    """got/ref: dicts with color (H,W,3), alpha, depth, transmittance, terminal."""
    t_got = np.asarray(got["terminal"]).reshape(-1)
    t_ref = np.asarray(ref["terminal"]).reshape(-1)
    match = t_got == t_ref
    rep = {"terminal_mismatch_frac": float(1.0 - match.mean()), "pixels": int(match.size)}
    for k in ("color", "alpha", "depth", "transmittance"):
        g = np.asarray(got[k], dtype=np.float64).reshape(match.size, -1)
        r = np.asarray(ref[k], dtype=np.float64).reshape(match.size, -1)
        d = np.abs(g - r).max(axis=1)
        rep[f"{k}_max_matched"] = float(d[match].max()) if match.any() else 0.0
        rep[f"{k}_max_all"] = float(d.max())
    return rep


def assert_images(got, ref, depth_atol=None):
    rep = image_report(got, ref)
    assert rep["terminal_mismatch_frac"] <= TERMINAL_MISMATCH_FRAC, rep
    for k in ("color", "alpha", "transmittance"):
        assert rep[f"{k}_max_matched"] <= PIXEL_ATOL, (k, rep)
    # depth is an un-normalised sum of w*T*z (z ~ 2..6): same relative budget
    tol = depth_atol if depth_atol is not None else PIXEL_ATOL * 10
    assert rep["depth_max_matched"] <= tol, rep
    return rep


def grad_report(got, ref, groups=GRAD_GROUPS):
    rep = {}
    for k in groups:
        g = np.asarray(got[k], dtype=np.float64)
        r = np.asarray(ref[k], dtype=np.float64)
        den = np.linalg.norm(r)
        rep[k] = float(np.linalg.norm(g - r) / den) if den > 0 else float(np.linalg.norm(g))
    return rep


def assert_grads(got, ref, groups=GRAD_GROUPS, tol=GRAD_REL):
    rep = grad_report(got, ref, groups)
    for k, v in rep.items():
        assert v <= tol, (k, rep)
    return rep
