"""Blend-core plugin with the reference's signature, executed on the GPU.

Drop-in for ``halfsplat._blend_cy`` (_blend_cy.pyx:74-83, 190-199): the same
two functions over the same host arrays (layout contract _blend_py.py:1-19).
Each call binds the C-ABI entry points hs_forward_tiles / hs_backward_tiles of
libhalfsplat_b200.so, which upload the reference-packed splats, run the K5/K6
kernels over tiles [tile_lo, tile_hi) and write back only those tiles' pixels
and pair rows (pair rows accumulate, +=, as in the reference).

Dtype/contiguity mismatches raise ValueError, as the Cython memoryview
conversion does.
"""

import ctypes

import numpy as np

from . import _native


def _arr(a, dtype, ndim, name, writable=False):
    if not isinstance(a, np.ndarray) or a.dtype != dtype or a.ndim != ndim:
        raise ValueError(f"{name}: expected {ndim}-d {np.dtype(dtype)} array")
    if not a.flags.c_contiguous:
        raise ValueError(f"{name}: array is not C-contiguous")
    if writable and not a.flags.writeable:
        raise ValueError(f"{name}: array is read-only")
    return ctypes.c_void_p(a.ctypes.data)


def forward_tiles(packed, mode, pair_splat, tile_starts, height, width, tiles_x, background,
                  color, alpha, depth, transmittance, terminal, tile_lo, tile_hi):
    lib = _native.load()
    st = lib.hs_forward_tiles(
        _arr(packed, np.float64, 2, "packed"), _arr(mode, np.int8, 1, "mode"),
        _arr(pair_splat, np.int32, 1, "pair_splat"), _arr(tile_starts, np.int64, 1, "tile_starts"),
        packed.shape[0], pair_splat.shape[0], int(height), int(width), int(tiles_x),
        _arr(background, np.float64, 1, "background"),
        _arr(color, np.float64, 3, "color", True), _arr(alpha, np.float64, 2, "alpha", True),
        _arr(depth, np.float64, 2, "depth", True),
        _arr(transmittance, np.float64, 2, "transmittance", True),
        _arr(terminal, np.int32, 2, "terminal", True), int(tile_lo), int(tile_hi))
    _native.check(st, "hs_forward_tiles")


def backward_tiles(packed, mode, pair_splat, tile_starts, height, width, tiles_x, background,
                   d_color, transmittance, terminal, pair_grads, tile_lo, tile_hi):
    lib = _native.load()
    st = lib.hs_backward_tiles(
        _arr(packed, np.float64, 2, "packed"), _arr(mode, np.int8, 1, "mode"),
        _arr(pair_splat, np.int32, 1, "pair_splat"), _arr(tile_starts, np.int64, 1, "tile_starts"),
        packed.shape[0], pair_splat.shape[0], int(height), int(width), int(tiles_x),
        _arr(background, np.float64, 1, "background"), _arr(d_color, np.float64, 3, "d_color"),
        _arr(transmittance, np.float64, 2, "transmittance"), _arr(terminal, np.int32, 2, "terminal"),
        _arr(pair_grads, np.float64, 2, "pair_grads", True), int(tile_lo), int(tile_hi))
    _native.check(st, "hs_backward_tiles")
