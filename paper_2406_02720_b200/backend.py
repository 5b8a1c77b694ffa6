"""Blend-core selection seam, mirroring backend.py:1-48 of the reference.

This package ships exactly one blend core, the sm_100a kernels behind
``cuda_blend``; there is no CPU fallback and no multi-backend dispatch.  The
functions keep the reference's names so code that calls ``set_backend`` /
``get_backend`` keeps working: "auto" and "cuda" select the GPU core, anything
else raises.  ``HALFSPLAT_BACKEND`` is honoured the same way.
"""

import os

from . import cuda_blend

_forced = None


def available_backends():
    return ["cuda"]


def set_backend(name):
    """Force a backend for this process ('cuda', or None/'auto')."""
    global _forced
    if name not in (None, "auto", "cuda"):
        raise ValueError(f"unknown backend {name!r} (this package only has 'cuda')")
    _forced = None if name in (None, "auto") else name


def backend_name():
    choice = _forced or os.environ.get("HALFSPLAT_BACKEND", "auto")
    if choice not in ("auto", "cuda"):
        raise RuntimeError(f"HALFSPLAT_BACKEND={choice} is not available; only 'cuda'")
    return "cuda"


def get_backend():
    backend_name()
    return cuda_blend
