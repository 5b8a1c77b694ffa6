"""The C-ABI library loads and exports exactly what include/halfsplat_b200.h
declares; host-only entry points behave (no GPU needed)."""

import ctypes
import os
import re
import subprocess

import pytest

from conftest import REPO
from paper_2406_02720_b200 import _native, errors

HEADER = os.path.join(REPO, "include", "halfsplat_b200.h")


def header_functions():
    text = open(HEADER).read()
    text = re.sub(r"/\*.*?\*/", "", text, flags=re.S)
    return sorted(set(re.findall(r"\b(hs_[a-z0-9_]+)\s*\(", text)))


def test_header_declares_the_bound_functions():
    assert header_functions() == sorted(_native.EXPORTED_SYMBOLS)


def test_library_exports_every_header_symbol(native_lib):
    out = subprocess.run(["nm", "-D", "--defined-only", _native.library_path()],
                         capture_output=True, text=True, check=True).stdout
    exported = set(re.findall(r"\bT (hs_[a-z0-9_]+)", out))
    missing = set(header_functions()) - exported
    assert not missing, missing
    for name in header_functions():
        assert hasattr(native_lib, name)


def test_library_is_sm100a(native_lib):
    res = subprocess.run(["cuobjdump", "--list-elf", _native.library_path()], capture_output=True,
                         text=True)
    assert "sm_100a" in res.stdout


def _kernel_sass(native_lib, symbol_re, _dump={}):
    """SASS of the library's functions whose mangled names match symbol_re."""
    if "text" not in _dump:
        _dump["text"] = subprocess.run(["cuobjdump", "-sass", _native.library_path()],
                                       capture_output=True, text=True, check=True).stdout
    out, keep = [], False
    for line in _dump["text"].splitlines():
        m = re.match(r"\s+Function : (\S+)", line)
        if m:
            keep = re.search(symbol_re, m.group(1)) is not None
        elif keep:
            out.append(line)
    return "\n".join(out)


def test_sass_uses_sm100_features(native_lib):
    """The hot kernels use what DESIGN.md says they use: packed FP32 pipe
    instructions in the blends, bulk copies on an mbarrier in K1/K7's scene staging."""
    blends = _kernel_sass(native_lib, r"blend_(fwd|bwd)_kernel")
    assert "FFMA2" in blends and "FMUL2" in blends
    geom = _kernel_sass(native_lib, r"preprocess_(fwd|bwd)_kernelIfLi3E")
    assert "UBLKCP" in geom and "SYNCS.PHASECHK" in geom


def test_frame_init_error_codes(native_lib):
    f = _native.HsFrame()
    assert native_lib.hs_frame_init(ctypes.byref(f), 0, 64, 64, 0) == _native.HS_ERR_EMPTY_SCENE
    assert native_lib.hs_frame_init(ctypes.byref(f), 10, 65536, 65537, 0) == \
        _native.HS_ERR_IMAGE_TOO_LARGE
    assert native_lib.hs_frame_init(ctypes.byref(f), 10, 64, 64, 7) == \
        _native.HS_ERR_INVALID_KERNEL
    assert native_lib.hs_frame_init(ctypes.byref(f), 10, 1920, 1080, 0) == _native.HS_OK
    assert (f.tiles_x, f.tiles_y, f.n_tiles) == (120, 68, 8160)
    assert f.tile_bits == 13
    assert f.num_pairs == -1


def test_status_mapping(native_lib):
    with pytest.raises(errors.EmptyScene):
        _native.check(_native.HS_ERR_EMPTY_SCENE)
    with pytest.raises(errors.ImageTooLarge):
        _native.check(_native.HS_ERR_IMAGE_TOO_LARGE)
    with pytest.raises(errors.MismatchedForward):
        _native.check(_native.HS_ERR_MISMATCHED_FORWARD)
    with pytest.raises(ValueError):
        _native.check(_native.HS_ERR_INVALID_KERNEL)
    assert native_lib.hs_abi_version() == 2
    assert b"EmptyScene" in native_lib.hs_status_string(_native.HS_ERR_EMPTY_SCENE)


def test_stage_calls_refuse_missing_workspace(native_lib):
    f = _native.HsFrame()
    assert native_lib.hs_frame_init(ctypes.byref(f), 10, 64, 64, 0) == _native.HS_OK
    st = native_lib.hs_bin_and_sort(ctypes.byref(f), None)
    assert st == _native.HS_ERR_WORKSPACE


def test_struct_layouts_match_header():
    # field order/size of the ctypes mirrors (the C compiler's layout for x86-64)
    assert ctypes.sizeof(_native.HsCamera) == 16 * 8 + 5 * 8 + 3 * 8 + 2 * 4
    assert ctypes.sizeof(_native.HsScene) == 8 + 4 + 4 + 7 * 8 + 3 * 8
    assert ctypes.sizeof(_native.HsGrads) == 9 * 8 + 8  # + int32 accumulate, padded
    assert _native.HsFrame.num_pairs.offset == 40
