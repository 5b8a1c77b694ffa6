"""ctypes binding of libhalfsplat_b200.so (include/halfsplat_b200.h).

The shared library is the product: there is no Python or CPU implementation of
any kernel behind these calls.  Loading fails loudly if the library has not been
built (``python -m paper_2406_02720_b200.build``).
"""

import ctypes
import os

from . import errors

_LIB_PATH = os.path.join(os.path.dirname(os.path.abspath(__file__)), "lib", "libhalfsplat_b200.so")

HS_OK = 0
HS_ERR_EMPTY_SCENE = 1
HS_ERR_IMAGE_TOO_LARGE = 2
HS_ERR_INVALID_KERNEL = 3
HS_ERR_MISMATCHED_FORWARD = 4
HS_ERR_INVALID_ARG = 5
HS_ERR_CUDA = 6
HS_ERR_WORKSPACE = 7
HS_ERR_IMAGE_TOO_SMALL = 8
HS_ERR_INVALID_LAMBDA = 9

HS_DTYPE_F32 = 0
HS_DTYPE_F64 = 1
HS_COMM_ID_BYTES = 128
HS_FRAME_PAIR_OVERFLOW = 1
HS_FRAME_DEPTH_FALLBACK = 2
HS_KERNEL_HALF = 0
HS_KERNEL_FULL = 1

c_void_p = ctypes.c_void_p
c_int32 = ctypes.c_int32
c_int64 = ctypes.c_int64
c_size_t = ctypes.c_size_t
c_double_p = ctypes.POINTER(ctypes.c_double)


class HsCamera(ctypes.Structure):
    _fields_ = [
        ("world_to_cam", ctypes.c_double * 16),
        ("fx", ctypes.c_double), ("fy", ctypes.c_double),
        ("cx", ctypes.c_double), ("cy", ctypes.c_double),
        ("near_clip", ctypes.c_double),
        ("center", ctypes.c_double * 3),
        ("width", c_int32), ("height", c_int32),
    ]


class HsScene(ctypes.Structure):
    _fields_ = [
        ("n", c_int64), ("sh_degree", c_int32), ("dtype", c_int32),
        ("mu", c_void_p), ("log_scale", c_void_p), ("rotation", c_void_p),
        ("sh_coeffs", c_void_p), ("normal", c_void_p),
        ("raw_opacity_a", c_void_p), ("raw_opacity_b", c_void_p),
        ("background", ctypes.c_double * 3),
    ]


class HsFrame(ctypes.Structure):
    _fields_ = [
        ("n", c_int64), ("width", c_int32), ("height", c_int32),
        ("tiles_x", c_int32), ("tiles_y", c_int32), ("n_tiles", c_int32),
        ("kernel", c_int32), ("tile_bits", c_int32), ("sort_selector", c_int32),
        ("num_pairs", c_int64),
        ("frame_ws", c_void_p), ("frame_ws_bytes", c_size_t),
        ("bin_ws", c_void_p), ("bin_ws_bytes", c_size_t),
        ("pair_capacity", c_int64), ("depth_sort_full", c_int32),
    ]


class HsGrads(ctypes.Structure):
    _fields_ = [
        ("d_mu", c_void_p), ("d_log_scale", c_void_p), ("d_rotation", c_void_p),
        ("d_sh", c_void_p), ("d_normal", c_void_p),
        ("d_raw_opacity_a", c_void_p), ("d_raw_opacity_b", c_void_p),
        ("pos_grad_norm", c_void_p), ("touch_count", c_void_p), ("accumulate", c_int32),
    ]


class HsAdamState(ctypes.Structure):
    _fields_ = [("m", c_void_p * 7), ("v", c_void_p * 7), ("t", c_int64 * 8)]


class HsDensifyStats(ctypes.Structure):
    _fields_ = [("grad_sum", c_void_p), ("mu_grad_sum", c_void_p), ("count", c_void_p)]


class HsDensifyConfig(ctypes.Structure):
    _fields_ = [("densify_grad_threshold", ctypes.c_double),
                ("prune_opacity_threshold", ctypes.c_double),
                ("percent_dense", ctypes.c_double), ("prune_extent_factor", ctypes.c_double),
                ("scene_extent", ctypes.c_double), ("log_split_scale", ctypes.c_double),
                ("max_primitives", c_int64)]


class HsDensifyPlan(ctypes.Structure):
    _fields_ = [("n_in", c_int64), ("n_out", c_int64), ("kept", c_int64), ("cloned", c_int64),
                ("split", c_int64), ("pruned", c_int64)]


class HsPlyLayout(ctypes.Structure):
    _fields_ = [("n", c_int64), ("stride", c_int32), ("n_props", c_int32),
                ("sh_degree", c_int32), ("offset", ctypes.c_int16 * 128),
                ("type", ctypes.c_int8 * 128), ("column", ctypes.c_int16 * 66)]


# name -> (restype, argtypes); every symbol declared in include/halfsplat_b200.h
_SIGNATURES = {
    "hs_frame_init": (c_int32, [ctypes.POINTER(HsFrame), c_int64, c_int32, c_int32, c_int32]),
    "hs_frame_workspace_size": (c_size_t, [c_int64, c_int32, c_int32]),
    "hs_binning_workspace_size": (c_size_t, [c_int64, c_int64, c_int32, c_int32]),
    "hs_preprocess_fwd": (c_int32, [ctypes.POINTER(HsFrame), ctypes.POINTER(HsScene),
                                    ctypes.POINTER(HsCamera), c_void_p, c_void_p]),
    "hs_preprocess_fwd_views": (c_int32, [c_void_p, c_int32, ctypes.POINTER(HsScene),
                                          ctypes.POINTER(HsCamera), c_void_p, c_int32,
                                          c_void_p]),
    "hs_frame_rank": (c_int32, [ctypes.POINTER(HsFrame), c_void_p]),
    "hs_frame_read_num_pairs": (c_int32, [ctypes.POINTER(HsFrame), c_void_p]),
    "hs_read_pairs_and_bin": (c_int32, [ctypes.POINTER(HsFrame), c_void_p]),
    "hs_bin_and_sort": (c_int32, [ctypes.POINTER(HsFrame), c_void_p]),
    "hs_blend_fwd": (c_int32, [ctypes.POINTER(HsFrame), c_double_p, c_void_p, c_void_p,
                               c_void_p, c_void_p, c_void_p, c_void_p]),
    "hs_blend_bwd": (c_int32, [ctypes.POINTER(HsFrame), c_double_p, c_void_p, c_void_p,
                               c_void_p, c_void_p]),
    "hs_blend_window_stats": (c_int32, [ctypes.POINTER(HsFrame), c_void_p, c_void_p]),
    "hs_preprocess_bwd": (c_int32, [ctypes.POINTER(HsFrame), ctypes.POINTER(HsScene),
                                    ctypes.POINTER(HsCamera), ctypes.POINTER(HsGrads), c_void_p]),
    "hs_preprocess_bwd_range": (c_int32, [ctypes.POINTER(HsFrame), ctypes.POINTER(HsScene),
                                          ctypes.POINTER(HsCamera), ctypes.POINTER(HsGrads),
                                          c_int64, c_int64, c_void_p]),
    "hs_merge_rows": (c_int32, [ctypes.POINTER(HsFrame), c_void_p, c_void_p]),
    "hs_preprocess_bwd_views": (c_int32, [ctypes.POINTER(HsScene), c_int32,
                                          ctypes.POINTER(HsCamera), c_void_p, c_int32,
                                          ctypes.POINTER(HsGrads), c_int64, c_int64, c_void_p]),
    "hs_frame_export": (c_int32, [ctypes.POINTER(HsFrame), c_void_p, c_void_p, c_void_p,
                                  c_void_p, c_void_p, c_void_p, c_void_p, c_void_p]),
    "hs_screen_splats": (c_int32, [ctypes.POINTER(HsScene), ctypes.POINTER(HsCamera), c_int32,
                                   c_void_p, c_void_p]),
    "hs_forward_tiles": (c_int32, [c_void_p, c_void_p, c_void_p, c_void_p, c_int64, c_int64,
                                   c_int32, c_int32, c_int32, c_void_p, c_void_p, c_void_p,
                                   c_void_p, c_void_p, c_void_p, c_int32, c_int32]),
    "hs_backward_tiles": (c_int32, [c_void_p, c_void_p, c_void_p, c_void_p, c_int64, c_int64,
                                    c_int32, c_int32, c_int32, c_void_p, c_void_p, c_void_p,
                                    c_void_p, c_void_p, c_int32, c_int32]),
    "hs_loss_workspace_size": (c_size_t, [c_int32, c_int32, c_int32]),
    "hs_loss": (c_int32, [c_void_p, c_void_p, c_int32, c_int32, c_int32, ctypes.c_double,
                          c_void_p, c_void_p, c_void_p, c_void_p, c_size_t, c_void_p]),
    "hs_loss_f64": (c_int32, [c_void_p, c_void_p, c_int32, c_int32, c_int32, ctypes.c_double,
                              c_void_p, c_void_p, c_void_p, c_void_p, c_size_t, c_void_p]),
    "hs_adam_step": (c_int32, [ctypes.POINTER(HsScene), ctypes.POINTER(HsGrads),
                               ctypes.POINTER(HsAdamState), ctypes.POINTER(ctypes.c_double),
                               c_int32, c_void_p]),
    "hs_densify_stats_update": (c_int32, [ctypes.POINTER(HsDensifyStats),
                                          ctypes.POINTER(HsGrads), c_int64, c_int32, c_void_p]),
    "hs_densify_workspace_size": (c_size_t, [c_int64]),
    "hs_densify_plan_compute": (c_int32, [ctypes.POINTER(HsScene), ctypes.POINTER(HsDensifyStats),
                                          ctypes.POINTER(HsDensifyConfig),
                                          ctypes.POINTER(HsDensifyPlan), c_void_p, c_size_t,
                                          c_void_p]),
    "hs_densify_apply": (c_int32, [ctypes.POINTER(HsScene), ctypes.POINTER(HsDensifyStats),
                                   ctypes.POINTER(HsDensifyConfig), ctypes.POINTER(HsDensifyPlan),
                                   c_void_p, c_size_t, c_void_p, ctypes.c_uint64,
                                   ctypes.POINTER(HsAdamState), ctypes.POINTER(HsScene),
                                   ctypes.POINTER(HsAdamState), c_void_p]),
    "hs_reset_opacity": (c_int32, [ctypes.POINTER(HsScene), ctypes.c_double,
                                   ctypes.POINTER(HsAdamState), c_void_p]),
    "hs_ply_unpack": (c_int32, [c_void_p, ctypes.POINTER(HsPlyLayout), ctypes.POINTER(HsScene),
                                c_void_p]),
    "hs_ply_row_bytes": (c_int32, [c_int32, c_int32]),
    "hs_ply_pack": (c_int32, [ctypes.POINTER(HsScene), c_void_p, c_int32, c_void_p]),
    "hs_opacity_disparity_workspace_size": (c_size_t, [c_int64]),
    "hs_opacity_disparity": (c_int32, [ctypes.POINTER(HsScene), c_void_p, c_void_p, c_size_t,
                                       c_void_p]),
    "hs_comm_unique_id": (c_int32, [c_void_p]),
    "hs_comm_init": (c_int32, [ctypes.POINTER(c_void_p), c_int32, c_int32, c_void_p]),
    "hs_comm_destroy": (c_int32, [c_void_p]),
    "hs_comm_info": (c_int32, [c_void_p, ctypes.POINTER(c_int32), ctypes.POINTER(c_int32),
                               ctypes.POINTER(c_int32)]),
    "hs_grad_allreduce": (c_int32, [c_void_p, ctypes.POINTER(HsGrads), c_int64, c_int32, c_int32,
                                    c_int64, c_int64, c_int32, c_void_p]),
    "hs_bin_async": (c_int32, [ctypes.POINTER(HsFrame), c_void_p]),
    "hs_frame_status": (c_int32, [ctypes.POINTER(HsFrame), ctypes.POINTER(c_int64),
                                  ctypes.POINTER(c_int32), c_void_p]),
    "hs_frame_status_async": (c_int32, [ctypes.POINTER(HsFrame), c_void_p, c_void_p]),
    "hs_seam1_cache_clear": (None, []),
    "hs_status_string": (ctypes.c_char_p, [c_int32]),
    "hs_last_cuda_error": (ctypes.c_char_p, []),
    "hs_kernel_launch_count": (c_int64, []),
    "hs_abi_version": (c_int32, []),
    "hs_measure_fp32_peaks": (c_int32, [ctypes.POINTER(ctypes.c_double),
                                        ctypes.POINTER(ctypes.c_double)]),
    "hs_last_fma2_tflops": (ctypes.c_double, []),
    "hs_probe_erf32": (c_int32, [c_void_p, c_void_p, c_int64, c_void_p]),
}

EXPORTED_SYMBOLS = tuple(_SIGNATURES)

_lib = None


def library_path():
    return _LIB_PATH


def load():
    """Load (once) and return the ctypes handle; raises if the .so is missing."""
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(_LIB_PATH):
        raise errors.NativeLibraryMissing(
            f"{_LIB_PATH} not built; run `python -m paper_2406_02720_b200.build` "
            "(there is no CPU fallback)"
        )
    lib = ctypes.CDLL(_LIB_PATH)
    for name, (res, args) in _SIGNATURES.items():
        fn = getattr(lib, name)
        fn.restype = res
        fn.argtypes = args
    _lib = lib
    return lib


_STATUS_ERRORS = {
    HS_ERR_EMPTY_SCENE: errors.EmptyScene,
    HS_ERR_IMAGE_TOO_LARGE: errors.ImageTooLarge,
    HS_ERR_INVALID_KERNEL: ValueError,
    HS_ERR_MISMATCHED_FORWARD: errors.MismatchedForward,
    HS_ERR_INVALID_ARG: ValueError,
    HS_ERR_WORKSPACE: errors.WorkspaceError,
    HS_ERR_IMAGE_TOO_SMALL: errors.ImageTooSmall,
    HS_ERR_INVALID_LAMBDA: ValueError,
}


def check(status, what=""):
    """Raise the Python exception matching a C status code (errors.py names)."""
    if status == HS_OK:
        return
    lib = load()
    msg = lib.hs_status_string(status).decode()
    if status == HS_ERR_CUDA:
        raise errors.CudaError(f"{what}: {lib.hs_last_cuda_error().decode()}")
    raise _STATUS_ERRORS.get(status, errors.HalfSplatError)(f"{what}: {msg}")


def launch_count():
    return int(load().hs_kernel_launch_count())
