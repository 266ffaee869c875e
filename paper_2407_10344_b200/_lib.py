"""ctypes binding of libgvox.so (include/gvox.h).  Argument marshalling only:
every step of the hot path runs in the library's CUDA kernels.  There is no
fallback: if the library is missing or cannot be loaded, importing fails."""
from __future__ import annotations

import ctypes
import os

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
# GVOX_LIB overrides the library path (kernel-variant experiments; see tools/)
LIB_PATH = os.environ.get("GVOX_LIB") or os.path.join(HERE, "libgvox.so")

MAX_LEVELS = 8
GVOX_HOST = 0
GVOX_DEVICE = 1
F_VALIDATE_SURFACE = 1
F_ERROR_ONLY = 2
TIMERS = ("build", "overlap", "linearize", "reduce", "register", "preprocess", "solve")

STATUS = {0: "GVOX_OK", 1: "GVOX_ERR_INVALID", 2: "GVOX_ERR_RANGE", 3: "GVOX_ERR_CUDA",
          4: "GVOX_ERR_NOMEM"}

# numpy mirrors of the ABI structs (layouts asserted against sizeof in tests)
FACTOR_DTYPE = np.dtype([("source_cloud", "<i4"), ("target_map", "<i4"), ("pose_i", "<i4"),
                         ("pose_j", "<i4"), ("flags", "<u4")])
PAIR_DTYPE = np.dtype([("source_cloud", "<i4"), ("target_map", "<i4"), ("pose_i", "<i4"),
                       ("pose_j", "<i4")])
LINEAR_FACTOR_DTYPE = np.dtype([("H_ii", "<f8", (36,)), ("H_ij", "<f8", (36,)),
                                ("H_jj", "<f8", (36,)), ("b_i", "<f8", (6,)), ("b_j", "<f8", (6,)),
                                ("error", "<f8"), ("inliers", "<i4", (MAX_LEVELS,)),
                                ("num_invisible", "<i4"), ("num_degenerate", "<i4")])
FACTOR_ACCUM_DTYPE = np.dtype([("terms", "<f8", (28,)), ("inliers", "<i4", (MAX_LEVELS,)),
                               ("num_invisible", "<i4"), ("num_degenerate", "<i4"),
                               ("reserved", "<i4", (6,))])
REGISTER_PARAMS_DTYPE = np.dtype([("max_iterations", "<i4"), ("reserved", "<i4"), ("lambda", "<f8"),
                                  ("eps_rot", "<f8"), ("eps_trans", "<f8")])
REGISTER_RESULT_DTYPE = np.dtype([("status", "<i4"), ("iterations", "<i4"), ("inliers", "<i4"),
                                  ("reserved", "<i4"), ("error_initial", "<f8"),
                                  ("error_final", "<f8"), ("last_step", "<f8", (6,))])
UNION_QUERY_DTYPE = np.dtype([("source_cloud", "<i4"), ("pose_i", "<i4"), ("first", "<i4"),
                              ("count", "<i4")])
UNION_MEMBER_DTYPE = np.dtype([("target_map", "<i4"), ("pose_j", "<i4")])
GLOBAL_PARAMS_DTYPE = np.dtype([("max_iterations", "<i4"), ("reserved", "<i4"), ("tol", "<f8"),
                                ("lambda", "<f8")])
GLOBAL_RESULT_DTYPE = np.dtype([("iterations", "<i4"), ("converged", "<i4"), ("num_variables", "<i4"),
                                ("num_blocks", "<i4"), ("residual_initial", "<f8"),
                                ("residual_final", "<f8")])
OPTIMIZE_PARAMS_DTYPE = np.dtype([("max_iterations", "<i4"), ("pcg_max_iterations", "<i4"),
                                  ("pcg_tol", "<f8"), ("lambda", "<f8"), ("eps_rot", "<f8"),
                                  ("eps_trans", "<f8")])
OPTIMIZE_RESULT_DTYPE = np.dtype([("iterations", "<i4"), ("converged", "<i4"), ("pcg_iterations", "<i4"),
                                  ("reserved", "<i4"), ("error_initial", "<f8"), ("error_final", "<f8"),
                                  ("last_step_rot", "<f8"), ("last_step_trans", "<f8")])
REG_FIXED, REG_MAX_ITER, REG_CONVERGED, REG_SINGULAR = 0, 1, 2, 3

# exported symbols (tests check every one declared in include/gvox.h is here)
SYMBOLS = [
    "gvox_ctx_create", "gvox_ctx_set_stream", "gvox_ctx_destroy", "gvox_ctx_enable_timing",
    "gvox_ctx_timing", "gvox_cloud_create", "gvox_clouds_create", "gvox_cloud_size",
    "gvox_cloud_destroy",
    "gvox_create_voxelmap", "gvox_create_voxelmaps", "gvox_voxelmap_info", "gvox_voxelmap_levels",
    "gvox_voxelmap_export", "gvox_voxelmap_lookup", "gvox_map_destroy", "gvox_maps_destroy",
    "gvox_overlap", "gvox_overlap_select", "gvox_linearize_batch", "gvox_linearize_batch_accum",
    "gvox_linearize_batch_accum_select", "gvox_expand",
    "gvox_register_batch", "gvox_overlap_union", "gvox_keyframe_update",
    "gvox_keyframe_insert_test", "gvox_keyframe_update_counts", "gvox_knn",
    "gvox_estimate_covariances", "gvox_solve_global", "gvox_optimize_global",
    "gvox_status_string", "gvox_last_error", "gvox_launch_count", "gvox_last_linearize_variant",
    "gvox_version",
]


class GvoxError(RuntimeError):
    def __init__(self, status: int, message: str):
        super().__init__(f"{STATUS.get(status, status)}: {message}")
        self.status = status


_lib = None


def lib():
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(LIB_PATH):
        raise ImportError(f"libgvox.so not built at {LIB_PATH}: run __graft_entry__.build() "
                          "(there is no CPU fallback)")
    L = ctypes.CDLL(LIB_PATH)
    P, I64, I32, D = ctypes.c_void_p, ctypes.c_int64, ctypes.c_int, ctypes.c_double
    PP = ctypes.POINTER(ctypes.c_void_p)
    sig = {
        "gvox_ctx_create": (I32, [I32, P, PP]),
        "gvox_ctx_set_stream": (I32, [P, P]),
        "gvox_ctx_destroy": (None, [P]),
        "gvox_ctx_enable_timing": (I32, [P, I32]),
        "gvox_ctx_timing": (I32, [P, P, P, I32]),
        "gvox_cloud_create": (I32, [P, P, P, P, I64, I32, PP]),
        "gvox_clouds_create": (I32, [P, P, P, P, P, I64, I32, P]),
        "gvox_cloud_size": (I64, [P]),
        "gvox_cloud_destroy": (None, [P]),
        "gvox_create_voxelmap": (I32, [P, P, D, I32, PP]),
        "gvox_create_voxelmaps": (I32, [P, P, I64, D, I32, P]),
        "gvox_voxelmap_info": (I32, [P, I32, P, P]),
        "gvox_voxelmap_levels": (I32, [P]),
        "gvox_voxelmap_export": (I32, [P, P, I32, P, P, P, P]),
        "gvox_voxelmap_lookup": (I32, [P, P, I32, P, I64, P, I32]),
        "gvox_map_destroy": (None, [P]),
        "gvox_maps_destroy": (None, [P, I64]),
        "gvox_overlap": (I32, [P, P, I64, P, I64, P, I64, P, I64, I32, P, I32]),
        "gvox_overlap_select": (I32, [P, P, I64, P, I64, P, I64, P, I64, I32, I32, I32, P, I32]),
        "gvox_linearize_batch": (I32, [P, P, I64, P, I64, P, I64, P, I64, P, I32, P]),
        "gvox_linearize_batch_accum": (I32, [P, P, I64, P, I64, P, I64, P, I64, P, I32]),
        "gvox_linearize_batch_accum_select": (I32, [P, P, I64, P, I64, P, I64, P, P, I64, P, P, P]),
        "gvox_expand": (I32, [P, P, I64, P, I64, P, P, I32]),
        "gvox_solve_global": (I32, [P, P, I64, P, P, I64, P, P, P, P, P, P, I32]),
        "gvox_optimize_global": (I32, [P, P, I64, P, I64, P, I64, P, I64, P, P, P, P, P, I32]),
        "gvox_knn": (I32, [P, P, P, I64, I32, D, P, I32]),
        "gvox_estimate_covariances": (I32, [P, P, P, I64, P, I32, P, P, I32]),
        "gvox_overlap_union": (I32, [P, P, I64, P, I64, P, I64, P, I64, P, I64, I32, P, I32]),
        "gvox_keyframe_update": (I32, [P, I32, I32, D, P]),
        "gvox_keyframe_insert_test": (I32, [I64, I64, I32, I32, P]),
        "gvox_keyframe_update_counts": (I32, [P, P, I32, I32, D, P, P]),
        "gvox_register_batch": (I32, [P, P, I64, P, I64, P, I64, P, I64, P, P, P, P, I32]),
        "gvox_status_string": (ctypes.c_char_p, [I32]),
        "gvox_last_error": (ctypes.c_char_p, []),
        "gvox_launch_count": (I64, [I32]),
        "gvox_last_linearize_variant": (I32, []),
        "gvox_version": (ctypes.c_char_p, []),
    }
    for name, (res, args) in sig.items():
        fn = getattr(L, name)
        fn.restype = res
        fn.argtypes = args
    _lib = L
    return L


def check(status: int):
    if status != 0:
        msg = lib().gvox_last_error().decode(errors="replace")
        raise GvoxError(status, msg)


def launch_count(reset: bool = False) -> int:
    return int(lib().gvox_launch_count(int(reset)))


def last_linearize_variant() -> int:
    """GVOX_LINVAR_* bits | level capacity << 8 of the last k_linearize launch."""
    return int(lib().gvox_last_linearize_variant())


def version() -> str:
    return lib().gvox_version().decode()
