"""paper_2407_10344_b200 -- B200-native batched VGICP linearization (GLIM,
arXiv 2407.10344): libgvox.so (hand-written sm_100a CUDA behind the C ABI of
include/gvox.h) and its thin Python binding.

Importing this package loads libgvox.so and raises if it is missing; there is
no CPU fallback.
"""
from ._lib import (FACTOR_ACCUM_DTYPE, FACTOR_DTYPE, F_ERROR_ONLY, F_VALIDATE_SURFACE,
                   GVOX_DEVICE, GVOX_HOST, LINEAR_FACTOR_DTYPE, MAX_LEVELS, PAIR_DTYPE,
                   REG_CONVERGED, REG_FIXED, REG_MAX_ITER, REG_SINGULAR, REGISTER_PARAMS_DTYPE,
                   REGISTER_RESULT_DTYPE, GvoxError, launch_count, last_linearize_variant, lib,
                   version)
from .api import (Cloud, Context, HandleArray, VoxelMap, as_factors, as_pairs, as_poses,
                  corr_dump_size, create_clouds, create_voxelmap, create_voxelmaps, device_records, expand,
                  full_blocks, linearize_batch, linearize_batch_accum, linearize_batch_accum_select,
                  overlap, overlap_select,
                  records_to_numpy, register_batch, overlap_union, keyframe_update,
                  keyframe_insert_test, keyframe_update_counts,
                  KeyframeList, knn, estimate_covariances, solve_global,
                  optimize_global)

lib()  # fail loudly at import if the CUDA library is absent

__all__ = [
    "Cloud", "Context", "VoxelMap", "HandleArray", "create_clouds", "create_voxelmap", "create_voxelmaps",
    "overlap", "overlap_select", "linearize_batch", "linearize_batch_accum",
    "linearize_batch_accum_select", "expand", "device_records",
    "records_to_numpy", "register_batch", "overlap_union", "keyframe_update", "keyframe_insert_test", "keyframe_update_counts", "KeyframeList", "knn", "estimate_covariances", "solve_global", "optimize_global", "full_blocks", "corr_dump_size", "as_factors", "as_pairs", "as_poses",
    "FACTOR_DTYPE", "PAIR_DTYPE", "LINEAR_FACTOR_DTYPE", "FACTOR_ACCUM_DTYPE", "MAX_LEVELS",
    "F_VALIDATE_SURFACE", "F_ERROR_ONLY", "GVOX_HOST", "GVOX_DEVICE", "GvoxError",
    "launch_count", "last_linearize_variant", "version", "lib", "REG_FIXED", "REG_MAX_ITER", "REG_CONVERGED", "REG_SINGULAR",
    "REGISTER_PARAMS_DTYPE", "REGISTER_RESULT_DTYPE",
]
