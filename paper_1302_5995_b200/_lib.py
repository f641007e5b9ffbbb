"""ctypes binding of libdtn_b200.so (include/dtn_gpu.h). The product path has
no CPU fallback: a missing library or device raises."""
from __future__ import annotations

import ctypes as C
import os
import subprocess

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(_HERE, "_lib", "libdtn_b200.so")
HEADER = os.path.join(os.path.dirname(_HERE), "include", "dtn_gpu.h")

DTN_OK, DTN_EINVAL, DTN_ESINGULAR, DTN_ECUDA = 0, 2, 3, 5


class dtn_problem(C.Structure):
    _fields_ = [("n", C.c_int32), ("stencil", C.c_void_p), ("stencil_on_device", C.c_int32),
                ("shard_S", C.POINTER(C.c_void_p)), ("shard_S_on_device", C.c_int32)]


class dtn_opts(C.Structure):
    _fields_ = [("engine", C.c_int32), ("n_leaf", C.c_int32), ("leaf_side", C.c_int32), ("want_G", C.c_int32),
                ("micro_max", C.c_int32), ("profile", C.c_int32), ("epsilon", C.c_double),
                ("crossover", C.c_int64), ("nshards", C.c_int32), ("shard", C.c_int32),
                ("export_S", C.c_void_p), ("export_lds", C.c_int64),
                ("load_ids", C.c_void_p), ("nloads", C.c_int32), ("keep_boxes", C.c_int32),
                ("rank_base", C.c_int32), ("rank_step", C.c_int32)]


class dtn_level_stats(C.Structure):
    _fields_ = [("level", C.c_int32), ("boxes", C.c_int32), ("max_boundary", C.c_int64), ("seconds", C.c_double),
                ("flops", C.c_double), ("max_rank", C.c_int64), ("bytes", C.c_uint64)]


class dtn_build_stats(C.Structure):
    _fields_ = [("build_ms", C.c_double), ("leaf_ms", C.c_double), ("merge_ms", C.c_double),
                ("inverse_ms", C.c_double), ("merge_flops", C.c_double), ("leaf_flops", C.c_double),
                ("inverse_flops", C.c_double), ("waves", C.c_int32), ("launches", C.c_int32),
                ("arena_bytes", C.c_double), ("arena_sum_bytes", C.c_double), ("structured_merges", C.c_int32),
                ("max_rank", C.c_int32), ("sketch_tail", C.c_double), ("exec_flops", C.c_double),
                ("rank_attempts", C.c_int32)]


class dtn_kernel_stats(C.Structure):
    _fields_ = [("name", C.c_char * 16), ("launches", C.c_int32), ("ms", C.c_double), ("max_ms", C.c_double),
                ("flops", C.c_double), ("bytes", C.c_double)]


EXPORTS = [
    "dtn_gpu_create", "dtn_gpu_nccl_unique_id", "dtn_gpu_create_rank", "dtn_gpu_destroy", "dtn_gpu_last_error", "dtn_gpu_set_stream", "dtn_gpu_build",
    "dtn_gpu_free", "dtn_gpu_boundary", "dtn_gpu_export", "dtn_gpu_export_device", "dtn_gpu_device_ptrs",
    "dtn_gpu_apply", "dtn_gpu_ring_dtn", "dtn_gpu_body_map",
    "dtn_gpu_num_boxes", "dtn_gpu_box_info", "dtn_gpu_box_schur", "dtn_gpu_level_stats", "dtn_gpu_build_stats", "dtn_gpu_kernel_stats",
    "dtn_discretize_continuum", "dtn_discretize_network", "dtn_debug_partial_lu", "dtn_debug_gemm", "dtn_debug_fused_clocks", "dtn_gpu_shard_info",
    "dtn_gpu_hbs_compress", "dtn_gpu_hbs_compress_op", "dtn_gpu_hbs_free", "dtn_gpu_hbs_info", "dtn_gpu_hbs_tree",
    "dtn_gpu_hbs_factor", "dtn_gpu_hbs_apply", "dtn_gpu_hbs_serialize", "dtn_gpu_hbs_deserialize",
    "dtn_gpu_hbs_invert", "dtn_gpu_build_accel", "dtn_gpu_root_rhs", "dtn_gpu_hbs_launch_count", "dtn_gpu_collective_flops",
    "dtn_gpu_hbs_compress_tree", "dtn_gpu_hbs_reconstruct", "dtn_gpu_hbs_subtree", "dtn_gpu_hbs_flip",
    "dtn_gpu_hbs_scale", "dtn_gpu_hbs_scale_rows", "dtn_gpu_hbs_scale_cols", "dtn_gpu_hbs_add",
    "dtn_gpu_hbs_from_lowrank", "dtn_gpu_hbs_add_lowrank", "dtn_gpu_hbs_rebase", "dtn_gpu_hbs_split_at",
    "dtn_gpu_hbs_consolidate", "dtn_gpu_lowrank_create", "dtn_gpu_lowrank_from_dense", "dtn_gpu_lowrank_info",
    "dtn_gpu_lowrank_get", "dtn_gpu_lowrank_recompress", "dtn_gpu_lowrank_sum", "dtn_gpu_lowrank_free",
]

_lib = None


def build() -> str:
    """Compile the extension in-tree (nvcc, sm_100a)."""
    subprocess.run(["make", "-s", "-j8", "-C", _HERE], check=True)
    return LIB_PATH


def lib():
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(LIB_PATH):
        raise RuntimeError(f"libdtn_b200.so is not built ({LIB_PATH}); run paper_1302_5995_b200._lib.build()")
    L = C.CDLL(LIB_PATH)
    vp, i32, i64, f64 = C.c_void_p, C.c_int32, C.c_int64, C.c_double
    P = C.POINTER
    L.dtn_gpu_create.argtypes = [P(vp), C.c_int]
    L.dtn_gpu_destroy.argtypes = [vp]
    L.dtn_gpu_destroy.restype = None
    L.dtn_gpu_last_error.argtypes = [vp]
    L.dtn_gpu_last_error.restype = C.c_char_p
    L.dtn_gpu_set_stream.argtypes = [vp, vp]
    L.dtn_gpu_build.argtypes = [vp, P(dtn_problem), P(dtn_opts), P(vp)]
    L.dtn_gpu_free.argtypes = [vp]
    L.dtn_gpu_free.restype = None
    L.dtn_gpu_boundary.argtypes = [vp, vp, P(i64)]
    L.dtn_gpu_export.argtypes = [vp, vp, vp, P(f64)]
    L.dtn_gpu_device_ptrs.argtypes = [vp, P(vp), P(vp), P(i64)]
    L.dtn_gpu_export_device.argtypes = [vp, vp, i64, vp, i64]
    L.dtn_gpu_apply.argtypes = [vp, C.c_int, vp, i64, i64, vp, i64, C.c_int]
    L.dtn_gpu_ring_dtn.argtypes = [vp, vp, vp, i64, C.c_double, vp, i64, C.c_int]
    L.dtn_gpu_body_map.argtypes = [vp, vp, i64, C.c_int]
    L.dtn_gpu_num_boxes.argtypes = [vp, P(i32), P(i32)]
    L.dtn_gpu_box_info.argtypes = [vp, i32, P(i32)]
    L.dtn_gpu_box_schur.argtypes = [vp, i32, vp]
    L.dtn_gpu_level_stats.argtypes = [vp, P(dtn_level_stats), i32, P(i32)]
    L.dtn_gpu_build_stats.argtypes = [vp, P(dtn_build_stats)]
    L.dtn_gpu_kernel_stats.argtypes = [vp, P(dtn_kernel_stats), i32, P(i32)]
    L.dtn_discretize_continuum.argtypes = [i32, vp, vp, vp, vp]
    L.dtn_discretize_network.argtypes = [i32, f64, f64, C.c_uint64, vp]
    L.dtn_debug_partial_lu.argtypes = [i32, i32, vp, vp, vp, vp]
    L.dtn_debug_gemm.argtypes = [i32, i32, i32, vp, vp, vp, f64, f64, i32]
    L.dtn_debug_fused_clocks.argtypes = [vp]
    L.dtn_gpu_shard_info.argtypes = [i32, i32, i32, i32, i32, P(i32), P(i64)]
    L.dtn_gpu_hbs_compress.argtypes = [vp, vp, i64, i64, C.c_int, f64, i64, P(vp)]
    L.dtn_gpu_hbs_compress_op.argtypes = [vp, C.c_int, f64, i64, P(vp)]
    L.dtn_gpu_hbs_free.argtypes = [vp]
    L.dtn_gpu_hbs_free.restype = None
    L.dtn_gpu_hbs_info.argtypes = [vp, P(i64), P(i64), P(i32), P(i64), P(C.c_uint64)]
    L.dtn_gpu_hbs_tree.argtypes = [vp, vp, vp]
    L.dtn_gpu_hbs_factor.argtypes = [vp, i32, i32, vp, P(i64), P(i64)]
    L.dtn_gpu_hbs_apply.argtypes = [vp, vp, i64, i64, vp, i64, C.c_int]
    L.dtn_gpu_hbs_serialize.argtypes = [vp, vp, C.c_uint64, P(C.c_uint64)]
    L.dtn_gpu_hbs_deserialize.argtypes = [vp, vp, C.c_uint64, P(vp)]
    L.dtn_gpu_hbs_invert.argtypes = [vp, P(vp)]
    L.dtn_gpu_root_rhs.argtypes = [vp, vp, i64, C.c_int]
    L.dtn_gpu_nccl_unique_id.argtypes = [vp]
    L.dtn_gpu_create_rank.argtypes = [P(vp), C.c_int, C.c_int, C.c_int, vp]
    L.dtn_gpu_collective_flops.argtypes = [i32, i32, i32, i32, i32, vp, vp]
    L.dtn_gpu_hbs_launch_count.argtypes = []
    L.dtn_gpu_hbs_launch_count.restype = C.c_ulonglong
    L.dtn_gpu_build_accel.argtypes = [vp, vp, vp, i64, P(vp), P(vp), P(vp), P(f64)]
    ci = C.c_int
    L.dtn_gpu_hbs_compress_tree.argtypes = [vp, vp, i64, i64, ci, f64, vp, i64, P(vp)]
    L.dtn_gpu_hbs_reconstruct.argtypes = [vp, vp, i64, ci]
    L.dtn_gpu_hbs_subtree.argtypes = [vp, i32, P(vp)]
    L.dtn_gpu_hbs_flip.argtypes = [vp, P(vp)]
    L.dtn_gpu_hbs_scale.argtypes = [vp, f64]
    L.dtn_gpu_hbs_scale_rows.argtypes = [vp, vp, ci]
    L.dtn_gpu_hbs_scale_cols.argtypes = [vp, vp, ci]
    L.dtn_gpu_hbs_add.argtypes = [vp, vp, f64, P(vp)]
    L.dtn_gpu_hbs_from_lowrank.argtypes = [vp, vp, i64, vp, i64, i64, vp, i64, ci, P(vp)]
    L.dtn_gpu_hbs_add_lowrank.argtypes = [vp, vp, i64, vp, i64, i64, f64, ci, P(vp)]
    L.dtn_gpu_hbs_rebase.argtypes = [vp, vp, i64, f64, P(vp)]
    L.dtn_gpu_hbs_split_at.argtypes = [vp, i64, f64, P(vp), P(vp), P(vp), P(vp)]
    L.dtn_gpu_hbs_consolidate.argtypes = [vp, i64, i64, vp, vp, i64, vp, vp, f64, P(vp)]
    L.dtn_gpu_lowrank_create.argtypes = [vp, vp, i64, vp, i64, i64, i64, i64, ci, P(vp)]
    L.dtn_gpu_lowrank_from_dense.argtypes = [vp, vp, i64, i64, i64, ci, f64, P(vp)]
    L.dtn_gpu_lowrank_info.argtypes = [vp, P(i64), P(i64), P(i64)]
    L.dtn_gpu_lowrank_get.argtypes = [vp, vp, i64, vp, i64]
    L.dtn_gpu_lowrank_recompress.argtypes = [vp, f64, P(vp)]
    L.dtn_gpu_lowrank_sum.argtypes = [vp, i64, i64, i64, vp, vp, f64, P(vp)]
    L.dtn_gpu_lowrank_free.argtypes = [vp]
    L.dtn_gpu_lowrank_free.restype = None
    _lib = L
    return L
