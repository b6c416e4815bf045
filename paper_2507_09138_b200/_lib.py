"""ctypes binding of libhivf.so (include/hivf.h).

The library is the product: there is no Python/CPU fallback.  Loading fails
loudly if the in-tree libhivf.so is missing (build it with
``python -m paper_2507_09138_b200.build``).
"""
from __future__ import annotations

import ctypes as C
import os

PKG = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(PKG, "libhivf.so")

HIVF_OK, HIVF_EINVAL, HIVF_EINTERNAL, HIVF_ECUDA, HIVF_ENOMEM, HIVF_EUNSUPPORTED, HIVF_ECOMM = range(7)
SHARD_STRIPED = 0xFFFFFFFF

# hivf_allgather_fn: int (*)(void* user, const void* send, size_t bytes, void* recv)
ALLGATHER_FN = C.CFUNCTYPE(C.c_int, C.c_void_p, C.c_void_p, C.c_size_t, C.c_void_p)

# header-declared symbols (tests check every one is exported)
SYMBOLS = [
    "hivf_last_error", "hivf_version", "hivf_ctx_create", "hivf_ctx_destroy",
    "hivf_ctx_set_stream", "hivf_ctx_synchronize", "hivf_device_info", "hivf_index_upload",
    "hivf_index_upload_device", "hivf_index_begin", "hivf_index_add_rows_device",
    "hivf_index_add_rows_at_device", "hivf_index_finish", "hivf_index_get_rows",
    "hivf_index_destroy", "hivf_index_locate", "hivf_index_gather_rows", "hivf_index_info", "hivf_index_cluster_sizes",
    "hivf_assign", "hivf_search", "hivf_search_device", "hivf_assign_device",
    "hivf_search_planned_device", "hivf_scan_items", "hivf_compute_assignments",
    "hivf_train_kmeans", "hivf_compute_assignments_host", "hivf_train_kmeans_host",
    "hivf_merge_parts_device", "hivf_residency_set", "hivf_residency_get",
    "hivf_residency_sync", "hivf_last_stats",
    "hivf_set_option", "hivf_shard_plan", "hivf_shard_local_lists", "hivf_index_upload_shard",
    "hivf_group_create", "hivf_nccl_unique_id", "hivf_group_create_nccl", "hivf_group_create_hostcb",
    "hivf_group_destroy", "hivf_group_search_device", "hivf_group_search", "hivf_train_kmeans_sampled_seeds",
    "hivf_index_row_distances", "hivf_debug_tc_dot", "hivf_debug_bound", "hivf_debug_tc_prof", "hivf_debug_tc2_dot", "hivf_debug_mma_rate",
]


class HivfError(RuntimeError):
    def __init__(self, status, msg):
        super().__init__(f"hivf status {status}: {msg}")
        self.status = status


class InvalidArgument(HivfError, ValueError):
    """std::invalid_argument of the reference."""


class InternalError(HivfError):
    """std::runtime_error of the reference."""


class Stats(C.Structure):
    _fields_ = [("kernels_launched", C.c_uint32), ("n_work_items", C.c_uint32),
                ("n_fallback", C.c_uint32), ("n_unique_lists", C.c_uint32),
                ("scan_bytes", C.c_uint64), ("timed_calls", C.c_uint32),
                ("assign_ms", C.c_double), ("scan_ms", C.c_double), ("finalize_ms", C.c_double),
                ("scan_kernel", C.c_uint32), ("scan_group", C.c_uint32),
                ("scan_filter_bits", C.c_uint32), ("coarse_filter_bits", C.c_uint32)]


_lib = None


def lib():
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(LIB_PATH):
        raise ImportError(f"{LIB_PATH} missing: build it with `python -m paper_2507_09138_b200.build`"
                          " (the CUDA path is the only path; there is no CPU fallback)")
    L = C.CDLL(LIB_PATH)
    vp, u32, u64, i32, f64 = C.c_void_p, C.c_uint32, C.c_uint64, C.c_int, C.c_double
    P = C.POINTER
    sig = {
        "hivf_last_error": (C.c_char_p, []),
        "hivf_version": (C.c_char_p, []),
        "hivf_ctx_create": (i32, [i32, vp, P(vp)]),
        "hivf_ctx_destroy": (i32, [vp]),
        "hivf_ctx_set_stream": (i32, [vp, vp]),
        "hivf_ctx_synchronize": (i32, [vp]),
        "hivf_device_info": (i32, [vp, P(i32), P(i32)]),
        "hivf_index_upload": (i32, [vp, u32, i32, u32, vp, vp, vp, vp, P(vp)]),
        "hivf_index_upload_device": (i32, [vp, u32, i32, u32, vp, vp, vp, vp, P(vp)]),
        "hivf_index_begin": (i32, [vp, u32, i32, u32, vp, i32, vp, P(vp)]),
        "hivf_index_add_rows_device": (i32, [vp, u64, u64, vp, vp]),
        "hivf_index_add_rows_at_device": (i32, [vp, u64, vp, vp, vp]),
        "hivf_index_finish": (i32, [vp]),
        "hivf_index_get_rows": (i32, [vp, u64, u64, vp, vp]),
        "hivf_index_destroy": (i32, [vp]),
        "hivf_index_locate": (i32, [vp, vp, u32, vp, vp]),
        "hivf_index_gather_rows": (i32, [vp, vp, u32, vp]),
        "hivf_index_info": (i32, [vp, P(u32), P(u32), P(u64), P(u64), P(f64)]),
        "hivf_index_cluster_sizes": (i32, [vp, vp]),
        "hivf_index_row_distances": (i32, [vp, vp]),
        "hivf_debug_tc_dot": (i32, [vp, vp, u32, u32, i32, vp]),
        "hivf_debug_tc2_dot": (i32, [vp, vp, u32, u32, i32, vp]),
        "hivf_debug_bound": (i32, [i32, u32, P(f64), P(f64), P(f64)]),
        "hivf_debug_tc_prof": (i32, [vp, i32]),
        "hivf_debug_mma_rate": (i32, [i32, u32, u32, vp, vp, vp, vp]),
        "hivf_assign": (i32, [vp, vp, u32, u32, vp, vp]),
        "hivf_search": (i32, [vp, vp, u32, u32, u32, vp, vp, vp]),
        "hivf_search_device": (i32, [vp, vp, u32, u32, u32, vp, vp, vp]),
        "hivf_assign_device": (i32, [vp, vp, u32, u32, vp, vp]),
        "hivf_compute_assignments": (i32, [vp, vp, u64, u32, vp, u32, vp]),
        "hivf_train_kmeans": (i32, [vp, vp, u64, u32, u32, u32, u64, vp]),
        "hivf_compute_assignments_host": (i32, [vp, vp, u64, u32, vp, u32, vp]),
        "hivf_train_kmeans_host": (i32, [vp, vp, u64, u32, u32, u32, u64, vp]),
        "hivf_train_kmeans_sampled_seeds": (i32, [vp, vp, u64, u32, u32, u32, u64, vp]),
        "hivf_search_planned_device": (i32, [vp, vp, u32, u32, u32, vp, vp, vp, vp]),
        "hivf_scan_items": (i32, [vp, vp, u32, vp, vp, vp, vp, vp, vp, u32, vp]),
        "hivf_merge_parts_device": (i32, [vp, u32, u32, u32, vp, vp, vp, vp, vp, vp]),
        "hivf_residency_set": (i32, [vp, vp, u32]),
        "hivf_residency_get": (i32, [vp, vp]),
        "hivf_residency_sync": (i32, [vp]),
        "hivf_last_stats": (i32, [vp, P(Stats)]),
        "hivf_set_option": (i32, [vp, C.c_char_p, C.c_int64]),
        "hivf_shard_plan": (i32, [vp, vp, u32, u32, C.c_int32, vp]),
        "hivf_shard_local_lists": (i32, [vp, vp, u32, u32, u32, vp, vp]),
        "hivf_index_upload_shard": (i32, [vp, u32, i32, u32, vp, vp, vp, vp, vp, u32, u32, P(vp)]),
        "hivf_group_create": (i32, [vp, u32, P(vp)]),
        "hivf_nccl_unique_id": (i32, [vp]),
        "hivf_group_create_nccl": (i32, [vp, u32, u32, vp, P(vp)]),
        "hivf_group_create_hostcb": (i32, [vp, u32, u32, ALLGATHER_FN, vp, P(vp)]),
        "hivf_group_destroy": (i32, [vp]),
        "hivf_group_search_device": (i32, [vp, vp, u32, u32, u32, vp, vp, vp]),
        "hivf_group_search": (i32, [vp, vp, u32, u32, u32, vp, vp, vp]),
    }
    for name, (res, args) in sig.items():
        f = getattr(L, name)
        f.restype = res
        f.argtypes = args
    _lib = L
    return L


def check(status: int) -> None:
    if status == HIVF_OK:
        return
    msg = lib().hivf_last_error().decode(errors="replace")
    if status == HIVF_EINVAL:
        raise InvalidArgument(status, msg)
    if status == HIVF_EINTERNAL:
        raise InternalError(status, msg)
    raise HivfError(status, msg)
