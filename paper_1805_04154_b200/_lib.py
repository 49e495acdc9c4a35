"""ctypes binding of librunsort_b200.so (C ABI declared in include/runsort_b200.h).

The product path has no CPU fallback: if the library is missing or no CUDA
device is visible, calls fail loudly.
"""
from __future__ import annotations

import ctypes
import os

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("RS_LIB") or os.path.join(HERE, "librunsort_b200.so")

RS_OK, RS_EINVAL, RS_EINVARIANT, RS_ENOMEM, RS_ECUDA, RS_EUNSUPPORTED = range(6)
RS_ALGO_POWERSORT, RS_ALGO_PEEKSORT = 0, 1
RS_ALGO_TOP_DOWN, RS_ALGO_BOTTOM_UP, RS_ALGO_ALPHA_STACK, RS_ALGO_ALPHA_MERGE = 2, 3, 4, 5
RS_KEY_I32, RS_KEY_I64 = 1, 2
RS_MERGE_BITONIC, RS_MERGE_CLASSIC = 0, 1
RS_EIO = 6
RS_ECAPACITY = 7  # peeksort's compact replay workspace overflowed (input unchanged): retry with RS_ALGO_FULL_WS
RS_ALGO_FULL_WS = 0x100

# every symbol include/runsort_b200.h declares
EXPORTS = ("rs_workspace_bytes", "rs_sort", "rs_sort_ex", "rs_fetch_metrics", "rs_sort_host", "rs_sort_host_ex", "rs_export_tree", "rs_profile",
           "rs_profile_read", "rs_debug_counters", "rs_max_min_run_len", "rs_load_bin", "rs_corank", "rs_kway_workspace_bytes", "rs_kway_merge",
           "rs_corank_rank", "rs_kway_split_workspace_bytes", "rs_kway_merge_split",
           "rs_merge_runs_workspace_bytes", "rs_merge_runs",
           "rs_ipc_alloc", "rs_ipc_open", "rs_ipc_close", "rs_ipc_free", "rs_last_error",
           "rs_version")


class RsMetrics(ctypes.Structure):
    _fields_ = [("merge_cost", ctypes.c_uint64), ("comparisons", ctypes.c_uint64),
                ("runs_detected", ctypes.c_uint64), ("max_stack_height", ctypes.c_uint64)]


class RsTree(ctypes.Structure):
    _fields_ = [("capacity", ctypes.c_int64), ("n_leaves", ctypes.c_int64),
                ("leaf_len", ctypes.c_void_p), ("node_power", ctypes.c_void_p),
                ("node_depth", ctypes.c_void_p)]


class RsShard(ctypes.Structure):
    _fields_ = [("keys", ctypes.c_void_p), ("tags", ctypes.c_void_p), ("lo", ctypes.c_int64),
                ("hi", ctypes.c_int64)]


_lib = None


def lib():
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            raise RuntimeError(
                f"{LIB_PATH} is missing: build the CUDA extension with "
                "`python -c 'import __graft_entry__ as g; g.build()'` (no CPU fallback exists)")
        L = ctypes.CDLL(LIB_PATH)
        L.rs_workspace_bytes.restype = ctypes.c_size_t
        L.rs_workspace_bytes.argtypes = [ctypes.c_int, ctypes.c_int, ctypes.c_int, ctypes.c_int64, ctypes.c_int32]
        L.rs_sort.restype = ctypes.c_int
        L.rs_sort.argtypes = [ctypes.c_int, ctypes.c_int, ctypes.c_void_p, ctypes.c_int, ctypes.c_void_p,
                              ctypes.c_int64, ctypes.c_int32, ctypes.c_int32, ctypes.c_void_p, ctypes.c_size_t,
                              ctypes.c_void_p, ctypes.POINTER(RsMetrics), ctypes.POINTER(RsTree)]
        L.rs_sort_ex.restype = ctypes.c_int
        L.rs_sort_ex.argtypes = [ctypes.c_int, ctypes.c_int, ctypes.c_void_p, ctypes.c_int, ctypes.c_void_p,
                                 ctypes.c_int64, ctypes.c_int32, ctypes.c_int32, ctypes.c_double, ctypes.c_void_p,
                                 ctypes.c_size_t, ctypes.c_void_p, ctypes.POINTER(RsMetrics), ctypes.POINTER(RsTree)]
        L.rs_fetch_metrics.restype = ctypes.c_int
        L.rs_fetch_metrics.argtypes = [ctypes.c_int, ctypes.c_int, ctypes.c_int, ctypes.c_int64, ctypes.c_int32,
                                       ctypes.c_void_p, ctypes.c_void_p, ctypes.POINTER(RsMetrics)]
        L.rs_sort_host.restype = ctypes.c_int
        L.rs_sort_host.argtypes = [ctypes.c_int, ctypes.c_int, ctypes.c_void_p, ctypes.c_int, ctypes.c_void_p,
                                   ctypes.c_int64, ctypes.c_int32, ctypes.c_int32, ctypes.POINTER(RsMetrics),
                                   ctypes.POINTER(RsTree)]
        L.rs_sort_host_ex.restype = ctypes.c_int
        L.rs_sort_host_ex.argtypes = [ctypes.c_int, ctypes.c_int, ctypes.c_void_p, ctypes.c_int, ctypes.c_void_p,
                                      ctypes.c_int64, ctypes.c_int32, ctypes.c_int32, ctypes.c_double,
                                      ctypes.POINTER(RsMetrics), ctypes.POINTER(RsTree)]
        L.rs_export_tree.restype = ctypes.c_int
        L.rs_export_tree.argtypes = [ctypes.c_int, ctypes.c_int, ctypes.c_int, ctypes.c_int64, ctypes.c_int32,
                                     ctypes.c_void_p, ctypes.c_void_p, ctypes.POINTER(RsTree)]
        L.rs_profile.restype = ctypes.c_int
        L.rs_profile.argtypes = [ctypes.c_int]
        L.rs_profile_read.restype = ctypes.c_int
        L.rs_profile_read.argtypes = [ctypes.POINTER(ctypes.c_double), ctypes.c_int]
        L.rs_debug_counters.restype = ctypes.c_int
        L.rs_debug_counters.argtypes = [ctypes.c_int, ctypes.c_int, ctypes.c_int64, ctypes.c_int32, ctypes.c_void_p,
                                        ctypes.POINTER(ctypes.c_uint64), ctypes.c_int]
        L.rs_max_min_run_len.restype = ctypes.c_int32
        L.rs_max_min_run_len.argtypes = [ctypes.c_int, ctypes.c_int]
        L.rs_load_bin.restype = ctypes.c_int
        L.rs_load_bin.argtypes = [ctypes.c_char_p, ctypes.POINTER(ctypes.c_int64), ctypes.c_void_p, ctypes.c_int64,
                                  ctypes.c_void_p]
        L.rs_corank.restype = ctypes.c_int
        L.rs_corank.argtypes = [ctypes.c_int, ctypes.POINTER(RsShard), ctypes.c_int, ctypes.POINTER(ctypes.c_int64),
                                ctypes.c_int, ctypes.POINTER(ctypes.c_int64), ctypes.c_void_p, ctypes.c_size_t,
                                ctypes.c_void_p]
        L.rs_kway_workspace_bytes.restype = ctypes.c_size_t
        L.rs_kway_workspace_bytes.argtypes = [ctypes.c_int, ctypes.c_int, ctypes.POINTER(RsShard), ctypes.c_int]
        L.rs_kway_merge.restype = ctypes.c_int
        L.rs_kway_merge.argtypes = [ctypes.c_int, ctypes.c_int, ctypes.POINTER(RsShard), ctypes.c_int, ctypes.c_void_p,
                                    ctypes.c_void_p, ctypes.c_void_p, ctypes.c_size_t, ctypes.c_void_p]
        L.rs_corank_rank.restype = ctypes.c_int
        L.rs_corank_rank.argtypes = [ctypes.c_int, ctypes.POINTER(RsShard), ctypes.c_int, ctypes.c_void_p,
                                     ctypes.c_int, ctypes.c_void_p, ctypes.c_void_p]
        L.rs_kway_split_workspace_bytes.restype = ctypes.c_size_t
        L.rs_kway_split_workspace_bytes.argtypes = [ctypes.c_int, ctypes.c_int, ctypes.c_int, ctypes.c_int64]
        L.rs_merge_runs_workspace_bytes.restype = ctypes.c_size_t
        L.rs_merge_runs_workspace_bytes.argtypes = [ctypes.c_int, ctypes.c_int, ctypes.c_int64, ctypes.c_int]
        L.rs_merge_runs.restype = ctypes.c_int
        L.rs_merge_runs.argtypes = [ctypes.c_int, ctypes.c_void_p, ctypes.c_int, ctypes.c_void_p, ctypes.c_int64,
                                    ctypes.POINTER(ctypes.c_int64), ctypes.c_int, ctypes.c_void_p, ctypes.c_size_t,
                                    ctypes.c_void_p]
        L.rs_kway_merge_split.restype = ctypes.c_int
        L.rs_kway_merge_split.argtypes = [ctypes.c_int, ctypes.c_int, ctypes.POINTER(RsShard), ctypes.c_int,
                                          ctypes.c_void_p, ctypes.c_int64, ctypes.c_void_p, ctypes.c_void_p,
                                          ctypes.c_void_p, ctypes.c_size_t, ctypes.c_void_p]
        L.rs_ipc_alloc.restype = ctypes.c_int
        L.rs_ipc_alloc.argtypes = [ctypes.c_size_t, ctypes.POINTER(ctypes.c_void_p), ctypes.c_void_p]
        L.rs_ipc_open.restype = ctypes.c_int
        L.rs_ipc_open.argtypes = [ctypes.c_void_p, ctypes.POINTER(ctypes.c_void_p)]
        L.rs_ipc_close.restype = ctypes.c_int
        L.rs_ipc_close.argtypes = [ctypes.c_void_p]
        L.rs_ipc_free.restype = ctypes.c_int
        L.rs_ipc_free.argtypes = [ctypes.c_void_p]
        L.rs_last_error.restype = ctypes.c_char_p
        L.rs_last_error.argtypes = []
        L.rs_version.restype = ctypes.c_int
        L.rs_version.argtypes = []
        _lib = L
    return _lib


def check(rc: int) -> None:
    """Map C status codes onto the reference's exception types."""
    if rc == RS_OK:
        return
    msg = lib().rs_last_error().decode(errors="replace")
    if rc == RS_EINVAL:
        raise ValueError(msg)
    if rc == RS_EINVARIANT:
        raise AssertionError(msg)
    if rc == RS_EIO:
        raise OSError(msg)
    if rc == RS_ENOMEM:
        raise MemoryError(msg)
    if rc == RS_EUNSUPPORTED:
        raise NotImplementedError(msg)
    raise RuntimeError(msg)
