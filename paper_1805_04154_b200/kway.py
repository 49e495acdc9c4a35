"""Device-side pieces of the cross-GPU merge (C ABI: rs_corank, rs_kway_merge,
rs_ipc_*; kernels in csrc/rs_kway.cuh).

A *shard* is a sorted device array given by a pointer (local, or a peer GPU's
buffer mapped over NVLink by CUDA IPC) and a range [lo, hi).  The global order
is (key, shard index, position) -- the stable order of the shards'
concatenation, as the reference's left-wins merges define it (reference
runcore.py:262-263).
"""
from __future__ import annotations

import ctypes
from typing import List, Optional, Sequence, Tuple

import numpy as np

from . import _lib

MAX_SHARDS = 8
_TYPESTR = {4: "<i4", 8: "<i8"}


def _torch():
    import torch

    return torch


def key_code(dtype) -> int:
    torch = _torch()
    if dtype == torch.int32:
        return _lib.RS_KEY_I32
    if dtype == torch.int64:
        return _lib.RS_KEY_I64
    raise NotImplementedError(f"keys must be int32 or int64, got {dtype}")


class Shard:
    """One sorted input of a k-way merge: device pointers plus a range."""

    def __init__(self, keys_ptr: int, tags_ptr: Optional[int], lo: int, hi: int):
        self.keys_ptr, self.tags_ptr, self.lo, self.hi = int(keys_ptr), tags_ptr, int(lo), int(hi)

    @classmethod
    def of(cls, keys, tags=None, lo: int = 0, hi: Optional[int] = None) -> "Shard":
        return cls(keys.data_ptr(), tags.data_ptr() if tags is not None else None, lo,
                   int(keys.numel()) if hi is None else hi)

    def with_range(self, lo: int, hi: int) -> "Shard":
        return Shard(self.keys_ptr, self.tags_ptr, lo, hi)


def _shard_array(shards: Sequence[Shard]):
    if not 1 <= len(shards) <= MAX_SHARDS:
        raise ValueError(f"between 1 and {MAX_SHARDS} shards")
    arr = (_lib.RsShard * len(shards))()
    for i, s in enumerate(shards):
        arr[i].keys = s.keys_ptr
        arr[i].tags = s.tags_ptr
        arr[i].lo = s.lo
        arr[i].hi = s.hi
    return arr


def corank(shards: Sequence[Shard], targets: Sequence[int], key_dtype, device=None, stream=None) -> np.ndarray:
    """Split vectors (len(targets), W): absolute positions c[b][i] such that the
    first targets[b] elements of the global order are shard i's [lo_i, c[b][i])."""
    torch = _torch()
    L = _lib.lib()
    W = len(shards)
    T = len(targets)
    out = np.zeros((max(T, 1), W), dtype=np.int64)
    if T == 0:
        return out[:0]
    tg = np.ascontiguousarray(np.asarray(targets, dtype=np.int64))
    dev = device or torch.device("cuda", torch.cuda.current_device())
    ws = torch.empty(T * 8 * (1 + W) + 1024, dtype=torch.uint8, device=dev)
    st = stream or torch.cuda.current_stream(dev)
    arr = _shard_array(shards)
    _lib.check(L.rs_corank(key_code(key_dtype), arr, W, tg.ctypes.data_as(ctypes.POINTER(ctypes.c_int64)), T,
                           out.ctypes.data_as(ctypes.POINTER(ctypes.c_int64)), ws.data_ptr(), ws.numel(),
                           st.cuda_stream))
    return out[:T]


def kway_merge(shards: Sequence[Shard], out_keys, out_tags=None, stream=None, workspace=None):
    """Stable W-way merge of the shard ranges into out_keys (+ out_tags); async."""
    torch = _torch()
    L = _lib.lib()
    W = len(shards)
    tb = out_tags.element_size() if out_tags is not None else 0
    kc = key_code(out_keys.dtype)
    arr = _shard_array(shards)
    need = L.rs_kway_workspace_bytes(kc, tb, arr, W)
    if need == 0:
        _lib.check(_lib.RS_EINVAL)
    if workspace is None or workspace.numel() < need:
        workspace = torch.empty(need, dtype=torch.uint8, device=out_keys.device)
    st = stream or torch.cuda.current_stream(out_keys.device)
    _lib.check(L.rs_kway_merge(kc, tb, arr, W, out_keys.data_ptr(),
                               out_tags.data_ptr() if out_tags is not None else None,
                               workspace.data_ptr(), workspace.numel(), st.cuda_stream))
    return workspace


def corank_rank(shards: Sequence[Shard], dlens, rank: int, dsplit, key_dtype, stream=None) -> None:
    """Device-only co-rank of rank `rank`'s output range: shard i is
    [0, dlens[i]) (device int64 tensor of W lengths); dsplit (device int64,
    2 x W) receives the start and end split vectors.  Async."""
    torch = _torch()
    L = _lib.lib()
    st = stream or torch.cuda.current_stream(dsplit.device)
    arr = _shard_array(shards)
    _lib.check(L.rs_corank_rank(key_code(key_dtype), arr, len(shards), dlens.data_ptr(), int(rank),
                                dsplit.data_ptr(), st.cuda_stream))


def kway_merge_split(shards: Sequence[Shard], dsplit, out_len: int, out_keys, out_tags=None, stream=None,
                     workspace=None):
    """W-way merge of the ranges in dsplit (device, 2 x W); async."""
    torch = _torch()
    L = _lib.lib()
    W = len(shards)
    tb = out_tags.element_size() if out_tags is not None else 0
    kc = key_code(out_keys.dtype)
    need = L.rs_kway_split_workspace_bytes(kc, tb, W, int(out_len))
    if workspace is None or workspace.numel() < need:
        workspace = torch.empty(max(need, 256), dtype=torch.uint8, device=out_keys.device)
    st = stream or torch.cuda.current_stream(out_keys.device)
    arr = _shard_array(shards)
    _lib.check(L.rs_kway_merge_split(kc, tb, arr, W, dsplit.data_ptr(), int(out_len), out_keys.data_ptr(),
                                     out_tags.data_ptr() if out_tags is not None else None,
                                     workspace.data_ptr(), workspace.numel(), st.cuda_stream))
    return workspace


def merge_runs(keys, tags, run_lengths: Sequence[int], stream=None, workspace=None):
    """Merge the sorted runs stored back to back in `keys` (and `tags`) in place
    into one sorted run, ties to the earlier run (rs_merge_runs: the executor
    along a balanced binary tree, log2 W passes); async.  Returns the workspace."""
    torch = _torch()
    L = _lib.lib()
    n = int(keys.numel())
    starts = np.concatenate([[0], np.cumsum(np.asarray(run_lengths, dtype=np.int64))]).astype(np.int64)
    if int(starts[-1]) != n:
        raise ValueError("run lengths must add up to the array length")
    W = len(run_lengths)
    tb = tags.element_size() if tags is not None else 0
    kc = key_code(keys.dtype)
    need = L.rs_merge_runs_workspace_bytes(kc, tb, n, W)
    if workspace is None or workspace.numel() < need:
        workspace = torch.empty(max(need, 256), dtype=torch.uint8, device=keys.device)
    st = stream or torch.cuda.current_stream(keys.device)
    _lib.check(L.rs_merge_runs(kc, keys.data_ptr(), tb, tags.data_ptr() if tags is not None else None, n,
                               starts.ctypes.data_as(ctypes.POINTER(ctypes.c_int64)), W, workspace.data_ptr(),
                               workspace.numel(), st.cuda_stream))
    return workspace


# ------------------------------------------------------------------ IPC ----
class _CAI:
    def __init__(self, ptr: int, n: int, itemsize: int):
        self.__cuda_array_interface__ = {"shape": (n,), "typestr": _TYPESTR[itemsize], "data": (ptr, False),
                                         "version": 3}


def tensor_at(ptr: int, n: int, dtype, device):
    """A torch tensor viewing n elements of device memory at `ptr` (no ownership)."""
    torch = _torch()
    item = torch.empty(0, dtype=dtype).element_size()
    return torch.as_tensor(_CAI(ptr, n, item), device=device).view(dtype)


class IpcBuffer:
    """Device memory this process owns and peers can map (CUDA IPC)."""

    def __init__(self, nbytes: int):
        L = _lib.lib()
        self.nbytes = int(nbytes)
        self.ptr = ctypes.c_void_p()
        self.handle = ctypes.create_string_buffer(64)
        _lib.check(L.rs_ipc_alloc(self.nbytes, ctypes.byref(self.ptr), self.handle))

    @property
    def address(self) -> int:
        return int(self.ptr.value)

    def handle_bytes(self) -> bytes:
        return bytes(self.handle.raw)

    def free(self):
        if self.ptr.value:
            _lib.check(_lib.lib().rs_ipc_free(self.ptr))
            self.ptr = ctypes.c_void_p()


def ipc_open(handle: bytes) -> int:
    """Map a peer's IpcBuffer (its handle_bytes()) into this process."""
    ptr = ctypes.c_void_p()
    buf = ctypes.create_string_buffer(bytes(handle), 64)
    _lib.check(_lib.lib().rs_ipc_open(buf, ctypes.byref(ptr)))
    return int(ptr.value)


def ipc_close(ptr: int) -> None:
    _lib.check(_lib.lib().rs_ipc_close(ctypes.c_void_p(ptr)))
