"""Drop-in powersort / peeksort entry points backed by the B200 CUDA path.

Mirrors reference sorters.py (calling convention :3-8, SortConfig :63-87,
peeksort :146-361, node powers :368-423, powersort :430-519, SORTERS
:671-678).  The keys are sorted in place, the optional ``tags`` payload moves
identically, and a ``Metrics`` is returned (created if not passed, otherwise
accumulated into), with the reference's exact counter values.

Inputs: numpy arrays (staged through the GPU and written back in place) or
torch tensors (CUDA tensors are sorted in place on their device).  Keys of
int32/int64 are sorted natively; narrower integers are widened and unsigned
ones sign-flipped to an order-preserving signed type.  There is no CPU
fallback: without a CUDA device or the built library, calls raise.
"""
from __future__ import annotations

import ctypes
from dataclasses import dataclass
from typing import Optional

import numpy as np

from . import _lib
from .opttree import MergeLeaf, tree_from_depths
from .runcore import Metrics

__all__ = [
    "SortConfig",
    "peeksort",
    "powersort",
    "node_power_def",
    "node_power_bitwise",
    "SORTERS",
    "sort_async",
]

MERGE_KINDS = ("bitonic", "classic")


@dataclass(frozen=True)
class SortConfig:
    """Shared sorter knobs (reference sorters.py:63-87).

    min_run_len   runs shorter than this are extended by insertion sort
                  (powersort) or recursion bottoms out in insertion sort
                  (peeksort); 1 disables the cutoff entirely.
    merge_kind    "bitonic" (exactly m+n comparisons) or "classic"
                  (two-pointer, at most m+n-1).
    record_tree   record the merge tree into Metrics.merge_tree.
    alpha         growth ratio for the alpha-stack/alpha-merge rules.
    """

    min_run_len: int = 24
    merge_kind: str = "bitonic"
    record_tree: bool = False
    alpha: float = 2.0

    def __post_init__(self) -> None:
        if self.min_run_len < 1:
            raise ValueError("min_run_len must be >= 1")
        if self.merge_kind not in MERGE_KINDS:
            raise ValueError(f"merge_kind must be one of {MERGE_KINDS}")
        if not self.alpha > 1.0:
            raise ValueError("alpha must be > 1")


# ---------------------------------------------------------------------------
# Node powers (host integer functions; reference sorters.py:368-411)


def _validate_power_args(s1: int, e1: int, s2: int, e2: int, n: int) -> None:
    if not (1 <= s1 <= e1 < s2 <= e2 <= n):
        raise ValueError(
            f"invalid run positions: need 1 <= s1 <= e1 < s2 <= e2 <= n, "
            f"got ({s1}, {e1}, {s2}, {e2}, {n})"
        )


def node_power_def(s1: int, e1: int, s2: int, e2: int, n: int) -> int:
    """Smallest l >= 1 with the normalized run midpoints in different cells of
    the 2**-l grid (1-based runs, exact integers, any n)."""
    _validate_power_args(s1, e1, s2, e2, n)
    a2 = s1 + e1 - 1  # 2n * midpoint of run 1 (1-based)
    b2 = s2 + e2 - 1
    two_n = 2 * n
    level = 1
    while (a2 << level) // two_n == (b2 << level) // two_n:
        level += 1
    return level


def node_power_bitwise(s1: int, e1: int, s2: int, e2: int, n: int) -> int:
    """Loop-free node power via 31-bit fixed point (n < 2**31 only)."""
    _validate_power_args(s1, e1, s2, e2, n)
    if n >= 1 << 31:
        raise ValueError("bitwise node power supports n < 2**31 only")
    afix = ((s1 + e1 - 1) << 31) // (2 * n)
    bfix = ((s2 + e2 - 1) << 31) // (2 * n)
    return 32 - (afix ^ bfix).bit_length()


# ---------------------------------------------------------------------------
# Staging


def _torch():
    import torch

    if not torch.cuda.is_available():
        raise RuntimeError("no CUDA device visible: the B200 sort path has no CPU fallback")
    return torch


_SIGNED = {np.dtype(np.int32): _lib.RS_KEY_I32, np.dtype(np.int64): _lib.RS_KEY_I64}


class _Staged:
    """A contiguous CUDA int32/int64 view of the caller's keys or tags on
    device `dev`, plus the write-back that lands the result in the caller's
    object (numpy array, CPU tensor, or a CUDA tensor that could not be
    sorted in place)."""

    def __init__(self, obj, is_keys: bool, dev, stream):
        torch = _torch()
        self.obj = obj
        self.flip = None
        self.host_out = None
        self.zero_signs = None
        self.orig_dtype = None
        if isinstance(obj, torch.Tensor):
            self.is_torch = True
            if obj.dim() != 1:
                raise ValueError("expected a one-dimensional tensor")
            npdt = np.dtype(str(obj.dtype).replace("torch.", "")) if obj.dtype != torch.bool else np.dtype(bool)
        else:
            self.is_torch = False
            arr = np.asarray(obj)
            if arr.ndim != 1:
                raise ValueError("expected a one-dimensional array")
            npdt = arr.dtype
        self.n = int(obj.shape[0]) if hasattr(obj, "shape") else len(obj)
        if is_keys:
            self.kind, self.code = self._key_plan(npdt)
        else:
            if npdt.itemsize not in (4, 8):
                raise NotImplementedError("tags must have a 4- or 8-byte dtype")
            self.kind, self.code = "raw", npdt.itemsize
        self.on_host = not (self.is_torch and obj.device.type == "cuda")
        if self.is_torch:
            t = obj
            if t.device.type != "cuda":
                d = t.to(dev, non_blocking=t.is_pinned())
            elif not t.is_contiguous():
                d = t.contiguous()
            else:
                d = t
        else:
            arr = np.ascontiguousarray(np.asarray(obj))
            d = torch.from_numpy(arr).to(dev)
        self.dev_t = self._to_work(d)
        self.stream = stream

    def _key_plan(self, npdt):
        if npdt in _SIGNED:
            return "native", _SIGNED[npdt]
        if npdt in (np.dtype(np.int8), np.dtype(np.int16), np.dtype(np.uint8), np.dtype(np.uint16),
                    np.dtype(bool)):
            return "widen", _lib.RS_KEY_I32
        if npdt == np.dtype(np.uint32):
            return "flip32", _lib.RS_KEY_I32
        if npdt == np.dtype(np.uint64):
            return "flip64", _lib.RS_KEY_I64
        if npdt in (np.dtype(np.float16), np.dtype(np.float32)):
            return "float32", _lib.RS_KEY_I32
        if npdt == np.dtype(np.float64):
            return "float64", _lib.RS_KEY_I64
        raise NotImplementedError(f"keys of dtype {npdt} are not supported on the device path "
                                  "(integers and floats only)")

    # Floating-point keys sort as the order-preserving integers of their bit
    # patterns (i ^ ((i >> 63) & 0x7f..f): negative values reversed below the
    # non-negative ones), which compare exactly like the reference's float
    # comparisons (sorters.py / runcore.py use <= and <) for every pair except
    # -0.0 vs +0.0, equal as floats: both zeros map to key 0, so the stable
    # sort keeps all zeros in their input order, and the output's zero block
    # gets back the input zeros' signs in that same order.  NaN keys, which
    # the reference's comparisons do not order, are rejected.
    def _float_to_key(self, d):
        torch = _torch()
        if self.kind == "float32" and d.dtype != torch.float32:
            self.orig_dtype = d.dtype
            d = d.to(torch.float32)
        if bool(torch.isnan(d).any().item()):
            raise NotImplementedError("NaN keys are not supported: the reference's comparisons do not order them")
        zero = d == 0
        self.zero_signs = torch.signbit(d[zero]) if bool(zero.any().item()) else None
        it, bits, mask = (torch.int32, 31, 0x7fffffff) if self.kind == "float32" else \
            (torch.int64, 63, 0x7fffffffffffffff)
        i = torch.where(zero, torch.zeros_like(d), d).view(it)
        return i ^ ((i >> bits) & mask)

    def _key_to_float(self, k):
        torch = _torch()
        it, ft, bits, mask = (torch.int32, torch.float32, 31, 0x7fffffff) if self.kind == "float32" else \
            (torch.int64, torch.float64, 63, 0x7fffffffffffffff)
        f = (k ^ ((k >> bits) & mask)).view(ft)
        if self.zero_signs is not None:
            zs = self.zero_signs
            f = f.clone()
            f[f == 0] = torch.where(zs, torch.full_like(zs, -0.0, dtype=ft), torch.full_like(zs, 0.0, dtype=ft))
        if getattr(self, "orig_dtype", None) is not None:
            f = f.to(self.orig_dtype)
        return f

    def _to_work(self, d):
        torch = _torch()
        if self.kind == "raw":
            if d.element_size() == 4 and d.dtype != torch.int32:
                d = d.view(torch.int32)
            elif d.element_size() == 8 and d.dtype != torch.int64:
                d = d.view(torch.int64)
            return d
        if self.kind == "native":
            return d
        if self.kind == "widen":
            self.orig_dtype = d.dtype
            return d.to(torch.int32)
        if self.kind == "flip32":
            return d.view(torch.int32) ^ torch.tensor(-(1 << 31), dtype=torch.int32, device=d.device)
        if self.kind == "flip64":
            return d.view(torch.int64) ^ torch.tensor(-(1 << 63), dtype=torch.int64, device=d.device)
        if self.kind in ("float32", "float64"):
            return self._float_to_key(d)
        raise AssertionError(self.kind)

    def _result(self):
        torch = _torch()
        d = self.dev_t
        if self.kind == "widen":
            d = d.to(self.orig_dtype)
        elif self.kind == "flip32":
            d = (d ^ torch.tensor(-(1 << 31), dtype=torch.int32, device=d.device)).view(torch.uint32)
        elif self.kind == "flip64":
            d = (d ^ torch.tensor(-(1 << 63), dtype=torch.int64, device=d.device)).view(torch.uint64)
        elif self.kind in ("float32", "float64"):
            d = self._key_to_float(d)
        return d

    def finish_device(self):
        """Device-side write-back (CUDA tensors the sort could not run in place on)."""
        if self.on_host:
            return
        d = self._result()
        t = self.obj
        if d.data_ptr() != t.data_ptr() or d.dtype != t.dtype:
            if d.dtype != t.dtype:
                d = d.view(t.dtype) if d.element_size() == t.element_size() else d.to(t.dtype)
            t.copy_(d)

    def queue_host_copy(self):
        """Queue the device-to-host copy of the result into a staging buffer the
        caller does not see (numpy inputs); nothing for other inputs."""
        if not self.on_host or self.is_torch:
            return
        torch = _torch()
        d = self._result()
        self.host_out = torch.empty(d.shape, dtype=d.dtype, pin_memory=True)
        self.host_out.copy_(d, non_blocking=True)

    def finish_host(self):
        """Host write-back, called once the device reported no error: numpy
        arrays get the staged result, CPU tensors a copy straight into them."""
        if not self.on_host:
            return
        if self.is_torch:
            d = self._result()
            t = self.obj
            if d.dtype != t.dtype:
                d = d.view(t.dtype) if d.element_size() == t.element_size() else d.to(t.dtype)
            t.copy_(d, non_blocking=t.is_pinned())
            return
        host = self.host_out.numpy()
        arr = self.obj
        if host.dtype != arr.dtype:
            host = host.view(arr.dtype) if host.itemsize == arr.dtype.itemsize else host.astype(arr.dtype)
        arr[...] = host


def _target_device(a, tags):
    """The device the sort runs on: the keys' CUDA device, else the current one.
    CUDA tags must live on that same device."""
    torch = _torch()
    if isinstance(a, torch.Tensor) and a.device.type == "cuda":
        dev = a.device
    else:
        dev = torch.device("cuda", torch.cuda.current_device())
    if isinstance(tags, torch.Tensor) and tags.device.type == "cuda" and tags.device != dev:
        raise ValueError(f"tags are on {tags.device} but the keys sort on {dev}")
    return dev


def _host_native(a, tags) -> bool:
    """numpy keys/tags the host staging engine (rs_sort_host_ex) takes as they are."""
    if not isinstance(a, np.ndarray) or a.dtype not in _SIGNED or a.ndim != 1 or not a.flags.c_contiguous \
            or not a.flags.writeable:
        return False
    if tags is None:
        return True
    return isinstance(tags, np.ndarray) and tags.ndim == 1 and tags.flags.c_contiguous and \
        tags.flags.writeable and tags.dtype.itemsize in (4, 8) and len(tags) == len(a)


def _accumulate(algo: int, metrics: Metrics, out) -> None:
    metrics.merge_cost += int(out.merge_cost)
    metrics.comparisons += int(out.comparisons)
    if algo == _lib.RS_ALGO_PEEKSORT:
        metrics.runs_detected = int(out.runs_detected)  # sorters.py:358 assigns
    else:
        metrics.runs_detected += int(out.runs_detected)  # sorters.py:464 accumulates
        if int(out.max_stack_height) > metrics.max_stack_height:
            metrics.max_stack_height = int(out.max_stack_height)


def _host_sort(algo: int, a: np.ndarray, cfg: SortConfig, metrics: Metrics, tags) -> Metrics:
    """numpy in, numpy out through the library's host staging engine: chunked,
    multi-threaded copies through pinned slots overlapped with the DMAs, and the
    caller's arrays written only after the device reported success."""
    L = _lib.lib()
    out = _lib.RsMetrics()
    kind = _lib.RS_MERGE_CLASSIC if cfg.merge_kind == "classic" else _lib.RS_MERGE_BITONIC
    _lib.check(L.rs_sort_host_ex(algo, _SIGNED[a.dtype], a.ctypes.data, tags.dtype.itemsize if tags is not None else 0,
                                 tags.ctypes.data if tags is not None else None, len(a), int(cfg.min_run_len), kind,
                                 float(cfg.alpha), ctypes.byref(out), None))
    _accumulate(algo, metrics, out)
    return metrics


def _device_sort(algo: int, a, cfg: SortConfig, metrics: Metrics, tags) -> Metrics:
    torch = _torch()
    dev = _target_device(a, tags)
    with torch.cuda.device(dev):
        if not cfg.record_tree and _host_native(a, tags):
            return _host_sort(algo, a, cfg, metrics, tags)
        return _device_sort_on(algo, a, cfg, metrics, tags, dev)


def _device_sort_on(algo: int, a, cfg: SortConfig, metrics: Metrics, tags, dev) -> Metrics:
    L = _lib.lib()
    torch = _torch()
    stream = torch.cuda.current_stream(dev)
    keys = _Staged(a, True, dev, stream)
    n = keys.n
    tg = None
    if tags is not None:
        tg = _Staged(tags, False, dev, stream)
        if tg.n != n:
            raise ValueError("tags must have the same length as the keys")
    w = int(cfg.min_run_len)
    kind = _lib.RS_MERGE_CLASSIC if cfg.merge_kind == "classic" else _lib.RS_MERGE_BITONIC
    tb = tg.code if tg is not None else 0
    out = _lib.RsMetrics()
    staged = [keys] + ([tg] if tg is not None else [])
    # The sort is enqueued without a host sync; numpy results are copied back
    # into a staging buffer queued behind it, and one synchronizing Metrics
    # fetch follows.  Only when the device reported no invariant failure is
    # the caller's host object overwritten (CUDA tensors are sorted in place).
    # Peeksort runs with its compact replay workspace first; if the recursion
    # outgrows it the device restores the input and reports RS_ECAPACITY, and
    # the sort runs again with the worst-case workspace (RS_ALGO_FULL_WS).
    algo_ws = algo
    while True:
        ws_bytes = L.rs_workspace_bytes(algo_ws, keys.code, tb, n, w)
        ws = torch.empty(ws_bytes, dtype=torch.uint8, device=dev)
        rc = L.rs_sort_ex(algo_ws, keys.code, keys.dev_t.data_ptr(), tb,
                          tg.dev_t.data_ptr() if tg is not None else None, n, w, kind, float(cfg.alpha),
                          ws.data_ptr(), ws_bytes, stream.cuda_stream, None, None)
        _lib.check(rc)
        for s_ in staged:
            s_.finish_device()
            s_.queue_host_copy()
        rc = L.rs_fetch_metrics(algo_ws, keys.code, tb, n, w, ws.data_ptr(), stream.cuda_stream, ctypes.byref(out))
        if rc == _lib.RS_ECAPACITY and not (algo_ws & _lib.RS_ALGO_FULL_WS):
            algo_ws |= _lib.RS_ALGO_FULL_WS
            del ws
            continue
        _lib.check(rc)
        break
    tree = None
    if cfg.record_tree and algo in (_lib.RS_ALGO_POWERSORT, _lib.RS_ALGO_PEEKSORT):
        # host arrays sized by the leaf count r (not n): query r, then export
        probe = _lib.RsTree(0, 0, None, None, None)
        _lib.check(L.rs_export_tree(algo_ws, keys.code, tb, n, w, ws.data_ptr(), stream.cuda_stream,
                                    ctypes.byref(probe)))
        r = int(probe.n_leaves)
        bufs = (np.zeros(r, dtype=np.int64), np.zeros(r, dtype=np.uint8), np.zeros(r, dtype=np.uint8))
        tree = _lib.RsTree(r, 0, bufs[0].ctypes.data, bufs[1].ctypes.data, bufs[2].ctypes.data)
        _lib.check(L.rs_export_tree(algo_ws, keys.code, tb, n, w, ws.data_ptr(), stream.cuda_stream,
                                    ctypes.byref(tree)))
    for s_ in staged:
        s_.finish_host()
    if any(s_.on_host for s_ in staged):
        stream.synchronize()  # non-blocking copies into pinned CPU tensors have landed
    _accumulate(algo, metrics, out)
    if tree is not None:
        r = int(tree.n_leaves)
        lens = bufs[0][:r]
        depths = bufs[2][: r - 1]
        powers = bufs[1][: r - 1] if algo == _lib.RS_ALGO_POWERSORT else None
        metrics.merge_tree = tree_from_depths(lens, depths, powers)
    return metrics


class PendingSort:
    """A device sort enqueued by ``sort_async``; ``metrics()`` synchronizes the
    stream and returns the call's Metrics (the reference's counters)."""

    def __init__(self, algo, code, tb, n, w, ws, stream):
        self._args = (algo, code, tb, n, w)
        self.workspace = ws
        self.stream = stream

    def metrics(self) -> Metrics:
        algo, code, tb, n, w = self._args
        out = _lib.RsMetrics()
        _lib.check(_lib.lib().rs_fetch_metrics(algo, code, tb, n, w, self.workspace.data_ptr(),
                                               self.stream.cuda_stream, ctypes.byref(out)))
        m = Metrics()
        _accumulate(algo & ~_lib.RS_ALGO_FULL_WS, m, out)
        return m


def sort_async(keys, tags=None, cfg: Optional[SortConfig] = None, algo: str = "powersort",
               workspace=None) -> Optional[PendingSort]:
    """Enqueue powersort / peeksort of contiguous int32/int64 CUDA tensors (tags
    4 or 8 bytes) on the current stream, in place, without any host
    synchronisation (the building block of the sharded sort: the caller's
    next stream work follows the sort).  ``workspace`` (a uint8 CUDA tensor)
    is reused when large enough.  Returns None for n <= 1."""
    torch = _torch()
    L = _lib.lib()
    cfg = cfg or SortConfig()
    # no host round trip here, so no retry: peeksort takes its worst-case workspace
    code = {"powersort": _lib.RS_ALGO_POWERSORT, "peeksort": _lib.RS_ALGO_PEEKSORT | _lib.RS_ALGO_FULL_WS}[algo]
    n = int(keys.numel())
    if n <= 1:
        return None
    if keys.device.type != "cuda" or not keys.is_contiguous() or keys.dtype not in (torch.int32, torch.int64):
        raise NotImplementedError("sort_async takes contiguous int32/int64 CUDA tensors")
    if tags is not None and (tags.device != keys.device or not tags.is_contiguous() or
                             tags.element_size() not in (4, 8) or tags.numel() != n):
        raise ValueError("tags must be a contiguous 4/8-byte CUDA tensor of the keys' length and device")
    kc = _lib.RS_KEY_I32 if keys.dtype == torch.int32 else _lib.RS_KEY_I64
    tb = tags.element_size() if tags is not None else 0
    w = int(cfg.min_run_len)
    need = L.rs_workspace_bytes(code, kc, tb, n, w)
    if workspace is None or workspace.numel() < need:
        workspace = torch.empty(need, dtype=torch.uint8, device=keys.device)
    stream = torch.cuda.current_stream(keys.device)
    kind = _lib.RS_MERGE_CLASSIC if cfg.merge_kind == "classic" else _lib.RS_MERGE_BITONIC
    _lib.check(L.rs_sort_ex(code, kc, keys.data_ptr(), tb, tags.data_ptr() if tags is not None else None, n, w,
                            kind, float(cfg.alpha), workspace.data_ptr(), workspace.numel(), stream.cuda_stream,
                            None, None))
    return PendingSort(code, kc, tb, n, w, workspace, stream)


def _entry(algo, a, cfg, metrics, tags):
    cfg = cfg or SortConfig()
    metrics = metrics or Metrics()
    n = len(a)
    if n <= 1:
        if algo in (_lib.RS_ALGO_TOP_DOWN, _lib.RS_ALGO_BOTTOM_UP):  # sorters.py:533-535, :564-566
            return metrics
        metrics.runs_detected = n  # sorters.py:445-450 / :168-173 / :588-590
        if cfg.record_tree and n == 1 and algo in (_lib.RS_ALGO_POWERSORT, _lib.RS_ALGO_PEEKSORT):
            metrics.merge_tree = MergeLeaf(0, 1)
        return metrics
    return _device_sort(algo, a, cfg, metrics, tags)


def powersort(a, cfg: Optional[SortConfig] = None, metrics: Optional[Metrics] = None,
              tags=None) -> Metrics:
    """One-pass stack-based natural mergesort driven by node powers
    (reference sorters.py:430-519), executed on the GPU."""
    return _entry(_lib.RS_ALGO_POWERSORT, a, cfg, metrics, tags)


def peeksort(a, cfg: Optional[SortConfig] = None, metrics: Optional[Metrics] = None,
             tags=None) -> Metrics:
    """Top-down natural mergesort splitting at the run boundary closest to the
    midpoint (reference sorters.py:146-361), executed on the GPU."""
    return _entry(_lib.RS_ALGO_PEEKSORT, a, cfg, metrics, tags)


def top_down_mergesort(a, cfg: Optional[SortConfig] = None, metrics: Optional[Metrics] = None,
                       tags=None) -> Metrics:
    """Plain top-down mergesort: midpoint split, insertion sort below the
    cutoff, one comparison to skip an in-order merge (reference
    sorters.py:524-552), executed on the GPU."""
    return _entry(_lib.RS_ALGO_TOP_DOWN, a, cfg, metrics, tags)


def bottom_up_mergesort(a, cfg: Optional[SortConfig] = None, metrics: Optional[Metrics] = None,
                        tags=None) -> Metrics:
    """Plain bottom-up mergesort: insertion-sorted chunks of min_run_len, merge
    passes of doubling width with the same skip check (reference
    sorters.py:555-581), executed on the GPU."""
    return _entry(_lib.RS_ALGO_BOTTOM_UP, a, cfg, metrics, tags)


def alpha_stack_sort(a, cfg: Optional[SortConfig] = None, metrics: Optional[Metrics] = None,
                     tags=None) -> Metrics:
    """Merge the topmost two runs until stack lengths grow by factor alpha
    (reference sorters.py:638-647), executed on the GPU."""
    return _entry(_lib.RS_ALGO_ALPHA_STACK, a, cfg, metrics, tags)


def alpha_merge_sort(a, cfg: Optional[SortConfig] = None, metrics: Optional[Metrics] = None,
                     tags=None) -> Metrics:
    """alpha-stack rule plus pre-merging the stack top up to the new run's
    length before pushing (reference sorters.py:650-660), executed on the GPU."""
    return _entry(_lib.RS_ALGO_ALPHA_MERGE, a, cfg, metrics, tags)


SORTERS = {
    "peeksort": peeksort,
    "powersort": powersort,
    "top-down": top_down_mergesort,
    "bottom-up": bottom_up_mergesort,
    "alpha-stack": alpha_stack_sort,
    "alpha-merge": alpha_merge_sort,
}
