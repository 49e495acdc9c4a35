"""ctypes wrapper of the C oracle -- TEST INFRASTRUCTURE ONLY.

Only tests/, ``__graft_entry__.smoke()`` and bench.py's CPU-baseline legs may
import this module.  It wraps ``runsort_oracle.c``, a plain-C restatement of
the reference's powersort/peeksort (reference ``sorters.py:146-361`` and
``:430-519``), pinned against the reference through ``tests/golden``.

All calls sort numpy arrays in place on the CPU, exactly like the reference
entry points (``sorters.py:430-435``).
"""

from __future__ import annotations

import ctypes
import os
import subprocess
from dataclasses import dataclass, field
from typing import Optional

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_LIB_PATH = os.path.join(_HERE, "librunsort_oracle.so")
_lib = None


class OrcMetrics(ctypes.Structure):
    _fields_ = [
        ("merge_cost", ctypes.c_uint64),
        ("comparisons", ctypes.c_uint64),
        ("runs_detected", ctypes.c_uint64),
        ("max_stack_height", ctypes.c_uint64),
    ]


@dataclass
class OracleResult:
    merge_cost: int
    comparisons: int
    runs_detected: int
    max_stack_height: int
    leaf_starts: Optional[np.ndarray] = None  # powersort: r entries
    powers: Optional[np.ndarray] = None  # powersort: r-1 entries
    merges: Optional[np.ndarray] = None  # peeksort: (m, 4) = (l, mid, r, depth)
    extra: dict = field(default_factory=dict)

    def metrics_tuple(self):
        return (self.merge_cost, self.comparisons, self.runs_detected, self.max_stack_height)


def build(force: bool = False) -> str:
    """Compile the oracle with the committed Makefile (gcc)."""
    src = os.path.join(_HERE, "runsort_oracle.c")
    if force or not os.path.exists(_LIB_PATH) or os.path.getmtime(_LIB_PATH) < os.path.getmtime(src):
        subprocess.run(["make", "-s", "-C", _HERE], check=True)
    return _LIB_PATH


def lib():
    global _lib
    if _lib is None:
        build()
        L = ctypes.CDLL(_LIB_PATH)
        L.orc_powersort.restype = ctypes.c_int64
        L.orc_powersort.argtypes = [
            ctypes.c_int, ctypes.c_void_p, ctypes.c_int, ctypes.c_void_p, ctypes.c_int64,
            ctypes.c_int32, ctypes.c_int32, ctypes.POINTER(OrcMetrics),
            ctypes.c_void_p, ctypes.c_void_p, ctypes.c_int64,
        ]
        L.orc_peeksort.restype = ctypes.c_int64
        L.orc_peeksort.argtypes = [
            ctypes.c_int, ctypes.c_void_p, ctypes.c_int, ctypes.c_void_p, ctypes.c_int64,
            ctypes.c_int32, ctypes.c_int32, ctypes.POINTER(OrcMetrics),
            ctypes.c_void_p, ctypes.c_int64,
        ]
        L.orc_baseline.restype = ctypes.c_int64
        L.orc_baseline.argtypes = [
            ctypes.c_int, ctypes.c_int, ctypes.c_void_p, ctypes.c_int, ctypes.c_void_p, ctypes.c_int64,
            ctypes.c_int32, ctypes.c_int32, ctypes.c_double, ctypes.POINTER(OrcMetrics),
        ]
        L.orc_node_power_def.restype = ctypes.c_int
        L.orc_node_power_def.argtypes = [ctypes.c_int64] * 5
        L.orc_node_power0.restype = ctypes.c_int
        L.orc_node_power0.argtypes = [ctypes.c_int64] * 5
        _lib = L
    return _lib


def _key_kind(a: np.ndarray) -> int:
    if a.dtype == np.int32:
        return 0
    if a.dtype == np.int64:
        return 1
    raise TypeError(f"oracle supports int32/int64 keys, got {a.dtype}")


def _check(a, tags):
    if not (a.flags.c_contiguous and a.flags.writeable):
        raise ValueError("oracle needs a writable C-contiguous array")
    if tags is not None:
        if len(tags) != len(a) or tags.itemsize not in (4, 8) or not tags.flags.c_contiguous:
            raise ValueError("tags must be a contiguous 4/8-byte array of len(a)")


def powersort(a: np.ndarray, min_run_len: int = 24, merge_kind: str = "bitonic",
              tags: Optional[np.ndarray] = None, want_tree: bool = False) -> OracleResult:
    """Reference powersort (sorters.py:430-519) on the CPU, in place."""
    _check(a, tags)
    n = len(a)
    m = OrcMetrics()
    cap = 0
    powers = starts = None
    if want_tree and n > 0:
        cap = n
        powers = np.zeros(max(n, 1), dtype=np.int32)
        starts = np.zeros(max(n, 1), dtype=np.int64)
    r = lib().orc_powersort(
        _key_kind(a), a.ctypes.data, tags.itemsize if tags is not None else 0,
        tags.ctypes.data if tags is not None else None, n, int(min_run_len),
        1 if merge_kind == "classic" else 0, ctypes.byref(m),
        powers.ctypes.data if powers is not None else None,
        starts.ctypes.data if starts is not None else None, cap)
    if r < 0:
        raise AssertionError(f"oracle powersort invariant failure ({r})")
    res = OracleResult(m.merge_cost, m.comparisons, m.runs_detected, m.max_stack_height)
    if want_tree and n > 0:
        res.leaf_starts = starts[:r].copy()
        res.powers = powers[: max(r - 1, 0)].copy()
    return res


def peeksort(a: np.ndarray, min_run_len: int = 24, merge_kind: str = "bitonic",
             tags: Optional[np.ndarray] = None, want_tree: bool = False) -> OracleResult:
    """Reference peeksort (sorters.py:146-361) on the CPU, in place."""
    _check(a, tags)
    n = len(a)
    m = OrcMetrics()
    merges = None
    cap = 0
    if want_tree and n > 0:
        cap = n
        merges = np.zeros((max(n, 1), 4), dtype=np.int64)
    k = lib().orc_peeksort(
        _key_kind(a), a.ctypes.data, tags.itemsize if tags is not None else 0,
        tags.ctypes.data if tags is not None else None, n, int(min_run_len),
        1 if merge_kind == "classic" else 0, ctypes.byref(m),
        merges.ctypes.data if merges is not None else None, cap)
    res = OracleResult(m.merge_cost, m.comparisons, m.runs_detected, m.max_stack_height)
    if want_tree and n > 0:
        res.merges = merges[:k].copy()
    return res


BASELINES = {"top-down": 2, "bottom-up": 3, "alpha-stack": 4, "alpha-merge": 5}


def baseline(name: str, a: np.ndarray, min_run_len: int = 24, merge_kind: str = "bitonic",
             tags: Optional[np.ndarray] = None, alpha: float = 2.0) -> OracleResult:
    """Reference baseline sorters (sorters.py:524-660) on the CPU, in place."""
    _check(a, tags)
    m = OrcMetrics()
    r = lib().orc_baseline(BASELINES[name], _key_kind(a), a.ctypes.data, tags.itemsize if tags is not None else 0,
                           tags.ctypes.data if tags is not None else None, len(a), int(min_run_len),
                           1 if merge_kind == "classic" else 0, float(alpha), ctypes.byref(m))
    if r < 0:
        raise AssertionError(f"oracle baseline failure ({r})")
    return OracleResult(m.merge_cost, m.comparisons, m.runs_detected, m.max_stack_height)


def node_power_def(s1, e1, s2, e2, n) -> int:
    return int(lib().orc_node_power_def(s1, e1, s2, e2, n))


def node_power0(s1, e1, s2, e2, n) -> int:
    return int(lib().orc_node_power0(s1, e1, s2, e2, n))


def peek_tree_from_merges(n: int, merges: np.ndarray):
    """Nested-tuple tree shape from peeksort's post-order merge list.

    Leaves are ('L', length); nodes are ('N', left, right).  Used to compare
    against the reference's recorded MergeNode trees (opttree.py:60-75).
    """
    if n == 0:
        return None
    spans = {}
    for l, mid, r, _d in merges.tolist():
        spans[(l, r)] = mid

    def build(l, r):
        mid = spans.get((l, r))
        if mid is None:
            return ("L", r - l + 1)
        return ("N", build(l, mid - 1), build(mid, r))

    return build(0, n - 1)


def power_tree_from_powers(leaf_lengths, powers):
    """Nested-tuple min-Cartesian tree of the powers (opttree.py:308-336)."""
    r = len(leaf_lengths)
    if r == 1:
        return ("L", int(leaf_lengths[0]))
    m = len(powers)
    left = [0] * (m + 1)
    right = [0] * (m + 1)
    stack = []
    for j in range(1, m + 1):
        last = 0
        while stack and powers[stack[-1] - 1] > powers[j - 1]:
            last = stack.pop()
        left[j] = last
        if stack:
            right[stack[-1]] = j
        stack.append(j)

    def freeze(j):
        lt = freeze(left[j]) if left[j] else ("L", int(leaf_lengths[j - 1]))
        rt = freeze(right[j]) if right[j] else ("L", int(leaf_lengths[j]))
        return ("N", lt, rt)

    return freeze(stack[0])
