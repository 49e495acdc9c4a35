"""Powersort Metrics from the run structure alone -- TEST INFRASTRUCTURE ONLY.

Only tests/ (and bench.py's parity leg) may import this module.  It restates
the reference's powersort driver (``sorters.py:430-519``) over a run
description instead of an array, for inputs too large for the element-by-element
oracle (BASELINE config 5: n = 2^31 int64, 16 GiB):

* leaves: ``detect`` (``sorters.py:462-470``) over ``find_run_right``
  (``runcore.py:137-159``): the natural run from ``start`` is the weakly
  increasing / strictly decreasing run, i.e. it ends at the first run-boundary
  position after ``start``; runs shorter than ``min_run_len`` are extended and
  insertion-sorted (``runcore.py:215-248``, comparisons
  ``sum_{t >= npre} g_t + [g_t < t]``);
* node powers: ``_node_power0`` (``sorters.py:414-423``) -- the 31-bit
  fixed-point form below 2^31 and the definitional loop ``node_power_def``
  (``sorters.py:376-392``) at and above 2^31, both restated here in exact
  Python integers;
* the power-indexed run stack (``sorters.py:455-516``) simulated slot by slot:
  every merge adds its span to ``merge_cost`` and (bitonic, ``runcore.py:299-301``)
  to ``comparisons``; ``max_stack_height`` is the peak slot occupancy.

The caller supplies the data through three small callbacks so the 16 GiB array
never leaves the device: the sorted list of run-boundary positions, the
ascending flag at given positions, and the original values of short windows.
Pinned: ``tests/test_oracle.py`` checks this module against the reference's
node-power tuples (``tests/golden``) and against the C oracle on random arrays.
"""
from __future__ import annotations

import bisect
from typing import Callable, Dict, List, Sequence

import numpy as np


def node_power_def(s1: int, e1: int, s2: int, e2: int, n: int) -> int:
    """sorters.py:376-392 (1-based runs, exact integers, any n)."""
    if not (1 <= s1 <= e1 < s2 <= e2 <= n):
        raise ValueError("invalid run positions")
    a2 = 2 * (s1 - 1) + (e1 - s1 + 1)
    b2 = 2 * (s2 - 1) + (e2 - s2 + 1)
    two_n = 2 * n
    level = 1
    while (a2 << level) // two_n == (b2 << level) // two_n:
        level += 1
    return level


def node_power0(s1: int, e1: int, s2: int, e2: int, n: int) -> int:
    """sorters.py:414-423 (0-based adjacent runs)."""
    if n < 1 << 31:
        l = s1 + s2
        r = s2 + e2 + 1
        two_n = 2 * n
        return 32 - (((l << 31) // two_n) ^ ((r << 31) // two_n)).bit_length()
    return node_power_def(s1 + 1, e1 + 1, s2 + 1, e2 + 1, n)


def boundaries_numpy(a: np.ndarray) -> np.ndarray:
    """Run-boundary positions B = {k in [1, n-2] : asc_k != asc_{k-1}} U {n-1},
    asc_k = a[k] <= a[k+1] (the ends of find_run_right's scans)."""
    n = len(a)
    asc = a[:-1] <= a[1:]
    k = np.nonzero(asc[1:] != asc[:-1])[0] + 1
    return np.concatenate([k, [n - 1]]).astype(np.int64)


def insertion_comparisons(chunk: np.ndarray, npre: int) -> int:
    """runcore.py:232-244 on the (post-reversal) chunk."""
    length = len(chunk)
    npre = max(1, npre)
    if length <= 1 or npre >= length:
        return 0
    idx = np.arange(length)
    greater = (chunk[:, None] > chunk[None, :]) & (idx[:, None] < idx[None, :])
    g = greater.sum(axis=0)
    return int((g + (g < idx))[npre:].sum())


def powersort_metrics(n: int, min_run_len: int, bounds: Sequence[int],
                      asc_at: Callable[[np.ndarray], np.ndarray],
                      window: Callable[[int, int], np.ndarray],
                      merge_kind: str = "bitonic") -> Dict:
    """Metrics (and leaves / powers) of reference powersort on an array of n keys.

    bounds   sorted run-boundary positions (``boundaries_numpy`` semantics)
    asc_at   positions -> bool array of asc_k = a[k] <= a[k+1] (k < n-1)
    window   (lo, hi) -> original a[lo..hi] (inclusive), for extended leaves
    """
    if merge_kind != "bitonic":
        raise NotImplementedError("classic merge comparisons need the merged runs' contents")
    w = int(min_run_len)
    B = np.asarray(bounds, dtype=np.int64)
    # leaf chain (sorters.py:462-470): natural end = first boundary > start
    starts: List[int] = []
    nat_ends: List[int] = []
    ends: List[int] = []
    p = 0
    while p < n:
        if p >= n - 1:
            ne = n - 1
        else:
            ne = int(B[bisect.bisect_right(B, p)])
        e = ne if ne - p + 1 >= w else min(n - 1, p + w - 1)
        starts.append(p)
        nat_ends.append(ne)
        ends.append(e)
        p = e + 1
    r = len(starts)
    st = np.asarray(starts, dtype=np.int64)
    ne_a = np.asarray(nat_ends, dtype=np.int64)
    en = np.asarray(ends, dtype=np.int64)
    comparisons = 0
    # find_run_right comparisons (runcore.py:154,157): start == n-1 costs nothing
    scan = st < n - 1
    comparisons += int(np.where(ne_a[scan] < n - 1, ne_a[scan] - st[scan] + 1, ne_a[scan] - st[scan]).sum())
    # insertion sort of extended leaves, on the chunk after reversal (runcore.py:215-248)
    ext = np.nonzero(en > ne_a)[0]
    if len(ext):
        desc = ~np.asarray(asc_at(st[ext]), dtype=bool)
        desc &= st[ext] < n - 1
        for k, d in zip(ext.tolist(), desc.tolist()):
            lo, j, hi = starts[k], nat_ends[k], ends[k]
            chunk = np.asarray(window(lo, hi)).copy()
            if d:
                chunk[: j - lo + 1] = chunk[: j - lo + 1][::-1]
            comparisons += insertion_comparisons(chunk, j - lo + 1)
    # power stack (sorters.py:452-516)
    powers: List[int] = []
    merge_cost = 0
    max_power = n.bit_length()
    run_start = [-1] * (max_power + 1)
    top = 0
    occupied = 0
    max_stack = 0
    s1, e1 = starts[0], ends[0]
    for i in range(1, r):
        s2, e2 = starts[i], ends[i]
        pw = node_power0(s1, e1, s2, e2, n)
        powers.append(pw)
        for level in range(top, pw, -1):
            if run_start[level] < 0:
                continue
            merge_cost += e1 - run_start[level] + 1
            s1 = run_start[level]
            run_start[level] = -1
            occupied -= 1
        if run_start[pw] >= 0:
            raise AssertionError("node power repeated on the run stack")
        run_start[pw] = s1
        occupied += 1
        max_stack = max(max_stack, occupied)
        top = pw
        s1, e1 = s2, e2
    for level in range(top, 0, -1):
        if run_start[level] < 0:
            continue
        merge_cost += n - run_start[level]
        s1 = run_start[level]
        run_start[level] = -1
    comparisons += merge_cost  # bitonic: one comparison per merged element
    return dict(merge_cost=merge_cost, comparisons=comparisons, runs_detected=r,
                max_stack_height=max_stack, leaf_starts=st, leaf_lengths=en - st + 1,
                powers=np.asarray(powers, dtype=np.int64))


def powersort_metrics_numpy(a: np.ndarray, min_run_len: int = 24) -> Dict:
    """powersort_metrics for a host array (used to pin this module)."""
    a = np.asarray(a)
    n = len(a)
    if n <= 1:
        return dict(merge_cost=0, comparisons=0, runs_detected=n, max_stack_height=0)
    asc = a[:-1] <= a[1:]
    return powersort_metrics(n, min_run_len, boundaries_numpy(a), lambda pos: asc[pos],
                             lambda lo, hi: a[lo: hi + 1])
