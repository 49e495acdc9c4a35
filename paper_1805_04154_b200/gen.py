"""Input generators and run profiles of the reference harness (gen.py:1-236).

These produce the host arrays the reference's ``run_experiment`` feeds to the
sorters (``bench.py:111-118``), bit-identical to the reference for the same
(generator, parameters, seed): one ``PCG64(seed)`` Generator per call, the same
draws in the same order.  They are the data source on one side of the sort
path, not the path itself; the sort runs on the device.

Differences from the reference are in the mechanics only:
  * ``random_runs`` draws the same geometric batches (``gen.py:91-99``) but
    sorts all segments with one ``lexsort`` instead of a Python loop (the keys
    are a permutation, so the result is identical);
  * ``run_profile`` finds the maximal runs from the boundary set of the pair
    bits (from boundary b the next run ends at the first
    boundary >= b + 2) instead of walking the array element by element.
"""
from __future__ import annotations

from dataclasses import dataclass
from pathlib import Path
from typing import Iterable, Union

import numpy as np

from .io import load_array, save_array

__all__ = [
    "RunProfile",
    "random_permutation",
    "random_runs",
    "timsort_drag",
    "timsort_drag_lengths",
    "from_run_lengths",
    "run_profile",
    "save_array",
    "load_array",
]


@dataclass(frozen=True)
class RunProfile:
    """Lengths of the maximal runs of an array, left to right (gen.py:39-61)."""

    lengths: tuple

    def __post_init__(self) -> None:
        if any(L < 1 for L in self.lengths):
            raise ValueError("run lengths must be positive")

    @property
    def n(self) -> int:
        return sum(self.lengths)

    @property
    def r(self) -> int:
        return len(self.lengths)

    def __iter__(self):
        return iter(self.lengths)

    def __len__(self) -> int:
        return len(self.lengths)


def _rng(seed: int) -> np.random.Generator:
    return np.random.Generator(np.random.PCG64(seed))


def random_permutation(n: int, seed: int) -> np.ndarray:
    """Uniform permutation of 1..n (gen.py:68-73)."""
    if n < 0:
        raise ValueError("n must be >= 0")
    return (_rng(seed).permutation(n) + 1).astype(np.int64)


def random_runs(n: int, mean_len: int, seed: int) -> np.ndarray:
    """Permutation of 1..n with geometric(1/mean_len) segments sorted (gen.py:76-100)."""
    if mean_len < 1:
        raise ValueError("mean_len must be >= 1")
    rng = _rng(seed)
    a = (rng.permutation(n) + 1).astype(np.int64)
    if n == 0:
        return a
    batch = max(16, n // mean_len + 1)
    draws = []
    covered = 0
    while covered < n:  # the reference draws a new batch only while pos < n
        b = rng.geometric(1.0 / mean_len, size=batch)
        draws.append(b)
        covered += int(b.sum())
    ends = np.minimum(np.cumsum(np.concatenate(draws)), n)
    last = int(np.searchsorted(ends, n))  # first segment reaching n
    seg = np.zeros(n, dtype=np.int64)
    inner = ends[:last]
    inner = inner[inner < n]
    seg[inner] = 1
    seg = np.cumsum(seg)
    return a[np.lexsort((a, seg))]


def timsort_drag_lengths(n: int) -> list:
    """R(m) = R(m/2) ++ R(m/4) ++ [m/4], R(m) = [m] for m <= 3 (gen.py:103-126)."""
    if n < 1:
        raise ValueError("n must be >= 1")
    if n > 3 and (n & (n - 1)) != 0:
        raise ValueError("drag profile needs a power-of-two length")
    out: list = []
    stack = [n]  # explicit pre-order walk of the same recursion
    while stack:
        m = stack.pop()
        if m < 0:
            out.append(-m)
        elif m <= 3:
            out.append(m)
        else:
            stack.extend((-(m // 4), m // 4, m // 2))
    return out


def timsort_drag(n: int, run_scale: int = 32,
                 lengths_path: Union[str, Path, None] = None) -> np.ndarray:
    """Drag profile scaled by run_scale (gen.py:129-150)."""
    if run_scale < 1:
        raise ValueError("run_scale must be >= 1")
    if n % run_scale != 0:
        raise ValueError("n must be a multiple of run_scale")
    if lengths_path is not None:
        with open(lengths_path) as fh:
            base = [int(line) for line in fh if line.strip()]
    else:
        base = timsort_drag_lengths(n // run_scale)
    lens = [L * run_scale for L in base]
    if sum(lens) != n:
        raise ValueError(f"scaled run lengths sum to {sum(lens)}, expected n={n}")
    return from_run_lengths(lens)


def from_run_lengths(lengths: Iterable[int], seed: int = 0) -> np.ndarray:
    """Blocks of consecutive values assigned from the top down (gen.py:153-171)."""
    lengths = np.asarray([int(L) for L in lengths], dtype=np.int64)
    if np.any(lengths < 1):
        raise ValueError("run lengths must be >= 1")
    n = int(lengths.sum())
    if n == 0:
        return np.empty(0, dtype=np.int64)
    starts = np.cumsum(lengths) - lengths          # position of each block
    tops = n - starts                              # top value of each block
    block = np.repeat(np.arange(len(lengths)), lengths)
    offs = np.arange(n, dtype=np.int64) - starts[block]
    return tops[block] - lengths[block] + 1 + offs


def run_profile(a) -> RunProfile:
    """Maximal weakly-increasing / strictly-decreasing runs (gen.py:174-202)."""
    a = np.asarray(a)
    n = len(a)
    if n == 0:
        return RunProfile(())
    if n == 1:
        return RunProfile((1,))
    asc = a[:-1] <= a[1:]
    # run ends: k with asc_k != asc_{k-1} (k in 1..n-2) plus n-1; from a run
    # ending at b the next run starts at b+1 and ends at the first end >= b+2,
    # so inside a block of consecutive candidates every other one is taken.
    cand = np.flatnonzero(asc[1:] != asc[:-1]) + 1
    cand = np.append(cand, n - 1)
    newblk = np.ones(len(cand), dtype=bool)
    newblk[1:] = cand[1:] != cand[:-1] + 1
    blk_start = np.maximum.accumulate(np.where(newblk, np.arange(len(cand)), 0))
    ends = cand[((np.arange(len(cand)) - blk_start) & 1) == 0]
    if ends[-1] != n - 1:  # n-1 skipped as b+1: it forms a 1-run of its own
        ends = np.append(ends, n - 1)
    lengths = np.diff(np.concatenate(([-1], ends)))
    return RunProfile(tuple(int(L) for L in lengths))
