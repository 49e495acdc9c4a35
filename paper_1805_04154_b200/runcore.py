"""Result records of the sort entry points (reference runcore.py:40-67).

Same fields, defaults and accumulate semantics as the reference, so a
reference user's `Metrics` handling is unchanged.
"""
from __future__ import annotations

from dataclasses import dataclass
from typing import Optional

__all__ = ["Metrics", "Run"]


@dataclass
class Metrics:
    """Instrumentation counters for one sort invocation (runcore.py:40-55).

    merge_cost        sum of output sizes over all executed merges
    comparisons       key comparisons (run detection + merging + insertion)
    runs_detected     number of leaves the sorter worked from
    max_stack_height  peak number of pending runs (powersort)
    merge_tree        recorded merge tree when SortConfig.record_tree is set
    """

    merge_cost: int = 0
    comparisons: int = 0
    runs_detected: int = 0
    max_stack_height: int = 0
    merge_tree: Optional[object] = None


@dataclass(frozen=True)
class Run:
    """Inclusive index range [start, end]; descending means it was reversed
    (runcore.py:58-67)."""

    start: int
    end: int
    descending: bool = False

    def __len__(self) -> int:
        return self.end - self.start + 1
