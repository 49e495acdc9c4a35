"""Merge-tree records (reference opttree.py:60-75) and their reconstruction
from the device's per-boundary depths.

Equality is on shape only (leaf index and children); `length`, `size` and
`power` are metadata, exactly as in the reference.
"""
from __future__ import annotations

from dataclasses import dataclass, field
from typing import Optional, Sequence, Union

__all__ = ["MergeLeaf", "MergeNode", "MergeTree", "tree_from_depths", "internal_nodes_inorder"]


@dataclass(frozen=True)
class MergeLeaf:
    """Leaf i of a merge tree.  ``length`` is metadata (run length)."""

    index: int
    length: object = field(default=None, compare=False)


@dataclass(frozen=True)
class MergeNode:
    """Internal node; ``size``/``power`` are metadata, equality is shape-only."""

    left: "MergeTree"
    right: "MergeTree"
    size: object = field(default=None, compare=False)
    power: Optional[int] = field(default=None, compare=False)


MergeTree = Union[MergeLeaf, MergeNode]


def tree_from_depths(leaf_lengths: Sequence[int], depths: Sequence[int],
                     powers: Optional[Sequence[int]] = None) -> MergeTree:
    """Rebuild the merge tree from internal-node depths in boundary order.

    Boundary j (1-based) separates leaf j-1 and leaf j; its node is the
    min-Cartesian tree of the depths (ancestors are strictly shallower and two
    nodes of equal depth always have a shallower node between them), the same
    construction as reference opttree.py:308-336 applied to depths.
    """
    r = len(leaf_lengths)
    if r == 1:
        return MergeLeaf(0, int(leaf_lengths[0]))
    m = r - 1
    left = [0] * (m + 1)
    right = [0] * (m + 1)
    stack: list = []
    for j in range(1, m + 1):
        last = 0
        while stack and depths[stack[-1] - 1] > depths[j - 1]:
            last = stack.pop()
        left[j] = last
        if stack:
            right[stack[-1]] = j
        stack.append(j)
    prefix = [0]
    for L in leaf_lengths:
        prefix.append(prefix[-1] + int(L))

    # iterative post-order to avoid deep recursion on skewed trees
    built: dict = {}
    lo = {}
    hi = {}
    order = []
    todo = [stack[0]]
    while todo:
        j = todo.pop()
        order.append(j)
        if left[j]:
            todo.append(left[j])
        if right[j]:
            todo.append(right[j])
    for j in reversed(order):
        if left[j]:
            lt, a = built[left[j]], lo[left[j]]
        else:
            lt, a = MergeLeaf(j - 1, int(leaf_lengths[j - 1])), j - 1
        if right[j]:
            rt, b = built[right[j]], hi[right[j]]
        else:
            rt, b = MergeLeaf(j, int(leaf_lengths[j])), j
        lo[j], hi[j] = a, b
        size = prefix[b + 1] - prefix[a]
        built[j] = MergeNode(lt, rt, size=size, power=None if powers is None else int(powers[j - 1]))
    return built[stack[0]]


def internal_nodes_inorder(tree: MergeTree) -> list:
    out = []
    todo = [(tree, False)]
    while todo:
        t, seen = todo.pop()
        if isinstance(t, MergeLeaf):
            continue
        if seen:
            out.append(t)
        else:
            todo.append((t.right, False))
            todo.append((t, True))
            todo.append((t.left, False))
    return out
