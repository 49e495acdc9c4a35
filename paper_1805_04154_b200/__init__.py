"""B200-native run-adaptive stable mergesort (powersort / peeksort of arXiv 1805.04154).

Drop-in for the reference package's sort entry points (reference
``runsort/__init__.py:9-61``): ``powersort``, ``peeksort``, ``SortConfig``,
``Metrics``, ``Run``, ``SORTERS``, ``MergeLeaf``, ``MergeNode`` and the node
power functions keep the reference names, arguments, return values and
exceptions; the sorting itself runs in hand-written sm_100a CUDA kernels
behind the C ABI in ``include/runsort_b200.h``.
"""
from .opttree import MergeLeaf, MergeNode, internal_nodes_inorder
from .runcore import Metrics, Run
from .io import load_array, load_array_device, save_array
from .sorters import (SORTERS, SortConfig, alpha_merge_sort, alpha_stack_sort, bottom_up_mergesort,
                      node_power_bitwise, node_power_def, peeksort, powersort, top_down_mergesort)

__all__ = [
    "load_array",
    "load_array_device",
    "save_array",
    "Metrics", "Run", "SortConfig", "SORTERS",
    "peeksort", "powersort",
    "top_down_mergesort", "bottom_up_mergesort", "alpha_stack_sort", "alpha_merge_sort",
    "node_power_def", "node_power_bitwise",
    "MergeLeaf", "MergeNode", "internal_nodes_inorder",
]

__version__ = "0.1.0"
