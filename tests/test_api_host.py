"""Host-side API mirror: SortConfig, node powers, tree reconstruction, n <= 1 paths (CPU only)."""
import numpy as np
import pytest

import paper_1805_04154_b200 as rs
from oracle import oracle
from paper_1805_04154_b200.opttree import tree_from_depths
from tests import device_model as DM
from tests import golden_data as G


def test_config_validation_matches_reference():
    with pytest.raises(ValueError):
        rs.SortConfig(min_run_len=0)
    with pytest.raises(ValueError):
        rs.SortConfig(merge_kind="galloping")
    with pytest.raises(ValueError):
        rs.SortConfig(alpha=1.0)
    assert rs.SortConfig() == rs.SortConfig(24, "bitonic", False, 2.0)


def test_node_power_functions_match_reference_golden():
    meta, _ = G.load()
    for s1, e1, s2, e2, n, p in meta["node_powers"]:
        assert rs.node_power_def(s1, e1, s2, e2, n) == p
        if n < 1 << 31:
            assert rs.node_power_bitwise(s1, e1, s2, e2, n) == p
    with pytest.raises(ValueError):
        rs.node_power_def(0, 1, 2, 3, 4)
    with pytest.raises(ValueError):
        rs.node_power_bitwise(1, 1, 2, 2, 1 << 31)


def test_empty_and_single_need_no_device():
    for n in (0, 1):
        m = rs.powersort(np.arange(n, dtype=np.int64), rs.SortConfig(record_tree=True))
        assert (m.merge_cost, m.comparisons, m.runs_detected) == (0, 0, n)
        assert (m.merge_tree == rs.MergeLeaf(0, 1)) if n == 1 else m.merge_tree is None
        m = rs.peeksort(np.arange(n, dtype=np.int64))
        assert m.runs_detected == n


def _shape(t):
    if isinstance(t, rs.MergeLeaf):
        return ("L", t.length)
    return ("N", _shape(t.left), _shape(t.right))


def test_tree_from_depths_rebuilds_reference_trees():
    """Depths from the device formulation (la + ra scans) rebuild the exact
    reference powersort trees, including sizes and powers."""
    meta, arrays = G.load()
    checked = 0
    for case in meta["cases"]:
        if case["algo"] != "powersort" or "tree" not in case or case["tree"][0] != "N":
            continue
        a, _ = G.case_inputs(case, arrays)
        res = oracle.powersort(a.copy(), case["w"], case["merge_kind"], want_tree=True)
        starts = list(res.leaf_starts) + [len(a)]
        lens = np.diff(starts)
        depth, _ = DM.depth_by_scans(list(res.powers))
        t = tree_from_depths(lens, depth[1:], list(res.powers))
        assert _shape(t) == G.tree_shape(case["tree"])
        want_nodes = []

        def walk(x):
            if x[0] == "N":
                walk(x[3]); want_nodes.append((x[1], x[2])); walk(x[4])
        walk(case["tree"])
        got = [(nd.size, nd.power) for nd in rs.internal_nodes_inorder(t)]
        assert got == want_nodes
        checked += 1
    assert checked > 100


def test_unsupported_key_dtype_is_loud():
    torch = pytest.importorskip("torch")
    if torch.cuda.is_available():
        with pytest.raises(NotImplementedError):
            rs.powersort(np.array([1.5, np.nan]))  # NaN keys: no order to follow
        with pytest.raises(NotImplementedError):
            rs.powersort(np.array(["b", "a"]))
    else:
        with pytest.raises(RuntimeError):
            rs.powersort(np.array([3, 1, 2], dtype=np.int64))
