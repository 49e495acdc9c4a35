"""Pin the C oracle against the reference's own outputs (tests/golden).

CPU only.  The oracle is the checker for every GPU parity test, so it must
reproduce the reference bit for bit: sorted keys and tags, all four Metrics
counters, the merge-tree shape, and node powers (reference sorters.py:376-423).
"""

import numpy as np
import pytest

from oracle import oracle
from tests import golden_data as G


def _tree_nodes_inorder(t, out):
    if t[0] == "N":
        _tree_nodes_inorder(t[3], out)
        out.append(t[2])
        _tree_nodes_inorder(t[4], out)
    return out


@pytest.fixture(scope="module")
def golden():
    return G.load()


def _run(case, arrays, want_tree=False):
    a, tags = G.case_inputs(case, arrays)
    work = a.copy()
    tw = tags.copy() if tags is not None else None
    fn = oracle.powersort if case["algo"] == "powersort" else oracle.peeksort
    res = fn(work, case["w"], case["merge_kind"], tw, want_tree=want_tree)
    return a, tags, work, tw, res


def test_oracle_matches_reference_metrics_and_outputs(golden):
    meta, arrays = golden
    bad = []
    for case in meta["cases"]:
        a, tags, work, tw, res = _run(case, arrays)
        got_sha = G.sha(work) if tw is None else G.sha(work, tw)
        if res.metrics_tuple() != G.metrics_of(case) or got_sha != case["out_sha"]:
            bad.append((case["input"], case["algo"], case["w"], case["merge_kind"],
                        res.metrics_tuple(), G.metrics_of(case)))
    assert not bad, f"{len(bad)} mismatches, first: {bad[:3]}"


def test_oracle_trees_match_reference(golden):
    meta, arrays = golden
    n_checked = 0
    for case in meta["cases"]:
        if "tree" not in case:
            continue
        a, tags, work, tw, res = _run(case, arrays, want_tree=True)
        want = G.tree_shape(case["tree"])
        n = len(a)
        if case["algo"] == "powersort":
            starts = list(res.leaf_starts) + [n]
            lens = np.diff(starts)
            got = oracle.power_tree_from_powers(lens, list(res.powers))
            if case["tree"][0] == "N":
                assert list(res.powers) == _tree_nodes_inorder(case["tree"], [])
        else:
            got = oracle.peek_tree_from_merges(n, res.merges)
        assert got == want, (case["input"], case["algo"], case["w"])
        n_checked += 1
    assert n_checked >= 400


def test_six_run_golden_values(golden):
    """Reference tests/test_acceptance.py:205-215 (criterion 4)."""
    a = golden[1]["fig"]
    r = oracle.powersort(a.copy(), 1, "classic", want_tree=True)
    assert list(r.powers) == [3, 2, 1, 2, 4] and r.merge_cost == 67
    assert oracle.peeksort(a.copy(), 1, "classic").merge_cost == 65


def test_reference_unit_examples():
    """Reference tests/test_sorters.py:61-112."""
    a = np.arange(1, 101, dtype=np.int64)
    r = oracle.peeksort(a, 1, "classic")
    assert (r.merge_cost, r.comparisons, r.runs_detected) == (0, 99, 1)
    a = np.arange(100, 0, -1).astype(np.int64)
    r = oracle.peeksort(a, 1, "classic")
    assert r.merge_cost == 0 and r.comparisons == 99 and np.all(a[:-1] <= a[1:])
    a = np.concatenate([np.arange(32, 64), np.arange(0, 32)]).astype(np.int64)
    r = oracle.powersort(a, 1, "classic")
    assert r.merge_cost == 64 and r.runs_detected == 2
    for n in (0, 1):
        r = oracle.peeksort(np.arange(n, dtype=np.int64), 1, "classic")
        assert r.merge_cost == 0 and r.comparisons == 0 and r.runs_detected == n


def test_node_powers_match_reference(golden):
    meta, _ = golden
    for s1, e1, s2, e2, n, p in meta["node_powers"]:
        assert oracle.node_power_def(s1, e1, s2, e2, n) == p
        assert oracle.node_power0(s1 - 1, e1 - 1, s2 - 1, e2 - 1, n) == p


# --------------------------------------------------------------- analytic
def test_analytic_node_powers_match_reference(golden):
    """oracle/analytic.py's node_power_def / node_power0 vs the reference's own
    node_power_def outputs (including n = 2^31, where powersort uses the loop)."""
    from oracle import analytic

    meta, _ = golden
    big = 0
    for s1, e1, s2, e2, n, p in meta["node_powers"]:
        assert analytic.node_power_def(s1, e1, s2, e2, n) == p
        assert analytic.node_power0(s1 - 1, e1 - 1, s2 - 1, e2 - 1, n) == p
        big += n >= 1 << 31
    assert big > 0


def test_analytic_metrics_match_oracle():
    """Metrics from the run structure alone == the element-by-element oracle,
    on inputs with duplicates, strictly descending runs and short runs."""
    from oracle import analytic

    rng = np.random.default_rng(11)
    for it in range(300):
        n = int(rng.integers(2, 3000))
        kind = it % 4
        if kind == 0:
            a = rng.integers(0, 5, n)
        elif kind == 1:
            a = rng.integers(0, 1 << 40, n)
            b = np.sort(rng.choice(n, size=min(n - 1, int(rng.integers(1, 40))), replace=False))
            for s, e in zip(np.r_[0, b], np.r_[b, n]):
                a[s:e] = np.sort(a[s:e])[:: (1 if rng.random() < 0.5 else -1)]
        elif kind == 2:
            a = np.arange(n)[:: -1].copy()
        else:
            a = np.repeat(rng.integers(0, 100, n // 7 + 1), 7)[:n]
        a = a.astype(np.int64)
        w = int(rng.choice([1, 2, 3, 7, 24, 100]))
        got = analytic.powersort_metrics_numpy(a, w)
        res = oracle.powersort(a.copy(), w, "bitonic", want_tree=True)
        assert (got["merge_cost"], got["comparisons"], got["runs_detected"], got["max_stack_height"]) == \
            res.metrics_tuple(), (it, n, w)
        assert np.array_equal(got["leaf_starts"], res.leaf_starts)
        assert np.array_equal(got["powers"], res.powers)
