"""GPU parity: the CUDA powersort vs the reference (golden fixtures) and the C oracle.

Bit-exact on keys and tags (stability through index payloads) and on all four
Metrics counters; merge trees equal on shape, sizes and powers.
"""
import numpy as np
import pytest

import paper_1805_04154_b200 as rs
from oracle import oracle
from paper_1805_04154_b200 import workloads
from tests import golden_data as G

pytestmark = pytest.mark.gpu


def _shape(t):
    if isinstance(t, rs.MergeLeaf):
        return ("L", t.length)
    return ("N", _shape(t.left), _shape(t.right))


def _run_gpu(a, w, mk, tags=None, record=False):
    work = a.copy()
    tw = tags.copy() if tags is not None else None
    m = rs.powersort(work, rs.SortConfig(min_run_len=w, merge_kind=mk, record_tree=record), tags=tw)
    return work, tw, m


def _mt(m):
    return (m.merge_cost, m.comparisons, m.runs_detected, m.max_stack_height)


def test_golden_small_and_medium_match_reference():
    meta, arrays = G.load()
    bad = []
    n_cases = 0
    for case in meta["cases"]:
        if case["algo"] != "powersort":
            continue
        a, tags = G.case_inputs(case, arrays)
        work, tw, m = _run_gpu(a, case["w"], case["merge_kind"], tags)
        got_sha = G.sha(work) if tw is None else G.sha(work, tw)
        if _mt(m) != G.metrics_of(case) or got_sha != case["out_sha"]:
            bad.append((case["input"], case["w"], case["merge_kind"], _mt(m), G.metrics_of(case)))
        n_cases += 1
    assert not bad, f"{len(bad)}/{n_cases} mismatches, first: {bad[:4]}"


def test_golden_trees_match_reference():
    meta, arrays = G.load()
    for case in meta["cases"]:
        if case["algo"] != "powersort" or "tree" not in case:
            continue
        a, _ = G.case_inputs(case, arrays)
        _, _, m = _run_gpu(a, case["w"], case["merge_kind"], record=True)
        assert _shape(m.merge_tree) == G.tree_shape(case["tree"]), case["input"]
        if case["tree"][0] == "N":
            want = []

            def walk(x):
                if x[0] == "N":
                    walk(x[3]); want.append((x[1], x[2])); walk(x[4])
            walk(case["tree"])
            assert [(nd.size, nd.power) for nd in rs.internal_nodes_inorder(m.merge_tree)] == want


@pytest.mark.parametrize("key_dtype", [np.int32, np.int64])
@pytest.mark.parametrize("tag_dtype", [None, np.int32, np.int64])
def test_random_inputs_vs_oracle(key_dtype, tag_dtype):
    rng = np.random.default_rng(11 + (key_dtype == np.int64) + 3 * (tag_dtype is not None))
    for trial in range(40):
        n = int(rng.choice([2, 3, 5, 31, 33, 100, 1000, 4095, 4097, 5000, 20000, 70000]))
        kind = trial % 5
        if kind == 0:
            a = rng.permutation(n)
        elif kind == 1:
            a = rng.integers(0, max(2, n // 50), size=n)
        elif kind == 2:
            a = workloads.config4(n, seed=trial, mean=float(rng.integers(2, 300)))[0]
        elif kind == 3:
            a = workloads.config3(n, seed=trial)
        else:
            a = np.resize(np.repeat(rng.integers(-5, 5, size=max(1, n // 7 + 1)), 7), n)
            a[rng.integers(0, n, size=n // 10)] *= -1
        a = a.astype(key_dtype)
        tags = np.arange(n).astype(tag_dtype) if tag_dtype is not None else None
        w = int(rng.choice([1, 2, 3, 7, 24, 32, 33, 100]))
        mk = "classic" if trial % 2 else "bitonic"
        ref_a, ref_t = a.copy(), None if tags is None else tags.copy()
        ref = oracle.powersort(ref_a, w, mk, ref_t)
        work, tw, m = _run_gpu(a, w, mk, tags)
        assert np.array_equal(work, ref_a), (n, kind, w, mk)
        if tags is not None:
            assert np.array_equal(tw, ref_t), (n, kind, w, mk)
        assert _mt(m) == ref.metrics_tuple(), (n, kind, w, mk)


@pytest.mark.parametrize("n", [2, 3, 4, 24, 25, 4096, 4097, 9000, 100001])
def test_edge_shapes(n):
    cases = [
        np.zeros(n, dtype=np.int64),                       # all equal: one run
        np.arange(n, 0, -1).astype(np.int64),              # strictly descending: one reversed run
        np.arange(n).astype(np.int64),                     # sorted
        (np.arange(n) % 2).astype(np.int64),               # zig-zag
        np.concatenate([np.arange(n // 2, n), np.arange(n // 2)]).astype(np.int64),
        np.full(n, np.iinfo(np.int64).max, dtype=np.int64),
    ]
    for a in cases:
        for w in (1, 24, max(1, min(n, 1024))):
            tags = np.arange(n, dtype=np.int64)
            ref_a, ref_t = a.copy(), tags.copy()
            ref = oracle.powersort(ref_a, w, "classic", ref_t)
            work, tw, m = _run_gpu(a, w, "classic", tags)
            assert np.array_equal(work, ref_a) and np.array_equal(tw, ref_t)
            assert _mt(m) == ref.metrics_tuple()


def test_metrics_accumulate_like_reference():
    a = workloads.config2(50000, seed=2)
    m = rs.Metrics(merge_cost=5, comparisons=7, runs_detected=1, max_stack_height=100)
    ref = oracle.powersort(a.copy(), 24, "bitonic")
    rs.powersort(a.copy(), None, m)
    assert m.merge_cost == 5 + ref.merge_cost
    assert m.comparisons == 7 + ref.comparisons
    assert m.runs_detected == 1 + ref.runs_detected
    assert m.max_stack_height == 100


def test_torch_tensors_in_place_and_dtypes():
    import torch

    a = workloads.config2(30000, seed=5)
    ref = a.copy()
    oracle.powersort(ref, 24, "bitonic")
    t = torch.from_numpy(a.copy()).cuda()
    ptr = t.data_ptr()
    rs.powersort(t)
    assert t.data_ptr() == ptr and np.array_equal(t.cpu().numpy(), ref)
    p = torch.from_numpy(a.copy()).pin_memory()
    rs.powersort(p)
    assert np.array_equal(p.numpy(), ref)
    for dt in (np.uint32, np.uint64, np.int16, np.uint8):
        b = (a % 250).astype(dt) if dt in (np.int16, np.uint8) else a.astype(dt) * 3
        want = np.sort(b, kind="stable")
        rs.powersort(b)
        assert np.array_equal(b, want), dt


@pytest.mark.slow
@pytest.mark.parametrize("cfg", [1, 2, 3, 4])
def test_baseline_configs_full_size(cfg):
    a, tags = workloads.generate(cfg)
    ref_a, ref_t = a.copy(), None if tags is None else tags.copy()
    ref = oracle.powersort(ref_a, 24, "bitonic", ref_t)
    work, tw, m = _run_gpu(a, 24, "bitonic", tags)
    assert np.array_equal(work, ref_a)
    if tags is not None:
        assert np.array_equal(tw, ref_t)
    assert _mt(m) == ref.metrics_tuple()


# ---- thresholds of the device path: every size rule has a case on each side
def _segments(r, seg_len, rng, desc_every=0, dtype=np.int32):
    """r natural runs of seg_len keys (>= min_run_len, so exactly r leaves): each
    segment ascends over the same value range, so every boundary is a descent;
    every desc_every-th segment is strictly descending instead."""
    out = np.empty(r * seg_len, dtype=dtype)
    for k in range(r):
        seg = np.sort(rng.choice(1 << 20, size=seg_len, replace=False)).astype(dtype)
        if desc_every and k % desc_every == desc_every - 1:
            seg = seg[::-1] + (1 << 21)  # strictly descending, above its neighbours
        out[k * seg_len:(k + 1) * seg_len] = seg
    return out


@pytest.mark.parametrize("r", [2047, 2048, 2049, 2050])
@pytest.mark.parametrize("desc_every", [0, 3])
def test_small_tree_threshold(r, desc_every):
    """Trees of <= 2048 leaves are built by one CTA out of shared memory (ready-time
    job order, fused >= 3-leaf subtrees), larger ones by the grid phases."""
    rng = np.random.default_rng(100 + r + desc_every)
    a = _segments(r, 40, rng, desc_every)
    tags = np.arange(len(a), dtype=np.int32)
    for mk in ("bitonic", "classic"):
        work, tw, m = _run_gpu(a, 24, mk, tags)
        rk, rt = a.copy(), tags.copy()
        ref = oracle.powersort(rk, 24, mk, rt)
        assert np.array_equal(work, rk) and np.array_equal(tw, rt)
        assert _mt(m) == ref.metrics_tuple()
        if desc_every == 0:
            assert m.runs_detected == r


@pytest.mark.parametrize("n", [(1 << 22) - 1, 1 << 22, (1 << 22) + 1, 2048 * 3552 - 1, 2048 * 3552])
def test_chain_tile_thresholds(n):
    """The chain-tile size is chosen from n (512 / 1024 / 2560 positions)."""
    keys = workloads.config2(n, seed=3, mean=700.0)
    work, _, m = _run_gpu(keys, 24, "bitonic")
    ref_k = keys.copy()
    ref = oracle.powersort(ref_k, 24, "bitonic")
    assert np.array_equal(work, ref_k)
    assert _mt(m) == ref.metrics_tuple()


def test_long_leaves_small_tree_fuses_three_leaf_subtrees():
    """Long leaves on average (n >= 256 r) with clusters of short runs: the small-tree
    path fuses the clusters (>= 3 leaves within 4096 elements) and leaves pairs to the
    executor; output, payload and Metrics equal the oracle either way."""
    rng = np.random.default_rng(77)
    parts = []
    for k in range(40):
        parts.append(np.sort(rng.integers(0, 1 << 30, size=200_000, dtype=np.int64)).astype(np.int32))
        for length in rng.integers(25, 900, size=int(rng.integers(1, 6))):
            seg = np.sort(rng.integers(0, 1 << 30, size=int(length), dtype=np.int64)).astype(np.int32)
            parts.append(seg[::-1].copy() if k % 2 else seg)
    a = np.concatenate(parts)
    tags = np.arange(len(a), dtype=np.int64)
    work, tw, m = _run_gpu(a, 24, "classic", tags)
    rk, rt = a.copy(), tags.copy()
    ref = oracle.powersort(rk, 24, "classic", rt)
    assert np.array_equal(work, rk) and np.array_equal(tw, rt)
    assert _mt(m) == ref.metrics_tuple()
    assert len(a) >= 256 * m.runs_detected
