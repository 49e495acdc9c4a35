"""GPU parity for peeksort (reference sorters.py:146-361): outputs, all Metrics
(runs_detected is assigned, max_stack_height untouched) and recorded trees vs
the reference fixtures and the C oracle."""
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


def _run(a, w, mk, tags=None, record=False):
    work = a.copy()
    tw = tags.copy() if tags is not None else None
    m = rs.peeksort(work, rs.SortConfig(min_run_len=w, merge_kind=mk, record_tree=record), tags=tw)
    return work, tw, m


def _mt(m):
    return (m.merge_cost, m.comparisons, m.runs_detected, m.max_stack_height)


def test_golden_peeksort_matches_reference():
    meta, arrays = G.load()
    bad = []
    n_cases = 0
    for case in meta["cases"]:
        if case["algo"] != "peeksort":
            continue
        a, tags = G.case_inputs(case, arrays)
        work, tw, m = _run(a, case["w"], case["merge_kind"], tags)
        got_sha = G.sha(work) if tw is None else G.sha(work, tw)
        if _mt(m) != G.metrics_of(case) or got_sha != case["out_sha"]:
            bad.append((case["input"], case["w"], case["merge_kind"], _mt(m), G.metrics_of(case)))
        n_cases += 1
    assert not bad, f"{len(bad)}/{n_cases} mismatches, first: {bad[:4]}"


def test_golden_peeksort_trees():
    meta, arrays = G.load()
    for case in meta["cases"]:
        if case["algo"] != "peeksort" or "tree" not in case:
            continue
        a, _ = G.case_inputs(case, arrays)
        _, _, m = _run(a, case["w"], case["merge_kind"], record=True)
        assert _shape(m.merge_tree) == G.tree_shape(case["tree"]), case["input"]


@pytest.mark.parametrize("key_dtype", [np.int32, np.int64])
def test_peeksort_random_vs_oracle(key_dtype):
    rng = np.random.default_rng(5 + (key_dtype == np.int64))
    for trial in range(40):
        n = int(rng.choice([2, 3, 7, 50, 1000, 5000, 20000, 70000]))
        kind = trial % 4
        if kind == 0:
            a = rng.permutation(n)
        elif kind == 1:
            a = rng.integers(0, max(2, n // 50), size=n)
        elif kind == 2:
            a = workloads.config4(n, seed=trial, mean=float(rng.integers(2, 300)))[0]
        else:
            a = workloads.config3(n, seed=trial)
        a = a.astype(key_dtype)
        tags = np.arange(n, dtype=np.int64)
        w = int(rng.choice([1, 2, 3, 7, 24, 100]))
        mk = "classic" if trial % 2 else "bitonic"
        ref_a, ref_t = a.copy(), tags.copy()
        ref = oracle.peeksort(ref_a, w, mk, ref_t)
        work, tw, m = _run(a, w, mk, tags)
        assert np.array_equal(work, ref_a) and np.array_equal(tw, ref_t), (n, kind, w, mk)
        assert _mt(m) == ref.metrics_tuple(), (n, kind, w, mk)


@pytest.mark.slow
def test_peeksort_config2_full():
    a, _ = workloads.generate(2)
    ref_a = a.copy()
    ref = oracle.peeksort(ref_a, 24, "bitonic")
    work, _, m = _run(a, 24, "bitonic")
    assert np.array_equal(work, ref_a)
    assert _mt(m) == ref.metrics_tuple()


def _runs_array(rng, lens, key_dtype):
    """Consecutive runs alternately ascending and strictly descending."""
    parts = []
    for i, L in enumerate(lens):
        v = np.sort(rng.choice(1 << 30, size=int(L), replace=False))
        parts.append(v if i % 2 == 0 else v[::-1])
    return np.concatenate(parts).astype(key_dtype)


@pytest.mark.parametrize("key_dtype", [np.int32, np.int64])
def test_peeksort_long_descending_runs_vs_oracle(key_dtype):
    """Few very long strictly descending runs (reversed by all blocks at once)
    and many short ones (one block per segment); both pass through the
    multi-level run-scan summaries."""
    rng = np.random.default_rng(11)
    cases = [
        [1 << 18, 3, 1 << 19, 5, (1 << 18) + 7],          # 5 long runs, 2^20 elements
        [int(x) for x in rng.integers(2, 3000, size=600)],  # > 64 descending runs per level
        [1 << 20, 1 << 20],                                  # one ascending + one descending run
    ]
    for lens in cases:
        a = _runs_array(rng, lens, key_dtype)
        n = len(a)
        tags = np.arange(n, dtype=np.int64)
        for w in (1, 24):
            ref_a, ref_t = a.copy(), tags.copy()
            ref = oracle.peeksort(ref_a, w, "bitonic", ref_t)
            work, tw, m = _run(a, w, "bitonic", tags)
            assert np.array_equal(work, ref_a) and np.array_equal(tw, ref_t), (len(lens), w)
            assert _mt(m) == ref.metrics_tuple(), (len(lens), w)


# ---- compact replay workspace: overflow -> input restored -> worst-case retry
def _zigzag(n, seed):
    """Runs of 2-3 elements in both directions: with min_run_len = 1 peeksort makes
    ~n / 2.5 leaves, far beyond the compact capacity n / 12 + 4096."""
    rng = np.random.default_rng(seed)
    return rng.integers(0, 1 << 30, size=n, dtype=np.int64)


@pytest.mark.parametrize("key_dtype,tag_dtype", [(np.int32, None), (np.int64, np.int32), (np.int32, np.int64)])
def test_peeksort_compact_overflow_c_abi(key_dtype, tag_dtype):
    """rs_sort with the compact workspace reports RS_ECAPACITY and leaves keys and
    tags exactly as they came; with RS_ALGO_FULL_WS the sort matches the oracle."""
    import ctypes

    import torch

    from paper_1805_04154_b200 import _lib

    L = _lib.lib()
    n, w = 300_000, 1
    a = _zigzag(n, 11).astype(key_dtype)
    # strictly descending stretches so that reversals are applied before the overflow
    a[1000:1400] = np.arange(400, 0, -1, dtype=key_dtype)
    a[150_000:150_900] = np.arange(900, 0, -1, dtype=key_dtype)
    tags = np.arange(n, dtype=tag_dtype) if tag_dtype is not None else None
    kc = _lib.RS_KEY_I32 if a.itemsize == 4 else _lib.RS_KEY_I64
    tb = tags.itemsize if tags is not None else 0
    dk = torch.from_numpy(a).cuda()
    dt = torch.from_numpy(tags).cuda() if tags is not None else None
    st = torch.cuda.current_stream()
    small = L.rs_workspace_bytes(_lib.RS_ALGO_PEEKSORT, kc, tb, n, w)
    full = L.rs_workspace_bytes(_lib.RS_ALGO_PEEKSORT | _lib.RS_ALGO_FULL_WS, kc, tb, n, w)
    assert small < full
    ws = torch.empty(full, dtype=torch.uint8, device="cuda")
    out = _lib.RsMetrics()
    rc = L.rs_sort(_lib.RS_ALGO_PEEKSORT, kc, dk.data_ptr(), tb, dt.data_ptr() if dt is not None else None, n, w, 0,
                   ws.data_ptr(), small, st.cuda_stream, ctypes.byref(out), None)
    assert rc == _lib.RS_ECAPACITY
    assert np.array_equal(dk.cpu().numpy(), a), "keys changed by an overflowed replay"
    if dt is not None:
        assert np.array_equal(dt.cpu().numpy(), tags), "tags changed by an overflowed replay"
    rc = L.rs_sort(_lib.RS_ALGO_PEEKSORT | _lib.RS_ALGO_FULL_WS, kc, dk.data_ptr(), tb,
                   dt.data_ptr() if dt is not None else None, n, w, 0, ws.data_ptr(), full, st.cuda_stream,
                   ctypes.byref(out), None)
    assert rc == _lib.RS_OK
    ref_k, ref_t = a.copy(), (tags.copy() if tags is not None else None)
    ref = oracle.peeksort(ref_k, w, "bitonic", ref_t)
    assert np.array_equal(dk.cpu().numpy(), ref_k)
    if dt is not None:
        assert np.array_equal(dt.cpu().numpy(), ref_t)
    assert (out.merge_cost, out.comparisons, out.runs_detected) == ref.metrics_tuple()[:3]
    assert ref.runs_detected > n // 12 + 4096  # the input does exceed the compact capacity


@pytest.mark.parametrize("how", ["numpy", "cuda", "pinned"])
def test_peeksort_compact_overflow_public_api(how):
    """The public entry points retry by themselves (numpy: rs_sort_host_ex; torch: the
    Python shim): output, tags, Metrics and the recorded tree equal the oracle's."""
    import torch

    n, w = 200_000, 2
    a = _zigzag(n, 12).astype(np.int32)
    tags = np.arange(n, dtype=np.int32)
    ref_k, ref_t = a.copy(), tags.copy()
    ref = oracle.peeksort(ref_k, w, "classic", ref_t)
    assert ref.runs_detected > n // 12 + 4096
    cfg = rs.SortConfig(min_run_len=w, merge_kind="classic")
    if how == "numpy":
        k, t = a.copy(), tags.copy()
        m = rs.peeksort(k, cfg, tags=t)
        got_k, got_t = k, t
    else:
        k, t = torch.from_numpy(a.copy()), torch.from_numpy(tags.copy())
        k, t = (k.cuda(), t.cuda()) if how == "cuda" else (k.pin_memory(), t.pin_memory())
        m = rs.peeksort(k, cfg, tags=t)
        got_k, got_t = k.cpu().numpy(), t.cpu().numpy()
    assert np.array_equal(got_k, ref_k) and np.array_equal(got_t, ref_t)
    assert _mt(m)[:3] == ref.metrics_tuple()[:3]


def test_peeksort_compact_overflow_recorded_tree():
    """record_tree after the worst-case retry: the exported tree is the oracle's."""
    import sys

    n, w = 60_000, 2
    a = _zigzag(n, 14).astype(np.int64)
    ref_k = a.copy()
    ref = oracle.peeksort(ref_k, w, "bitonic", want_tree=True)
    assert ref.runs_detected > n // 12 + 4096
    work, _, m = _run(a, w, "bitonic", record=True)
    assert np.array_equal(work, ref_k)
    assert _mt(m)[:3] == ref.metrics_tuple()[:3]
    old = sys.getrecursionlimit()
    sys.setrecursionlimit(10000)
    try:
        assert _shape(m.merge_tree) == oracle.peek_tree_from_merges(n, ref.merges)
    finally:
        sys.setrecursionlimit(old)
