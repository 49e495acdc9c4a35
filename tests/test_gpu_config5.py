"""BASELINE config 5 on one GPU, bit-exact: n = 2^31 int64 keys (generated on the
device), powersort through the public API.

n = 2^31 is exactly where the reference switches node-power arithmetic from
31-bit fixed point to the definitional loop (reference sorters.py:416-423 ->
:376-392), so this is the one config whose powers the smaller configs do not
cover.  The checks:

* output: equal, element for element, to torch's own sort of a copy (two
  halves sorted by ``torch.sort``, merged by rank; keys only, so any correct
  sort is the reference's output);
* Metrics: all four counters equal the analytic oracle (``oracle/analytic.py``,
  a restatement of sorters.py:430-519 over the run structure of the ORIGINAL
  array, with node powers from the reference's ``node_power_def`` loop);
* the exported merge tree: every leaf length and every node power (in-order)
  equals the oracle's, i.e. each device power equals node_power_def.

The same machinery is cross-checked against the element-by-element C oracle on
a config-5-shaped array of 2^22 keys first (test_config5_shape_small).
"""
import numpy as np
import pytest

pytestmark = [pytest.mark.gpu]


def _analytic_from_device(a, w=24):
    """Analytic Metrics of reference powersort for the device array `a`
    (computed before the in-place sort; only small pieces come to the host)."""
    import torch

    from oracle import analytic

    n = int(a.numel())
    asc = a[:-1] <= a[1:]
    k = torch.nonzero(asc[1:] != asc[:-1]).flatten() + 1
    bounds = torch.cat([k, torch.tensor([n - 1], device=a.device)]).cpu().numpy()
    del k

    def asc_at(pos):
        return asc[torch.from_numpy(np.asarray(pos, dtype=np.int64)).to(a.device)].cpu().numpy()

    def window(lo, hi):
        return a[lo: hi + 1].cpu().numpy()

    res = analytic.powersort_metrics(n, w, bounds, asc_at, window)
    del asc
    return res


def _reference_sorted(a):
    """torch's own sort of a copy (independent of this repo's kernels).
    torch.sort handles at most INT_MAX elements per call, so the two halves are
    sorted by torch and placed by rank: h1[i] goes to i + #(h2 < h1[i]), h2[j]
    to j + #(h1 <= h2[j]) (a stable two-way merge by searchsorted)."""
    import torch

    n = a.numel()
    h = n // 2
    h1 = torch.sort(a[:h].clone()).values
    h2 = torch.sort(a[h:].clone()).values
    torch.cuda.empty_cache()
    ref = torch.empty_like(a)
    pos = torch.searchsorted(h2, h1, right=False)
    pos += torch.arange(h, device=a.device)
    ref[pos] = h1
    del pos
    pos = torch.searchsorted(h1, h2, right=True)
    pos += torch.arange(n - h, device=a.device)
    ref[pos] = h2
    del pos, h1, h2
    torch.cuda.empty_cache()
    return ref


def _check_against(a, res, m):
    from paper_1805_04154_b200 import MergeLeaf, internal_nodes_inorder

    got = (m.merge_cost, m.comparisons, m.runs_detected, m.max_stack_height)
    want = (res["merge_cost"], res["comparisons"], res["runs_detected"], res["max_stack_height"])
    assert got == want, (got, want)
    t = m.merge_tree
    nodes = internal_nodes_inorder(t)
    powers = np.asarray([x.power for x in nodes], dtype=np.int64)
    assert np.array_equal(powers, res["powers"])
    leaves = []
    todo = [t]
    while todo:
        x = todo.pop()
        if isinstance(x, MergeLeaf):
            leaves.append(x.length)
        else:
            todo.append(x.right)
            todo.append(x.left)
    assert np.array_equal(np.asarray(leaves, dtype=np.int64), res["leaf_lengths"])


def test_config5_shape_small():
    """Config-5-shaped array at 2^22: analytic oracle == C oracle == device."""
    import torch

    import paper_1805_04154_b200 as rs
    from oracle import oracle
    from paper_1805_04154_b200 import workloads

    n = 1 << 22
    a = workloads.config5_device(n, seed=3, mean=float(1 << 10))
    host = a.cpu().numpy().copy()
    res = _analytic_from_device(a)
    ref = oracle.powersort(host, 24, "bitonic", want_tree=True)
    assert (res["merge_cost"], res["comparisons"], res["runs_detected"], res["max_stack_height"]) == \
        ref.metrics_tuple()
    assert np.array_equal(res["powers"], ref.powers)
    m = rs.powersort(a, rs.SortConfig(record_tree=True))
    torch.cuda.synchronize()
    assert np.array_equal(a.cpu().numpy(), host)
    _check_against(a, res, m)


@pytest.mark.slow
def test_config5_full_size_bit_exact():
    import torch

    import paper_1805_04154_b200 as rs
    from paper_1805_04154_b200 import workloads

    torch.cuda.empty_cache()
    free, _ = torch.cuda.mem_get_info()
    if free < 120 * (1 << 30):
        pytest.skip("needs ~120 GB of free device memory")
    n = workloads.CONFIG5_N
    assert n == 1 << 31
    a = workloads.config5_device(n, seed=1)
    res = _analytic_from_device(a)
    assert res["runs_detected"] > 30000
    ref = _reference_sorted(a)
    m = rs.powersort(a, rs.SortConfig(record_tree=True))
    torch.cuda.synchronize()
    assert torch.equal(a, ref)
    del ref
    _check_against(a, res, m)


@pytest.mark.slow
def test_above_2_31_int32_bit_exact():
    """n = 2^31 + 3*2^20 + 7 int32 keys: above 2^31 the device's node powers
    take the 63-bit midpoint-key path (128-bit division) and 64-bit positions
    with 32-bit keys; the reference takes node_power_def (sorters.py:416-423).
    Output vs torch's sort, all Metrics and every node power vs the analytic
    oracle, as for config 5."""
    import torch

    import paper_1805_04154_b200 as rs
    from paper_1805_04154_b200 import workloads

    torch.cuda.empty_cache()  # blocks cached by the tests before
    free, _ = torch.cuda.mem_get_info()
    if free < 110 * (1 << 30):
        pytest.skip("needs ~110 GB of free device memory")
    n = (1 << 31) + 3 * (1 << 20) + 7
    a64 = workloads.config5_device(n, seed=5, mean=float(1 << 15))
    a = (a64 >> 33).to(torch.int32)  # monotone: the sorted segments stay sorted, with many ties
    del a64
    torch.cuda.empty_cache()
    res = _analytic_from_device(a)
    ref = _reference_sorted(a)
    m = rs.powersort(a, rs.SortConfig(record_tree=True))
    torch.cuda.synchronize()
    assert torch.equal(a, ref)
    del ref
    _check_against(a, res, m)
