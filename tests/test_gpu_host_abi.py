"""The reference-side binding (Option 2) and concurrency.

* ``rs_sort_host`` through the EXACT ctypes binding INTEGRATION.md shows a
  maintainer adding to the reference package: the code block is read out of
  INTEGRATION.md and executed verbatim (only the library name becomes this
  tree's path), then driven with numpy int32/int64 arrays like the reference's
  callers do (sorters.py:430-450): every golden powersort fixture and BASELINE
  configs 1-4 at full size, keys + tags + Metrics vs the oracle.
* Reentrancy (reference runcore.py:17-18): four host threads, each
  on its own CUDA stream with its own min_run_len, sort concurrently through
  the public API; every result equals the oracle's.
"""
import os
import re
import threading

import numpy as np
import pytest

import paper_1805_04154_b200 as rs
from oracle import oracle
from paper_1805_04154_b200 import _lib, workloads
from tests import golden_data as G

REPO = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def option2_binding_source():
    with open(os.path.join(REPO, "INTEGRATION.md")) as fh:
        doc = fh.read()
    sec = doc[doc.index("## Option 2"):]
    return re.search(r"```python\n(.*?)```", sec, re.S).group(1)


def test_option2_block_binds_rs_sort_host():
    """CPU: the documented binding names the symbol and signature the header declares."""
    src = option2_binding_source()
    assert "rs_sort_host" in src and "rs_last_error" in src
    with open(os.path.join(REPO, "include", "runsort_b200.h")) as fh:
        hdr = fh.read()
    assert re.search(r"int rs_sort_host\(int algo, int key_dtype, void\* keys, int tag_bytes, void\* tags, "
                     r"int64_t n,\s*int32_t min_run_len, int32_t merge_kind, rs_metrics\* out, rs_tree\* tree\)",
                     hdr)


@pytest.fixture(scope="module")
def b200():
    src = option2_binding_source().replace('"librunsort_b200.so"', repr(_lib.LIB_PATH))
    ns = {}
    exec(compile(src, "INTEGRATION.md:Option2", "exec"), ns)
    return ns["powersort_b200"]


def _mt(m):
    return (m.merge_cost, m.comparisons, m.runs_detected, m.max_stack_height)


@pytest.mark.gpu
def test_option2_binding_golden(b200):
    meta, arrays = G.load()
    bad, count = [], 0
    for case in meta["cases"]:
        if case["algo"] != "powersort":
            continue
        a, tags = G.case_inputs(case, arrays)
        if a.dtype not in (np.int32, np.int64) or len(a) <= 1:
            continue
        work = np.ascontiguousarray(a.copy())
        tw = None if tags is None else np.ascontiguousarray(tags.copy())
        m = b200(work, rs.SortConfig(min_run_len=case["w"], merge_kind=case["merge_kind"]), rs.Metrics(), tw)
        got = G.sha(work) if tw is None else G.sha(work, tw)
        if _mt(m) != G.metrics_of(case) or got != case["out_sha"]:
            bad.append((case["input"], case["w"], case["merge_kind"]))
        count += 1
    assert count > 100
    assert not bad, f"{len(bad)}/{count} mismatches: {bad[:4]}"


@pytest.mark.gpu
def test_rs_sort_host_status_codes():
    a = np.arange(100, dtype=np.int32)
    with pytest.raises(ValueError):
        _raw_host(a, w=0)
    with pytest.raises(NotImplementedError):
        _raw_host(a, w=1 << 20)
    assert np.array_equal(a, np.arange(100, dtype=np.int32))


def _raw_host(a, w):
    import ctypes

    L = _lib.lib()
    m = _lib.RsMetrics()
    rc = L.rs_sort_host(0, _lib.RS_KEY_I32, a.ctypes.data, 0, None, len(a), w, 0, ctypes.byref(m), None)
    _lib.check(rc)


@pytest.mark.gpu
@pytest.mark.slow
@pytest.mark.parametrize("cfg", [1, 2, 3, 4])
def test_option2_binding_configs_full_size(b200, cfg):
    a, tags = workloads.generate(cfg)
    ref_a, ref_t = a.copy(), None if tags is None else tags.copy()
    ref = oracle.powersort(ref_a, 24, "bitonic", ref_t)
    m = b200(a, rs.SortConfig(), rs.Metrics(), tags)
    assert np.array_equal(a, ref_a)
    if tags is not None:
        assert np.array_equal(tags, ref_t)
    assert _mt(m) == ref.metrics_tuple()


@pytest.mark.gpu
def test_concurrent_sorts_on_four_threads():
    import torch

    cases = []
    for i, (w, kind, dt) in enumerate([(1, "bitonic", np.int32), (24, "classic", np.int64),
                                       (7, "bitonic", np.int64), (100, "classic", np.int32)]):
        keys, tags = workloads.config4(300_000 + 77_777 * i, seed=20 + i, mean=40.0 + 100 * i)
        keys = (keys.astype(np.int64) * 1_000_003 + i).astype(dt)
        ref_k, ref_t = keys.copy(), tags.copy()
        ref = oracle.powersort(ref_k, w, kind, ref_t)
        cases.append((keys, tags, w, kind, ref_k, ref_t, ref.metrics_tuple()))
    errors = []

    def worker(idx):
        try:
            keys, tags, w, kind, ref_k, ref_t, ref_m = cases[idx]
            s = torch.cuda.Stream()
            with torch.cuda.stream(s):
                for rep in range(6):
                    dk = torch.from_numpy(keys).cuda()
                    dtg = torch.from_numpy(tags).cuda()
                    m = rs.powersort(dk, rs.SortConfig(min_run_len=w, merge_kind=kind), tags=dtg)
                    s.synchronize()
                    if not (np.array_equal(dk.cpu().numpy(), ref_k) and np.array_equal(dtg.cpu().numpy(), ref_t)
                            and _mt(m) == ref_m):
                        errors.append((idx, rep))
        except Exception as e:  # noqa: BLE001
            errors.append((idx, repr(e)))

    threads = [threading.Thread(target=worker, args=(i,)) for i in range(4)]
    for t in threads:
        t.start()
    for t in threads:
        t.join()
    assert not errors, errors


@pytest.mark.gpu
def test_tensor_on_other_device_rejected_or_sorted_on_its_device():
    import torch

    if torch.cuda.device_count() < 2:
        pytest.skip("needs two CUDA devices")
    a = torch.randint(0, 1000, (100000,), device="cuda:1", dtype=torch.int64)
    ref = torch.sort(a.clone(), stable=True).values
    with torch.cuda.device(0):
        rs.powersort(a)
    assert torch.equal(a, ref)
    with pytest.raises(ValueError):
        rs.powersort(a, tags=torch.arange(100000, device="cuda:0"))
