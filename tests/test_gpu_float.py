"""Floating-point keys on the device path, against fixtures the REFERENCE
produced (tests/golden/make_golden_float.py): negative / positive zeros (equal
as floats: their input order must survive), infinities, subnormals, heavy
duplicates; float16 / float32 / float64 keys, int64 tags, powersort and
peeksort, both merge kinds.  NaN keys are rejected loudly."""
import hashlib
import json
import os

import numpy as np
import pytest

import paper_1805_04154_b200 as rs

pytestmark = pytest.mark.gpu
G = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")


def sha(*arrays):
    h = hashlib.sha256()
    for a in arrays:
        h.update(np.ascontiguousarray(a).tobytes())
    return h.hexdigest()[:24]


def test_float_keys_match_reference_fixtures():
    with open(os.path.join(G, "golden_float.json")) as fh:
        cases = json.load(fh)["cases"]
    arrays = dict(np.load(os.path.join(G, "golden_float_inputs.npz")))
    bad = []
    for c in cases:
        a = arrays[c["input"]].copy()
        t = np.arange(len(a), dtype=np.int64)
        m = rs.SORTERS[c["sorter"]](a, rs.SortConfig(min_run_len=c["w"], merge_kind=c["merge_kind"]), None, t)
        got = (m.merge_cost, m.comparisons, m.runs_detected, m.max_stack_height)
        want = (c["merge_cost"], c["comparisons"], c["runs_detected"], c["max_stack_height"])
        if got != want or sha(a, t) != c["out_sha"]:
            bad.append((c["input"], c["sorter"], c["w"], c["merge_kind"], got, want))
    assert not bad, f"{len(bad)}/{len(cases)} mismatches: {bad[:4]}"


def test_float_cuda_tensor_in_place_and_zero_signs():
    import torch

    rng = np.random.default_rng(3)
    a = rng.integers(-2, 3, size=200000).astype(np.float32)
    z = a == 0
    a[z] = np.where(rng.random(int(z.sum())) < 0.5, -0.0, 0.0)
    want = a[np.argsort(a, kind="stable")]  # numpy's stable order treats -0.0 == 0.0
    d = torch.from_numpy(a.copy()).cuda()
    rs.powersort(d)
    got = d.cpu().numpy()
    assert np.array_equal(got.view(np.uint32), want.view(np.uint32))  # bit patterns, zero signs included


def test_nan_keys_are_rejected_and_input_kept():
    a = np.array([3.0, np.nan, 1.0, 2.0])
    before = a.copy()
    with pytest.raises(NotImplementedError):
        rs.powersort(a)
    assert np.array_equal(a, before, equal_nan=True)
