"""The device algorithm (tests/device_model.py) reproduces the oracle exactly.

This validates the math the CUDA kernels rely on -- tile-table min-run chain,
32-bit midpoint powers, trie ranges, depth = la + ra via (mask, const) scans,
depth-parity ping-pong -- on CPU, before any kernel runs.
"""
import numpy as np

from oracle import oracle
from tests import device_model as DM
from tests import golden_data as G


def test_model_matches_oracle_on_golden_small():
    meta, arrays = G.load()
    seen = set()
    for case in meta["cases"]:
        if case["algo"] != "powersort" or case["kind"] == "medium":
            continue
        key = (case["input"], case["w"], case["merge_kind"])
        if key in seen or len(seen) > 1500:
            continue
        seen.add(key)
        a, tags = G.case_inputs(case, arrays)
        out, tout, met, starts, P = DM.simulate(a, case["w"], case["merge_kind"], tags, T=16)
        assert met == G.metrics_of(case), key
        order = np.argsort(a, kind="stable")
        assert np.array_equal(out, a[order])
        if tags is not None:
            assert np.array_equal(tout, tags[order])


def test_model_matches_oracle_medium():
    meta, arrays = G.load()
    a = arrays["cfg4_small_runs"][:6000]
    t = arrays["cfg4_small_runs__tags"][:6000]
    for w, mk in ((24, "bitonic"), (1, "classic"), (7, "classic")):
        ref = oracle.powersort(a.copy(), w, mk, t.copy(), want_tree=True)
        out, tout, met, starts, P = DM.simulate(a, w, mk, t, T=256)
        assert met == ref.metrics_tuple()
        assert list(starts) == list(ref.leaf_starts)
        assert list(P) == list(ref.powers)
