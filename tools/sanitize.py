"""Small sorts through the C ABI (rs_sort_host_ex, no torch) for compute-sanitizer.

usage: compute-sanitizer --tool racecheck python tools/sanitize.py
Each case is checked against the C oracle so a sanitizer-clean run is also a
correct one.  Sizes are small: racecheck/synccheck instrument every shared
memory access and run ~100x slower.
"""
import ctypes
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from oracle import oracle  # noqa: E402  (checker only)
from paper_1805_04154_b200 import _lib, workloads  # noqa: E402


def run(algo, keys, tags, w, kind):
    L = _lib.lib()
    out = _lib.RsMetrics()
    code = _lib.RS_KEY_I32 if keys.dtype == np.int32 else _lib.RS_KEY_I64
    k = _lib.RS_MERGE_CLASSIC if kind == "classic" else _lib.RS_MERGE_BITONIC
    _lib.check(L.rs_sort_host_ex(algo, code, keys.ctypes.data, tags.dtype.itemsize if tags is not None else 0,
                                 tags.ctypes.data if tags is not None else None, len(keys), w, k, 2.0,
                                 ctypes.byref(out), None))
    return (out.merge_cost, out.comparisons, out.runs_detected, out.max_stack_height)


def main():
    n = int(os.environ.get("RS_SAN_N", "200000"))
    cases = 0
    for algo_name, algo in (("powersort", _lib.RS_ALGO_POWERSORT), ("peeksort", _lib.RS_ALGO_PEEKSORT)):
        for w in (1, 24):
            for dt, tdt in ((np.int32, None), (np.int64, np.int64), (np.int32, np.int32)):
                for gen in ("runs", "small"):
                    if gen == "runs":
                        keys, _ = workloads.config4(n, seed=11 + w, mean=40.0)
                        keys = keys.astype(dt)
                    else:
                        rng = np.random.default_rng(5 + w)
                        keys = rng.integers(0, 50, size=n // 7, dtype=dt)
                    tags = None if tdt is None else np.arange(len(keys), dtype=tdt)
                    rk = keys.copy()
                    rt = None if tags is None else tags.copy()
                    kind = "classic" if w == 1 else "bitonic"
                    if algo_name == "powersort":
                        ref = oracle.powersort(rk, w, kind, rt)
                    else:
                        ref = oracle.peeksort(rk, w, kind, rt)
                    got = run(algo, keys, tags, w, kind)
                    ok = np.array_equal(keys, rk) and (tags is None or np.array_equal(tags, rt)) \
                        and got == ref.metrics_tuple()
                    print(f"{algo_name} w={w} keys={np.dtype(dt).name} tags={tdt and np.dtype(tdt).name} "
                          f"gen={gen} n={len(keys)} ok={ok}", flush=True)
                    assert ok
                    cases += 1
    print(f"sanitize: {cases} cases ok")


if __name__ == "__main__":
    main()
