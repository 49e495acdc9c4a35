"""Generate the golden fixtures from the REFERENCE implementation.

Run here (the reference is importable only in this container):

    python tests/golden/make_golden.py

It imports the reference package from /root/reference/pkg/src, runs its own
powersort / peeksort / node-power functions on seeded inputs, and commits the
results as small fixtures (golden.json + golden_inputs.npz).  The C oracle
(oracle/runsort_oracle.c) and the CUDA path are both checked against these.

Input shapes follow the reference's own test strategies
(reference tests/test_sorters.py:229-244 `arrays()`, :267-270
`run_length_vectors()`; tests/test_acceptance.py:61-74 `_instances`) plus
BASELINE-shaped inputs at desk size.
"""

from __future__ import annotations

import hashlib
import json
import os
import sys

import numpy as np

REF = "/root/reference/pkg/src"
HERE = os.path.dirname(os.path.abspath(__file__))
REPO = os.path.dirname(os.path.dirname(HERE))
sys.path.insert(0, REF)
sys.path.insert(0, REPO)

from runsort import gen as rgen  # noqa: E402
from runsort.opttree import MergeLeaf  # noqa: E402
from runsort.runcore import Metrics  # noqa: E402
from runsort.sorters import SortConfig, node_power_def, peeksort, powersort  # noqa: E402

from paper_1805_04154_b200 import workloads  # noqa: E402

ALGOS = {"powersort": powersort, "peeksort": peeksort}
WS = [1, 3, 7, 24]
KINDS = ["bitonic", "classic"]


def sha(*arrays) -> str:
    h = hashlib.sha256()
    for a in arrays:
        h.update(np.ascontiguousarray(a).tobytes())
    return h.hexdigest()[:24]


def tree_to_list(t):
    if isinstance(t, MergeLeaf):
        return ["L", int(t.index), int(t.length)]
    return ["N", int(t.size), None if t.power is None else int(t.power),
            tree_to_list(t.left), tree_to_list(t.right)]


def run_ref(algo, a, w, kind, tags=None, record=False):
    work = a.copy()
    tw = tags.copy() if tags is not None else None
    m = Metrics()
    ALGOS[algo](work, SortConfig(min_run_len=w, merge_kind=kind, record_tree=record), m, tw)
    out = dict(merge_cost=int(m.merge_cost), comparisons=int(m.comparisons),
               runs_detected=int(m.runs_detected), max_stack_height=int(m.max_stack_height))
    if record:
        out["tree"] = tree_to_list(m.merge_tree) if m.merge_tree is not None else None
    return work, tw, out


def small_arrays(rng, count):
    """Shapes of the reference's hypothesis strategy, plus mixed-direction runs."""
    out = []
    for n in (0, 1, 2, 3, 4, 5):
        for _ in range(3):
            out.append(("tiny", rng.integers(0, 3, size=n).astype(np.int64)))
    for _ in range(count):
        kind = int(rng.integers(0, 4))
        n = int(rng.integers(0, 401))
        if kind == 0:
            a = rng.permutation(n).astype(np.int64)
        elif kind == 1:
            a = rng.integers(0, max(1, n // 4 + 1), size=n).astype(np.int64)
        elif kind == 2:
            lens, left = [], n
            while left > 0:
                L = min(left, int(rng.integers(1, 20)))
                lens.append(L)
                left -= L
            a = rgen.from_run_lengths(lens) if lens else np.empty(0, dtype=np.int64)
        else:  # alternating ascending / strictly descending segments with ties
            parts, left, k = [], n, 0
            while left > 0:
                L = min(left, int(rng.integers(1, 40)))
                seg = np.sort(rng.integers(0, 50, size=L))
                if k % 2:
                    seg = np.unique(seg)[::-1]
                parts.append(seg)
                left -= len(seg)
                k += 1
            a = np.concatenate(parts).astype(np.int64) if parts else np.empty(0, np.int64)
        out.append((["perm", "dup", "runs", "mixed"][kind], a))
    return out


def main():
    rng = np.random.default_rng(20241019)
    inputs = {}
    cases = []

    # --- A: small arrays, every algo x w x merge kind, with index tags --------
    for idx, (kind, a) in enumerate(small_arrays(rng, 360)):
        key_dtype = "int32" if idx % 3 == 2 else "int64"
        a = a.astype(key_dtype)
        name = f"small{idx}"
        inputs[name] = a
        tags = np.arange(len(a), dtype=np.int64)
        expect_tags = np.argsort(a, kind="stable")
        for algo in ALGOS:
            for w in WS:
                for mk in KINDS:
                    work, tw, met = run_ref(algo, a, w, mk, tags)
                    assert np.array_equal(tw, expect_tags), (name, algo, w, mk)
                    assert np.array_equal(work, a[expect_tags])
                    cases.append(dict(input=name, kind=kind, algo=algo, w=w, merge_kind=mk,
                                      tags="int64", out_sha=sha(work, tw), **met))

    # --- B: recorded trees (reference tests/test_sorters.py:273-286) ----------
    for idx in range(120):
        r = int(rng.integers(1, 40))
        lens = [int(x) for x in rng.integers(2, 30, size=r)]
        if rng.random() < 0.25:
            lens[-1] = 1
        a = rgen.from_run_lengths(lens)
        if idx % 2:
            a = a % (len(a) // 5 + 2)  # ties change the run structure
        name = f"tree{idx}"
        inputs[name] = a
        for algo in ALGOS:
            for w, mk in ((1, "classic"), (24, "bitonic"), (3, "classic")):
                work, _, met = run_ref(algo, a, w, mk, None, record=True)
                cases.append(dict(input=name, kind="tree", algo=algo, w=w, merge_kind=mk,
                                  tags=None, out_sha=sha(work), **met))
    fig = rgen.from_run_lengths([5, 3, 3, 14, 1, 2])
    inputs["fig"] = fig
    for algo in ALGOS:
        for w, mk in ((1, "classic"), (24, "bitonic")):
            work, _, met = run_ref(algo, fig, w, mk, None, record=True)
            cases.append(dict(input="fig", kind="fig", algo=algo, w=w, merge_kind=mk,
                              tags=None, out_sha=sha(work), **met))

    # --- C: desk-size BASELINE-shaped and reference-generator inputs ----------
    medium = {
        "cfg1_2^14": (workloads.config1(1 << 14, 3), None),
        "cfg2_1e5": (workloads.config2(10**5, 3), None),
        "cfg3_2^16": (workloads.config3(1 << 16, 3), None),
        "cfg4_1e5": workloads.config4(10**5, 3),
        "cfg4_small_runs": workloads.config4(30000, 4, mean=40.0),
        "randruns_1e5_100": (rgen.random_runs(10**5, 100, 5), None),
        "perm_5e4": (rgen.random_permutation(50000, 9), None),
        "drag_2^14": (rgen.timsort_drag(1 << 14, run_scale=4), None),
        "dupruns_4e4": (rgen.random_runs(40000, 30, 6) % 97, None),
    }
    for name, (a, tags) in medium.items():
        inputs[name] = a
        if tags is not None:
            inputs[name + "__tags"] = tags
        for algo in ALGOS:
            for w, mk in ((24, "bitonic"), (1, "classic"), (7, "classic")):
                work, tw, met = run_ref(algo, a, w, mk, tags)
                order = np.argsort(a, kind="stable")
                assert np.array_equal(work, a[order])
                if tags is not None:
                    assert np.array_equal(tw, tags[order])
                cases.append(dict(input=name, kind="medium", algo=algo, w=w, merge_kind=mk,
                                  tags=None if tags is None else str(tags.dtype),
                                  out_sha=sha(work) if tags is None else sha(work, tw), **met))

    # --- D: node powers (reference sorters.py:376-392, tests :117-125) --------
    powers = []
    for args in ((1, 5, 6, 8, 28), (9, 11, 12, 25, 28), (1, 1, 2, 2, 2), (26, 26, 27, 28, 28)):
        powers.append(list(args) + [node_power_def(*args)])
    for _ in range(3000):
        n = int(rng.choice([int(rng.integers(2, 200)), int(rng.integers(2, 1 << 31)),
                            int(rng.integers(1 << 31, 1 << 40))]))
        s1 = int(rng.integers(1, n))
        e1 = int(rng.integers(s1, n))
        s2 = e1 + 1
        e2 = int(rng.integers(s2, n + 1))
        powers.append([s1, e1, s2, e2, n, node_power_def(s1, e1, s2, e2, n)])

    np.savez_compressed(os.path.join(HERE, "golden_inputs.npz"), **inputs)
    with open(os.path.join(HERE, "golden.json"), "w") as fh:
        json.dump(dict(source="reference runsort @ /root/reference/pkg/src (make_golden.py)",
                       cases=cases, node_powers=powers), fh, separators=(",", ":"))
    print(f"{len(cases)} sorter cases, {len(powers)} node-power tuples, {len(inputs)} inputs")


if __name__ == "__main__":
    main()
