"""Loader for the reference-generated fixtures in tests/golden (see make_golden.py)."""
import functools
import hashlib
import json
import os

import numpy as np

HERE = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")


@functools.lru_cache(maxsize=1)
def load():
    with open(os.path.join(HERE, "golden.json")) as fh:
        meta = json.load(fh)
    arrays = dict(np.load(os.path.join(HERE, "golden_inputs.npz")))
    return meta, arrays


def sha(*arrays) -> str:
    h = hashlib.sha256()
    for a in arrays:
        h.update(np.ascontiguousarray(a).tobytes())
    return h.hexdigest()[:24]


def case_inputs(case, arrays):
    a = arrays[case["input"]]
    tags = None
    if case["tags"] == "int64" and case["kind"] != "medium":
        tags = np.arange(len(a), dtype=np.int64)
    elif case["tags"] is not None:
        tags = arrays[case["input"] + "__tags"]
    return a, tags


def metrics_of(case):
    return (case["merge_cost"], case["comparisons"], case["runs_detected"], case["max_stack_height"])


def tree_shape(t):
    """Reference tree list -> nested ('L', length) / ('N', l, r) shape."""
    if t is None:
        return None
    if t[0] == "L":
        return ("L", t[2])
    return ("N", tree_shape(t[3]), tree_shape(t[4]))
