"""Differential fuzz on the GPU: random run structures, sizes, key/tag types, min_run_len and
merge kinds through the public API (numpy and CUDA-tensor inputs), every case compared with
the C oracle on keys, tags and all Metrics.  Test tooling (uses oracle/).

usage: python tools/fuzz.py --seconds 240 --seed 1
"""
import argparse, sys, time
sys.path.insert(0, '.')
import numpy as np
import torch
import paper_1805_04154_b200 as rs
from oracle import oracle

ap = argparse.ArgumentParser()
ap.add_argument('--seconds', type=float, default=120)
ap.add_argument('--seed', type=int, default=1)
ap.add_argument('--max-n', type=int, default=3_000_000)
a = ap.parse_args()
rng = np.random.default_rng(a.seed)


def make(n):
    """Concatenated runs: lengths from a random law, directions mixed, value range random."""
    law = rng.integers(0, 5)
    if law == 0:
        mean = float(rng.choice([2, 5, 30, 300, 3000, 50000]))
        lens = rng.geometric(1.0 / mean, size=max(4, int(2 * n / mean) + 4))
    elif law == 1:
        lens = np.minimum(rng.zipf(1.3, size=n // 2 + 4), max(2, n // 3))
    elif law == 2:
        lens = rng.integers(1, max(2, int(rng.choice([3, 25, 40, 5000]))), size=n + 4)
    elif law == 3:
        lens = np.full(n // 30 + 4, 30)
    else:
        lens = np.array([n])
    hi = int(rng.choice([2, 16, 1 << 10, 1 << 30]))
    keys = rng.integers(0, hi, size=n, dtype=np.int64)
    pos = 0
    pdesc = float(rng.choice([0.0, 0.1, 0.5]))
    for L in lens:
        if pos >= n:
            break
        e = min(n, pos + int(L))
        seg = np.sort(keys[pos:e])
        keys[pos:e] = seg[::-1] if rng.random() < pdesc else seg
        pos = e
    return keys


t0 = time.time()
cases = fails = 0
while time.time() - t0 < a.seconds:
    n = int(rng.choice([rng.integers(2, 300), rng.integers(300, 20000), rng.integers(20000, 400000),
                        rng.integers(400000, a.max_n)]))
    kd = rng.choice([np.int32, np.int64])
    keys = make(n).astype(kd)
    td = rng.choice([None, np.int32, np.int64])
    tags = np.arange(n, dtype=td) if td is not None else None
    w = int(rng.choice([1, 2, 3, 7, 24, 24, 24, 32, 33, 100, 500]))
    mk = str(rng.choice(["bitonic", "classic"]))
    algo = str(rng.choice(["powersort", "powersort", "peeksort"]))
    how = str(rng.choice(["numpy", "cuda"]))
    rk, rt = keys.copy(), (tags.copy() if tags is not None else None)
    ref = getattr(oracle, algo)(rk, w, mk, rt)
    cfg = rs.SortConfig(min_run_len=w, merge_kind=mk)
    fn = getattr(rs, algo)
    if how == "numpy":
        k, t = keys.copy(), (tags.copy() if tags is not None else None)
        m = fn(k, cfg, tags=t)
        gk, gt = k, t
    else:
        k = torch.from_numpy(keys.copy()).cuda()
        t = torch.from_numpy(tags.copy()).cuda() if tags is not None else None
        m = fn(k, cfg, tags=t)
        gk, gt = k.cpu().numpy(), (t.cpu().numpy() if t is not None else None)
    got = (m.merge_cost, m.comparisons, m.runs_detected, m.max_stack_height)
    exp = ref.metrics_tuple()
    if algo == "peeksort":
        got, exp = got[:3], exp[:3]
    ok = np.array_equal(gk, rk) and (gt is None or np.array_equal(gt, rt)) and got == exp
    cases += 1
    if not ok:
        fails += 1
        print("MISMATCH", dict(n=n, kd=kd.__name__, td=getattr(td, '__name__', None), w=w, mk=mk, algo=algo, how=how,
                               got=got, exp=exp), flush=True)
print(f"fuzz seed {a.seed}: {cases} cases in {time.time() - t0:.0f} s, {fails} mismatches")
