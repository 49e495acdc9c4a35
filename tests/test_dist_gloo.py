"""Multi-rank sharded sort host logic (splitters, exchange, final merge) with
the gloo backend on CPU, world sizes 2 and 3.

The local sorter here is a CPU stable sort standing in for the CUDA powersort
(test scaffolding only); what is tested is paper_1805_04154_b200.dist: the
exact (key, rank, position) splitters and the all-to-all-v exchange.  The
result must equal a stable sort of the concatenated shards, keys and tags.
"""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_1805_04154_b200 import dist as rsd


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _cpu_merge(out, tout, recv):
    """CPU stand-in for the CUDA W-way merge: the received runs in rank order,
    stably merged (a stable sort of their concatenation is that merge)."""
    order = torch.from_numpy(np.argsort(out.numpy(), kind="stable"))
    return out[order], (tout[order] if tout is not None else None)


def _cpu_stable_sort(keys, tags):
    order = torch.from_numpy(np.argsort(keys.numpy(), kind="stable"))
    keys.copy_(keys[order])
    if tags is not None:
        tags.copy_(tags[order])


def _shards(case, W, seed):
    rng = np.random.default_rng(seed)
    out = []
    base = 0
    for i in range(W):
        n = int(rng.integers(0, 3000)) if case != "equal" else 1000
        if case == "dups":
            k = rng.integers(0, 16, size=n)
        elif case == "allsame":
            k = np.full(n, 7)
        elif case == "skew":
            k = rng.integers(-10**9, 10**9, size=n) + (i * 10**9 if i % 2 else 0)
        else:
            k = rng.integers(-50, 50, size=n) * (i + 1)
        out.append((k.astype(np.int64), np.arange(base, base + n, dtype=np.int64)))
        base += n
    return out


CASES = ["dups", "allsame", "skew", "mixed", "equal"]
SAMPLES = (4, 64)


def _worker(rank, W, port, seed, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=W)
    try:
        for case in CASES:
            for samples in SAMPLES:
                k, t = _shards(case, W, seed)[rank]
                keys = torch.from_numpy(k.copy())
                tags = torch.from_numpy(t.copy())
                out, tout, info = rsd.sharded_sort(keys, tags, local_sort=_cpu_stable_sort, samples=samples,
                                                merge=_cpu_merge)
                q.put((case, samples, rank, out.numpy().copy(), tout.numpy().copy()))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("W", [2, 3])
def test_sharded_sort_matches_stable_sort(W):
    seed = 17 + W
    port = _free_port()
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    procs = [ctx.Process(target=_worker, args=(r, W, port, seed, q)) for r in range(W)]
    for p in procs:
        p.start()
    res = {}
    for _ in range(W * len(CASES) * len(SAMPLES)):
        case, samples, r, o, to = q.get(timeout=300)
        res[(case, samples, r)] = (o, to)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    for case in CASES:
        shards = _shards(case, W, seed)
        allk = np.concatenate([s[0] for s in shards])
        allt = np.concatenate([s[1] for s in shards])
        order = np.argsort(allk, kind="stable")
        for samples in SAMPLES:
            gotk = np.concatenate([res[(case, samples, r)][0] for r in range(W)])
            gott = np.concatenate([res[(case, samples, r)][1] for r in range(W)])
            assert np.array_equal(gotk, allk[order]), (case, samples)
            assert np.array_equal(gott, allt[order]), (case, samples)
            for r in range(W):  # each rank keeps its element count
                assert len(res[(case, samples, r)][0]) == len(shards[r][0])
