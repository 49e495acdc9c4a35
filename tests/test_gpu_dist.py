"""The sharded (multi-GPU) sort on B200s.

* world size 1 over NCCL: CUDA powersort of the shard, splitters, all-to-all-v,
  the CUDA W-way merge (trivially W = 1);
* the NVLink data plane (P2PShardSpace + sharded_sort_p2p) at world size 2:
  on a box with >= 2 GPUs one rank per GPU over NCCL; on a one-GPU box two
  processes share the GPU (gloo for the host plumbing, CUDA IPC mapping the
  other process's shard buffer).  No kernel waits on another process: the
  ranks only meet at host barriers, and every kernel reads buffers that are
  complete.  The concatenated slices must equal the stable sort of the
  concatenated shards, keys and payloads.
"""
import os
import socket

import numpy as np
import pytest

pytestmark = pytest.mark.gpu


def _port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def test_sharded_sort_world1_nccl():
    import torch
    import torch.distributed as dist

    from paper_1805_04154_b200 import dist as rsd
    from paper_1805_04154_b200 import workloads

    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(_port()), RANK="0", WORLD_SIZE="1")
    dist.init_process_group("nccl")
    try:
        k, t = workloads.config4(200000, seed=3, mean=100.0)
        keys = torch.from_numpy(k.copy()).cuda()
        tags = torch.from_numpy(t.copy()).cuda()
        out, tout, info = rsd.sharded_sort(keys, tags)
        order = np.argsort(k, kind="stable")
        assert np.array_equal(out.cpu().numpy(), k[order])
        assert np.array_equal(tout.cpu().numpy(), t[order])
    finally:
        dist.destroy_process_group()


def _shard(rank, W, case):
    rng = np.random.default_rng(1000 + 17 * rank + case)
    n = [120000, 0, 77777, 5][case % 4] + 31 * rank
    if case % 2:
        k = rng.integers(0, 8, n)
    else:
        k = rng.integers(-(1 << 40), 1 << 40, n)
    base = sum([120000, 0, 77777, 5][case % 4] + 31 * r for r in range(rank))
    return k.astype(np.int64), np.arange(base, base + n, dtype=np.int64)


def _p2p_worker(rank, W, port, backend, q):
    import torch
    import torch.distributed as dist

    from paper_1805_04154_b200 import dist as rsd

    ndev = torch.cuda.device_count()
    torch.cuda.set_device(rank % ndev)
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group(backend, rank=rank, world_size=W)
    try:
        space = rsd.P2PShardSpace(200000, torch.int64, torch.int64)
        for case in range(4):
            k, t = _shard(rank, W, case)
            space.keys[: len(k)].copy_(torch.from_numpy(k))
            space.tags[: len(t)].copy_(torch.from_numpy(t))
            out, tout, info = rsd.sharded_sort_p2p(space, len(k))
            q.put((case, rank, out.cpu().numpy().copy(), tout.cpu().numpy().copy()))
        space.close()
    finally:
        dist.destroy_process_group()


def test_p2p_world2():
    import torch
    import torch.multiprocessing as mp

    W = 2
    backend = "nccl" if torch.cuda.device_count() >= 2 else "gloo"
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _port()
    procs = [ctx.Process(target=_p2p_worker, args=(r, W, port, backend, q)) for r in range(W)]
    for p in procs:
        p.start()
    res = {}
    for _ in range(W * 4):
        case, r, o, to = q.get(timeout=600)
        res[(case, r)] = (o, to)
    for p in procs:
        p.join(timeout=120)
        assert p.exitcode == 0
    for case in range(4):
        sh = [_shard(r, W, case) for r in range(W)]
        allk = np.concatenate([s[0] for s in sh])
        allt = np.concatenate([s[1] for s in sh])
        order = np.argsort(allk, kind="stable")
        assert np.array_equal(np.concatenate([res[(case, r)][0] for r in range(W)]), allk[order]), case
        assert np.array_equal(np.concatenate([res[(case, r)][1] for r in range(W)]), allt[order]), case


def test_p2p_world1_nccl_stream_ordered():
    """The NCCL flavour of the NVLink plane (stream-ordered barriers, device
    co-rank) at world size 1, plus sort_async's deferred Metrics."""
    import torch
    import torch.distributed as dist

    from oracle import oracle
    from paper_1805_04154_b200 import dist as rsd
    from paper_1805_04154_b200 import workloads

    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(_port()), RANK="0", WORLD_SIZE="1")
    dist.init_process_group("nccl", device_id=torch.device("cuda", 0))
    try:
        space = rsd.P2PShardSpace(300000, torch.int32, torch.int32)
        for seed in (1, 2):
            k, t = workloads.config4(250000 + seed, seed=seed, mean=300.0)
            space.keys[: len(k)].copy_(torch.from_numpy(k))
            space.tags[: len(t)].copy_(torch.from_numpy(t))
            out, tout, info = rsd.sharded_sort_p2p(space, len(k))
            rk, rt = k.copy(), t.copy()
            ref = oracle.powersort(rk, 24, "bitonic", rt)
            assert np.array_equal(out.cpu().numpy(), rk)
            assert np.array_equal(tout.cpu().numpy(), rt)
            m = info["local"].metrics()
            assert (m.merge_cost, m.comparisons, m.runs_detected, m.max_stack_height) == ref.metrics_tuple()
        space.close()
    finally:
        dist.destroy_process_group()
