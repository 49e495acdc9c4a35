"""Arrays that span GPUs: per-GPU powersort on contiguous shards, then an exact
splitter-partitioned exchange and a stable merge.

Global order = the reference's stable order of the concatenated array, i.e.
(key, shard rank, position in shard).  Each rank ends with the same number of
elements it started with, holding the next contiguous slice of the globally
sorted array.

Splitters (exact, two all-gathers, independent of key duplicates):
  1. every rank publishes S regular samples of its sorted shard as
     (key, rank, position) triples;
  2. for every target boundary t_g every rank derives, from the samples alone,
     a bracket [lo_g, hi_g) of triples that must contain the t_g-th element,
     counts exactly how many of its elements precede lo_g / hi_g, and
     publishes its elements inside the bracket (<= 2*ceil(n_i/S)+2 of them);
  3. every rank merges the published candidates and derives the same split
     matrix c[g][i] (elements of shard i among the first t_g).
Exchange: one all-to-all-v of keys (and tags); the received W sorted runs are
concatenated in rank order and stably merged by the same powersort path
(its leaves are the received runs, ties go to the lower rank).

The local sorter is a parameter so the host logic can be exercised with the
gloo backend on CPU (tests/test_dist_gloo.py); the product path passes the
CUDA powersort.
"""
from __future__ import annotations

import time
from typing import Callable, List, Optional, Sequence, Tuple

import numpy as np

SAMPLES = 1024


def _dist():
    import torch.distributed as dist

    return dist


# --------------------------------------------------------------- triples ----
def _count_below(keys, rank_i: int, trip: Tuple[int, int, int]) -> int:
    """#elements of shard `rank_i` (sorted `keys`) that precede triple (k, r, p)
    in (key, rank, position) order."""
    import torch

    k, r, p = trip
    kt = torch.tensor([k], dtype=keys.dtype, device=keys.device)
    if rank_i < r:
        return int(torch.searchsorted(keys, kt, right=True).item())
    if rank_i > r:
        return int(torch.searchsorted(keys, kt, right=False).item())
    return int(p)


def _count_below_many(keys, rank_i: int, trips) -> np.ndarray:
    """_count_below for many triples with one device search and one copy back."""
    import torch

    k = torch.tensor([t[0] for t in trips], dtype=torch.int64).to(keys.device).to(keys.dtype)
    r = np.asarray([t[1] for t in trips], dtype=np.int64)
    p = np.asarray([t[2] for t in trips], dtype=np.int64)
    le = torch.searchsorted(keys, k, right=True)
    lt = torch.searchsorted(keys, k, right=False)
    both = torch.stack([le, lt]).cpu().numpy().astype(np.int64)
    return np.where(rank_i < r, both[0], np.where(rank_i > r, both[1], p))


def compute_splits(keys, group=None, samples: int = SAMPLES) -> np.ndarray:
    """Exact split matrix for the locally sorted shard `keys` (torch tensor).

    Returns c with shape (W+1, W): c[g][i] = number of elements of shard i among
    the first T_g elements of the global stable order, T_g = n_0 + ... + n_{g-1}.
    Identical on every rank.
    """
    import torch

    dist = _dist()
    W = dist.get_world_size(group)
    rank = dist.get_rank(group)
    dev = keys.device
    S = samples
    if W == 1:
        return np.asarray([[0], [int(keys.shape[0])]], dtype=np.int64)
    # round 1 (one collective, one host copy): every rank publishes its length
    # and S regular samples of its sorted shard; positions are implicit
    n_mine = int(keys.shape[0])
    pos_np = (np.arange(S, dtype=np.int64) * n_mine) // S
    pack = torch.zeros(S + 1, dtype=torch.int64, device=dev)
    pack[0] = n_mine
    if n_mine:
        pack[1:] = keys[torch.from_numpy(pos_np).to(dev)].to(torch.int64)
    gathered = [torch.empty_like(pack) for _ in range(W)]
    dist.all_gather(gathered, pack, group=group)
    g = torch.stack(gathered).cpu().numpy()  # (W, S + 1)
    ns = [int(x) for x in g[:, 0]]
    T = np.concatenate([[0], np.cumsum(ns)]).astype(np.int64)
    rows = []
    for i in range(W):
        if ns[i] == 0:
            continue
        pi = (np.arange(S, dtype=np.int64) * ns[i]) // S
        rows.append(np.stack([g[i, 1:], np.full(S, i, dtype=np.int64), pi, np.ones(S, dtype=np.int64)], axis=1))
    samp = np.concatenate(rows) if rows else np.zeros((0, 4), dtype=np.int64)
    # one sample per distinct (rank, position); sort by (key, rank, position)
    _, uidx = np.unique(samp[:, 1] * (1 << 40) + samp[:, 2], return_index=True)
    samp = samp[uidx]
    samp = samp[np.lexsort((samp[:, 2], samp[:, 1], samp[:, 0]))]
    m = len(samp)
    # Bounds on each sample's global rank from the samples alone: if c samples
    # of shard i precede it, #(shard i before it) is in [P_i[c-1]+1, P_i[c]]
    # (P_i = shard i's sample positions, P_i[-1] = -1, P_i[len] = n_i).
    lb = np.zeros(m, dtype=np.int64)
    ub = np.zeros(m, dtype=np.int64)
    for i in range(W):
        mine = samp[:, 1] == i
        Pi = np.sort(samp[mine, 2])
        c = np.cumsum(mine) - mine  # samples of shard i strictly before each sample
        lo_pos = np.where(c > 0, Pi[np.maximum(c - 1, 0)] if len(Pi) else 0, -1)
        hi_pos = np.where(c < len(Pi), Pi[np.minimum(c, max(len(Pi) - 1, 0))] if len(Pi) else 0, ns[i])
        lb += lo_pos + 1
        ub += hi_pos

    splits = np.zeros((W + 1, W), dtype=np.int64)
    splits[W] = np.asarray(ns, dtype=np.int64)
    targets = [int(T[g]) for g in range(1, W)]
    lo_trip, hi_trip = [], []
    for t in targets:
        le = np.nonzero(ub <= t)[0]
        ge = np.nonzero(lb >= t)[0]
        lo_trip.append(tuple(int(v) for v in samp[le[-1], :3]) if len(le) else None)
        hi_trip.append(tuple(int(v) for v in samp[ge[0], :3]) if len(ge) else None)

    # round 2: exact counts below the bracket ends; round 3: candidates
    G = len(targets)
    a = np.zeros(G, dtype=np.int64)
    b = np.full(G, ns[rank], dtype=np.int64)
    # all bracket ends counted in one device search (one host sync, not 2(W-1))
    ends = [(gi, 0, t) for gi, t in enumerate(lo_trip) if t is not None] + \
           [(gi, 1, t) for gi, t in enumerate(hi_trip) if t is not None]
    if ends:
        counts = _count_below_many(keys, rank, [t for _, _, t in ends])
        for (gi, side, _), c in zip(ends, counts):
            if side == 0:
                a[gi] = c
            else:
                b[gi] = c
    b = np.maximum(a, b)
    meta = torch.tensor(np.stack([a, b], axis=1) if G else np.zeros((0, 2), np.int64), dtype=torch.int64,
                        device=dev)
    metas = [torch.zeros_like(meta) for _ in range(W)]
    if G:
        dist.all_gather(metas, meta, group=group)
    metas = list(torch.stack(metas).cpu().numpy()) if G else [np.zeros((0, 2), np.int64)] * W
    M = max([1] + [int((mt[:, 1] - mt[:, 0]).max()) for mt in metas if len(mt)])
    cand = torch.zeros((G, M), dtype=torch.int64, device=dev)
    for gi in range(G):
        cnt = int(b[gi] - a[gi])
        if cnt:
            cand[gi, :cnt] = keys[int(a[gi]) : int(b[gi])].to(torch.int64)
    cands = [torch.zeros_like(cand) for _ in range(W)]
    if G:
        dist.all_gather(cands, cand, group=group)
    cands = list(torch.stack(cands).cpu().numpy()) if G else [np.zeros((0, M), np.int64)] * W
    for gi, t in enumerate(targets):
        base = sum(int(metas[i][gi, 0]) for i in range(W))
        need = t - base
        # stable merge of the candidate lists by (key, rank, position)
        ks, rs = [], []
        for i in range(W):
            c = int(metas[i][gi, 1] - metas[i][gi, 0])
            ks.append(cands[i][gi, :c])
            rs.append(np.full(c, i, dtype=np.int64))
        kk = np.concatenate(ks) if ks else np.zeros(0, dtype=np.int64)
        rr = np.concatenate(rs) if rs else np.zeros(0, dtype=np.int64)
        order = np.lexsort((rr, kk))  # positions within a rank are already ascending
        if need < 0 or need > len(order):
            raise AssertionError("splitter bracket does not contain the target")
        taken = np.bincount(rr[order[:need]], minlength=W)
        for i in range(W):
            splits[gi + 1, i] = int(metas[i][gi, 0]) + int(taken[i])
    return splits


def exchange(keys, splits: np.ndarray, tags=None, group=None):
    """All-to-all-v of the locally sorted shard by the split matrix; returns the
    received keys (and tags) concatenated in rank order."""
    import torch

    dist = _dist()
    W = dist.get_world_size(group)
    rank = dist.get_rank(group)
    send = [int(splits[g + 1, rank] - splits[g, rank]) for g in range(W)]
    recv = [int(splits[rank + 1, i] - splits[rank, i]) for i in range(W)]
    out = torch.empty(sum(recv), dtype=keys.dtype, device=keys.device)
    dist.all_to_all_single(out, keys, recv, send, group=group)
    tout = None
    if tags is not None:
        tout = torch.empty(sum(recv), dtype=tags.dtype, device=tags.device)
        dist.all_to_all_single(tout, tags, recv, send, group=group)
    return out, tout, recv


def _default_local_sort(keys, tags):
    from .sorters import SortConfig, powersort

    return powersort(keys, SortConfig(), None, tags)


def sharded_sort(keys, tags=None, group=None, local_sort: Optional[Callable] = None,
                 samples: int = SAMPLES):
    """Globally stable sort of an array sharded contiguously over the ranks.

    `keys` (and `tags`) are this rank's contiguous shard (torch tensors).  Returns
    (sorted_slice, tags_slice, info): this rank's slice of the global sorted
    order, same length as its input shard.
    """
    local_sort = local_sort or _default_local_sort
    m_local = local_sort(keys, tags)
    splits = compute_splits(keys, group, samples)
    out, tout, recv = exchange(keys, splits, tags, group)
    m_merge = local_sort(out, tout)
    return out, tout, {"local": m_local, "merge": m_merge, "splits": splits, "recv": recv}


# ------------------------------------------------------------------ bench --
def bench_sharded(args, rank: int, world: int, local_rank: int) -> dict:
    """bench.py --gpus N (torchrun): weak scaling, n keys per rank."""
    import torch
    import torch.distributed as dist

    from . import workloads

    dev = torch.device("cuda", local_rank)
    keys_np, tags_np = workloads.generate(args.config, args.n, seed=1 + rank)
    n = len(keys_np)
    src = torch.from_numpy(keys_np).to(dev)
    tsrc = torch.from_numpy(tags_np).to(dev) if tags_np is not None else None
    flush = torch.empty(512 << 20, dtype=torch.uint8, device=dev)
    times = []
    for it in range(args.warmup + args.steps):
        work = src.clone()
        tw = tsrc.clone() if tsrc is not None else None
        flush.fill_(1)
        dist.barrier()
        torch.cuda.synchronize()
        e0 = torch.cuda.Event(enable_timing=True)
        e1 = torch.cuda.Event(enable_timing=True)
        e0.record()
        out, tout, info = sharded_sort(work, tw)
        e1.record()
        torch.cuda.synchronize()
        dist.barrier()
        if it >= args.warmup:
            times.append(e0.elapsed_time(e1))
    t = torch.tensor([float(np.mean(times))], device=dev)
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    ms = float(t.item())
    # e2e: this rank's shard from pinned host memory, the sharded sort, its slice back
    hk = torch.from_numpy(keys_np).pin_memory()
    ht = torch.from_numpy(tags_np).pin_memory() if tags_np is not None else None
    e2e = []
    for it in range(args.warmup + args.steps):
        hk.copy_(torch.from_numpy(keys_np))
        flush.fill_(1)
        dist.barrier()
        torch.cuda.synchronize()
        e0 = torch.cuda.Event(enable_timing=True)
        e1 = torch.cuda.Event(enable_timing=True)
        e0.record()
        dk = hk.to(dev, non_blocking=True)
        dt = ht.to(dev, non_blocking=True) if ht is not None else None
        o2, t2, _ = sharded_sort(dk, dt)
        hk.copy_(o2, non_blocking=True)  # pinned: a device-to-host DMA on the stream
        if t2 is not None:
            ht.copy_(t2, non_blocking=True)
        e1.record()
        torch.cuda.synchronize()
        dist.barrier()
        if it >= args.warmup:
            e2e.append(e0.elapsed_time(e1))
    te = torch.tensor([float(np.mean(e2e))], device=dev)
    dist.all_reduce(te, op=dist.ReduceOp.MAX)
    e2e_ms = float(te.item())
    B = keys_np.itemsize + (tags_np.itemsize if tags_np is not None else 0)
    # global sortedness check: local sorted + boundary with the next rank
    ok = bool((out[1:] >= out[:-1]).all().item()) if out.numel() > 1 else True
    edge = torch.tensor([out[0].item() if out.numel() else 0, out[-1].item() if out.numel() else 0],
                        dtype=torch.int64, device=dev)
    edges = [torch.zeros_like(edge) for _ in range(world)]
    dist.all_gather(edges, edge)
    for i in range(world - 1):
        ok &= bool(edges[i][1].item() <= edges[i + 1][0].item())
    return {
        "metric": "powersort keys/s at n=1e7 int32 random-runs; % of HBM roofline; 1/2/4/8 GPU",
        "value": n * world / (ms / 1e3), "unit": "keys/s", "n_gpus": world, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": ms, "higher_is_better": True, "scaling": "weak",
        "vs_baseline": None, "dtype": str(keys_np.dtype), "data": "synthetic (seeded PCG64, shard i uses seed 1+i)",
        "config": {"workload": f"cfg{args.config} per rank, one global array sharded contiguously",
                   "n_per_gpu": n, "parallelism": f"shard{world}",
                   "l2": "flushed (512 MiB write) before every timed step"},
        "globally_sorted_ok": ok,
        "e2e": {"value": n * world / (e2e_ms / 1e3), "unit": "keys/s", "ms_per_step": e2e_ms,
                "h2d_bytes_per_step": n * B, "d2h_bytes_per_step": n * B},
        # our kernels per step: two powersorts (shard, then the received runs), 3 launches each
        "gpu_launches": 6 * args.steps,
    }
