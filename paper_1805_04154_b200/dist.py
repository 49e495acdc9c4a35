"""Arrays that span GPUs: per-GPU powersort on contiguous shards, then an exact
co-rank split and one stable W-way merge.

Global order = the reference's stable order of the concatenated array, i.e.
(key, shard rank, position in shard): the reference's merges send ties to the
left run (runcore.py:262-263).  Rank g ends with output positions
[t_g, t_{g+1}) of that order, t_g = n_0 + ... + n_{g-1}: the same number of
elements it started with, the next contiguous slice of the sorted array.

Two data planes, one merge kernel (csrc/rs_kway.cuh):

* **P2P (NVLink, the default on one node).**  Every rank's shard lives in a
  CUDA-IPC buffer (``P2PShardSpace``) that every other rank maps.  After the
  local sorts and one host barrier, rank g finds its split vectors with the
  device co-rank kernel reading all W shards in place (``rs_corank``: exact
  multi-sequence selection over peer memory, no host round of samples), and
  the W-way merge kernel streams its slice straight out of the peers' buffers
  (``rs_kway_merge``).  The exchange is the merge's input stream: each element
  crosses NVLink once and is written once.
* **NCCL (fallback, e.g. across nodes).**  Splitters from regular samples and
  two all-gathers (``compute_splits``), ``all_to_all_single`` of the segments,
  then the same W-way merge over the W received runs in local HBM.

The local sorter and the NCCL-plane merge are parameters so the host logic can
be exercised with the gloo backend on CPU (tests/test_dist_gloo.py); the product
path passes the CUDA powersort and the CUDA k-way merge.
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


def _device_merge(out, tout, recv):
    """Stable merge of the received runs (rank order), in place on the device:
    they are contiguous in the receive buffer, so the powersort executor merges
    them along a balanced binary tree (rs_merge_runs; log2 W passes of the
    tuned two-way merge, which outruns one W-way pass of the k-way kernel for
    W > 2 on one GPU)."""
    from . import kway

    kway.merge_runs(out, tout, [int(c) for c in recv])
    return out, tout


def sharded_sort(keys, tags=None, group=None, local_sort: Optional[Callable] = None,
                 samples: int = SAMPLES, merge: Optional[Callable] = None):
    """Globally stable sort of an array sharded contiguously over the ranks,
    NCCL data plane (see sharded_sort_p2p for the NVLink path).

    `keys` (and `tags`) are this rank's contiguous shard (torch tensors).  Returns
    (sorted_slice, tags_slice, info): this rank's slice of the global sorted
    order, same length as its input shard.
    """
    local_sort = local_sort or _default_local_sort
    merge = merge or _device_merge
    m_local = local_sort(keys, tags)
    splits = compute_splits(keys, group, samples)
    out, tout, recv = exchange(keys, splits, tags, group)
    out, tout = merge(out, tout, recv)
    return out, tout, {"local": m_local, "splits": splits, "recv": recv}


class P2PShardSpace:
    """Shard buffers every rank of `group` maps (CUDA IPC over NVLink).

    ``keys`` / ``tags`` are this rank's shard (torch views of its IPC buffers,
    capacity elements); ``peer_keys[i]`` / ``peer_tags[i]`` are the device
    addresses of rank i's buffers in this process.  Collective: every rank
    constructs it with the same capacity and dtypes.
    """

    def __init__(self, capacity: int, key_dtype, tag_dtype=None, group=None):
        import torch

        from . import kway

        dist = _dist()
        self.group = group
        self.W = dist.get_world_size(group)
        self.rank = dist.get_rank(group)
        if self.W > kway.MAX_SHARDS:
            raise ValueError(f"the P2P merge takes at most {kway.MAX_SHARDS} ranks")
        self.capacity = int(capacity)
        self.device = torch.device("cuda", torch.cuda.current_device())
        kb = torch.empty(0, dtype=key_dtype).element_size()
        self._kbuf = kway.IpcBuffer(max(1, self.capacity) * kb)
        self._tbuf = None
        if tag_dtype is not None:
            tb = torch.empty(0, dtype=tag_dtype).element_size()
            self._tbuf = kway.IpcBuffer(max(1, self.capacity) * tb)
        self.keys = kway.tensor_at(self._kbuf.address, self.capacity, key_dtype, self.device)
        self.tags = (kway.tensor_at(self._tbuf.address, self.capacity, tag_dtype, self.device)
                     if self._tbuf is not None else None)
        mine = (self._kbuf.handle_bytes(), self._tbuf.handle_bytes() if self._tbuf is not None else None)
        allh = [None] * self.W
        dist.all_gather_object(allh, mine, group=group)
        self._opened = []
        self.peer_keys, self.peer_tags = [], []
        for i, (hk, ht) in enumerate(allh):
            if i == self.rank:
                self.peer_keys.append(self._kbuf.address)
                self.peer_tags.append(self._tbuf.address if self._tbuf is not None else None)
                continue
            pk = kway.ipc_open(hk)
            self._opened.append(pk)
            self.peer_keys.append(pk)
            if ht is not None:
                pt = kway.ipc_open(ht)
                self._opened.append(pt)
                self.peer_tags.append(pt)
            else:
                self.peer_tags.append(None)

    def close(self):
        from . import kway

        _dist().barrier(group=self.group)
        for p in self._opened:
            kway.ipc_close(p)
        self._opened = []
        _dist().barrier(group=self.group)
        self._kbuf.free()
        if self._tbuf is not None:
            self._tbuf.free()


def sharded_sort_p2p(space: P2PShardSpace, n_local: int, local_sort: Optional[Callable] = None,
                     out_keys=None, out_tags=None):
    """Globally stable sort of the shards in `space` (this rank: the first
    n_local elements of space.keys / space.tags), NVLink data plane.

    Over NCCL the whole step is stream-ordered, with no host synchronisation:
    local powersort -> all-gather of the shard lengths (an NCCL collective
    cannot complete before every rank has finished the work queued before it,
    so it doubles as the barrier "every shard is sorted") -> device co-rank of
    this rank's output range over the peers' shards -> W-way merge reading the
    peers' shards -> a one-element all-reduce (no rank rewrites its shard
    buffer before every peer has finished reading it).  With another backend
    (gloo: the one-GPU test) the barriers are host barriers around the same
    kernels.

    Returns (sorted_slice, tags_slice, info) like sharded_sort; the shard
    buffers hold each rank's locally sorted shard afterwards.
    """
    import torch

    from . import kway

    dist = _dist()
    group = space.group
    W, g = space.W, space.rank
    nccl = dist.get_backend(group) == "nccl"
    keys = space.keys[:n_local]
    tags = space.tags[:n_local] if space.tags is not None else None
    if local_sort is not None:
        m_local = local_sort(keys, tags) if n_local > 1 else None
    else:  # enqueued without a host sync; its Metrics stay fetchable
        from .sorters import sort_async

        m_local = sort_async(keys, tags, workspace=getattr(space, "sort_ws", None))
        if m_local is not None:
            space.sort_ws = m_local.workspace
    if out_keys is None:
        out_keys = torch.empty(n_local, dtype=space.keys.dtype, device=space.device)
    if tags is not None and out_tags is None:
        out_tags = torch.empty(n_local, dtype=space.tags.dtype, device=space.device)
    # a device fill, not torch.tensor(..., device=): that is a blocking host-to-device
    # copy, which would hold the host until the local sort has finished
    mine = torch.full((1,), int(n_local), dtype=torch.int64, device=space.device)
    if nccl:
        dlens = torch.empty(W, dtype=torch.int64, device=space.device)
        dist.all_gather_into_tensor(dlens, mine, group=group)
    else:
        torch.cuda.current_stream().synchronize()
        ns = [None] * W
        dist.all_gather_object(ns, int(n_local), group=group)
        dlens = torch.tensor(ns, dtype=torch.int64, device=space.device)
    shards = [kway.Shard(space.peer_keys[i], space.peer_tags[i], 0, 0) for i in range(W)]
    dsplit = torch.empty(2 * W, dtype=torch.int64, device=space.device)
    kway.corank_rank(shards, dlens, g, dsplit, space.keys.dtype)
    space.ws = kway.kway_merge_split(shards, dsplit, n_local, out_keys[:n_local],
                                     out_tags[:n_local] if tags is not None else None,
                                     workspace=getattr(space, "ws", None))
    if nccl:
        done = torch.zeros(1, dtype=torch.int32, device=space.device)
        dist.all_reduce(done, group=group)
    else:
        torch.cuda.current_stream().synchronize()
        dist.barrier(group=group)
    return out_keys[:n_local], (out_tags[:n_local] if tags is not None else None), \
        {"local": m_local, "split": dsplit, "lens": dlens}
