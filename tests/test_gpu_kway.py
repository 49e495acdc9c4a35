"""The cross-GPU merge kernels (csrc/rs_kway.cuh) on one B200, ranks emulated.

Each "rank" g runs exactly what it runs in the sharded sort -- device co-rank of
its output range [t_g, t_{g+1}) over all W sorted shards, then the W-way merge
of its slice -- with every shard a local buffer instead of a peer mapping (the
kernels take plain pointers; nothing waits on another rank, so emulating the
ranks as consecutive launches on one GPU is exact).  The concatenated slices
must equal the stable sort of the concatenated shards, keys and tags
(tag = global index, so the order of equal keys is checked).
"""
import numpy as np
import pytest

pytestmark = pytest.mark.gpu


def _shards(rng, W, kind, dtype):
    out, base = [], 0
    for i in range(W):
        if kind == "ragged":
            n = int(rng.choice([0, 1, 2, 17, 1000, int(rng.integers(0, 200000))]))
        elif kind == "big":
            n = int(rng.integers(100000, 400000))
        else:
            n = int(rng.integers(0, 60000))
        if kind == "dups" or kind == "big":
            k = rng.integers(0, 16, n)
        elif kind == "allsame":
            k = np.full(n, 5)
        elif kind == "disjoint":
            k = rng.integers(0, 1000, n) + (W - i) * 1000
        else:
            k = rng.integers(-(1 << 30), 1 << 30, n)
        k = np.sort(k.astype(dtype), kind="stable")
        out.append((k, np.arange(base, base + n, dtype=np.int64)))
        base += n
    return out


def _run_ranks(shards, with_tags=True):
    import torch

    from paper_1805_04154_b200 import kway

    dev = torch.device("cuda", 0)
    W = len(shards)
    dk = [torch.from_numpy(k).to(dev) for k, _ in shards]
    dt = [torch.from_numpy(t).to(dev) for _, t in shards] if with_tags else [None] * W
    ns = [len(k) for k, _ in shards]
    T = np.concatenate([[0], np.cumsum(ns)]).astype(np.int64)
    full = [kway.Shard.of(dk[i], dt[i]) for i in range(W)]
    outs_k, outs_t = [], []
    for g in range(W):
        c = kway.corank(full, [int(T[g]), int(T[g + 1])], dk[0].dtype)
        assert c[0].sum() == T[g] and c[1].sum() == T[g + 1]
        mine = [full[i].with_range(int(c[0][i]), int(c[1][i])) for i in range(W)]
        ok = torch.empty(ns[g], dtype=dk[0].dtype, device=dev)
        ot = torch.empty(ns[g], dtype=torch.int64, device=dev) if with_tags else None
        kway.kway_merge(mine, ok, ot)
        torch.cuda.synchronize()
        outs_k.append(ok.cpu().numpy())
        if with_tags:
            outs_t.append(ot.cpu().numpy())
    return outs_k, outs_t


@pytest.mark.parametrize("W", [1, 2, 3, 5, 8])
@pytest.mark.parametrize("kind", ["dups", "allsame", "disjoint", "random", "ragged"])
def test_emulated_ranks_match_stable_sort(W, kind):
    rng = np.random.default_rng(100 * W + hash(kind) % 97)
    for dtype in (np.int32, np.int64):
        shards = _shards(rng, W, kind, dtype)
        allk = np.concatenate([s[0] for s in shards])
        allt = np.concatenate([s[1] for s in shards])
        order = np.argsort(allk, kind="stable")
        ok, ot = _run_ranks(shards)
        assert np.array_equal(np.concatenate(ok), allk[order]), (W, kind, dtype)
        assert np.array_equal(np.concatenate(ot), allt[order]), (W, kind, dtype)
        for g in range(W):
            assert len(ok[g]) == len(shards[g][0])


def test_big_shards_keys_only_and_int32_tags():
    import torch

    from paper_1805_04154_b200 import kway

    rng = np.random.default_rng(5)
    shards = _shards(rng, 8, "big", np.int64)
    allk = np.concatenate([s[0] for s in shards])
    order = np.argsort(allk, kind="stable")
    ok, _ = _run_ranks(shards, with_tags=False)
    assert np.array_equal(np.concatenate(ok), allk[order])
    # one merge of all ranges with 4-byte tags
    dev = torch.device("cuda", 0)
    dk = [torch.from_numpy(k).to(dev) for k, _ in shards]
    dt = [torch.from_numpy(t.astype(np.int32)).to(dev) for _, t in shards]
    out = torch.empty(len(allk), dtype=torch.int64, device=dev)
    tout = torch.empty(len(allk), dtype=torch.int32, device=dev)
    kway.kway_merge([kway.Shard.of(dk[i], dt[i]) for i in range(8)], out, tout)
    allt = np.concatenate([s[1] for s in shards]).astype(np.int32)
    assert np.array_equal(out.cpu().numpy(), allk[order])
    assert np.array_equal(tout.cpu().numpy(), allt[order])


def test_corank_every_target_small():
    """Every global rank t of a small heavy-tie instance: the split vector is the
    (key, shard, position) prefix of length t."""
    import torch

    from paper_1805_04154_b200 import kway

    rng = np.random.default_rng(9)
    shards = [np.sort(rng.integers(0, 4, int(rng.integers(0, 40)))).astype(np.int64) for _ in range(5)]
    dk = [torch.from_numpy(k).cuda() for k in shards]
    full = [kway.Shard.of(d) for d in dk]
    total = sum(len(k) for k in shards)
    allk = np.concatenate(shards)
    src = np.concatenate([np.full(len(k), i) for i, k in enumerate(shards)])
    order = np.argsort(allk, kind="stable")
    c = kway.corank(full, list(range(total + 1)), torch.int64)
    for t in range(total + 1):
        want = np.bincount(src[order[:t]], minlength=5)
        assert np.array_equal(c[t], want), t


def test_rejects_bad_shards():
    import torch

    from paper_1805_04154_b200 import kway

    d = torch.zeros(10, dtype=torch.int64, device="cuda")
    with pytest.raises(ValueError):
        kway.corank([kway.Shard.of(d, lo=5, hi=2)], [1], torch.int64)
    with pytest.raises(ValueError):
        kway.corank([kway.Shard.of(d)], [11], torch.int64)
    with pytest.raises(ValueError):
        kway.kway_merge([kway.Shard.of(d)] * 9, d)


@pytest.mark.parametrize("W", [2, 3, 5, 8])
def test_merge_runs_in_place_matches_stable_sort(W):
    """rs_merge_runs: W sorted runs back to back merged in place (the NCCL
    plane's merge of its received runs), ties to the earlier run; empty runs,
    heavy ties, int32 / int64 keys, no / 4- / 8-byte tags."""
    import torch

    from paper_1805_04154_b200 import kway

    rng = np.random.default_rng(7 * W)
    dev = torch.device("cuda", 0)
    for dtype, tdt, big in ((np.int32, None, False), (np.int64, np.int64, False), (np.int32, np.int32, True)):
        lens = [int(rng.choice([0, 1, 5, 3000, int(rng.integers(0, 400000 if big else 60000))])) for _ in range(W)]
        runs = [np.sort(rng.integers(0, 50, size=L).astype(dtype), kind="stable") for L in lens]
        k = np.concatenate(runs) if sum(lens) else np.zeros(0, dtype=dtype)
        t = np.arange(len(k)).astype(tdt) if tdt is not None else None
        order = np.argsort(k, kind="stable")
        dk = torch.from_numpy(k.copy()).to(dev)
        dt = torch.from_numpy(t.copy()).to(dev) if t is not None else None
        kway.merge_runs(dk, dt, lens)
        torch.cuda.synchronize()
        assert np.array_equal(dk.cpu().numpy(), k[order]), (W, dtype, lens)
        if t is not None:
            assert np.array_equal(dt.cpu().numpy(), t[order]), (W, dtype, lens)
