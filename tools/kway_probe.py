"""Probe: throughput of the W-way merge kernel (rs_kway_merge) on one GPU --
W sorted runs of total n in HBM, merged into one output; effective GB/s =
2 * n * element bytes / time (CUDA events, L2 flushed before each rep)."""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1805_04154_b200 import kway  # noqa: E402

dev = torch.device("cuda", 0)
flush = torch.empty(512 << 20, dtype=torch.uint8, device=dev)
for n, kdt, tdt in ((10**7, torch.int32, None), (10**8, torch.int32, torch.int64)):
    B = torch.empty(0, dtype=kdt).element_size() + (torch.empty(0, dtype=tdt).element_size() if tdt else 0)
    for W in (2, 4, 8):
        g = torch.Generator(device=dev).manual_seed(W)
        keys = torch.randint(0, 1 << 30, (n,), generator=g, device=dev, dtype=torch.int64).to(kdt)
        tags = torch.arange(n, device=dev, dtype=tdt) if tdt else None
        bounds = [n * i // W for i in range(W + 1)]
        for i in range(W):
            seg = keys[bounds[i]:bounds[i + 1]]
            keys[bounds[i]:bounds[i + 1]] = torch.sort(seg).values
        shards = [kway.Shard(keys.data_ptr(), tags.data_ptr() if tags is not None else None, bounds[i], bounds[i + 1])
                  for i in range(W)]
        out = torch.empty_like(keys)
        tout = torch.empty_like(tags) if tags is not None else None
        ws = None
        ts = []
        for rep in range(6):
            flush.fill_(1)
            torch.cuda.synchronize()
            e0 = torch.cuda.Event(enable_timing=True)
            e1 = torch.cuda.Event(enable_timing=True)
            e0.record()
            ws = kway.kway_merge(shards, out, tout, workspace=ws)
            e1.record()
            torch.cuda.synchronize()
            if rep >= 2:
                ts.append(e0.elapsed_time(e1))
        ms = sum(ts) / len(ts)
        ok = bool(torch.all(out[1:] >= out[:-1]).item())
        print(f"n={n} B={B} W={W} ms={ms:.4f} GB/s={2 * n * B / ms / 1e6:.0f} sorted={ok}", flush=True)
        # the same runs merged in place by the executor along a binary tree (rs_merge_runs)
        lens = [bounds[i + 1] - bounds[i] for i in range(W)]
        ts2 = []
        wsr = None
        for rep in range(6):
            kk = keys.clone()
            tt = tags.clone() if tags is not None else None
            flush.fill_(1)
            torch.cuda.synchronize()
            e0 = torch.cuda.Event(enable_timing=True)
            e1 = torch.cuda.Event(enable_timing=True)
            e0.record()
            wsr = kway.merge_runs(kk, tt, lens, workspace=wsr)
            e1.record()
            torch.cuda.synchronize()
            if rep >= 2:
                ts2.append(e0.elapsed_time(e1))
        ms2 = sum(ts2) / len(ts2)
        ok2 = bool(torch.equal(kk, out))
        print(f"   merge_runs (binary tree, in place) ms={ms2:.4f} GB/s(one-pass equiv)={2 * n * B / ms2 / 1e6:.0f} "
              f"same={ok2}", flush=True)
        del kk, tt, wsr
        del keys, tags, out, tout, ws
        torch.cuda.empty_cache()
