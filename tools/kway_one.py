"""One W-way merge (default W=8, n=1e8 int32 keys + int64 tags) for ncu captures."""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1805_04154_b200 import kway  # noqa: E402

W = int(os.environ.get("W", "8"))
n = int(os.environ.get("N", str(10**8)))
dev = torch.device("cuda", 0)
g = torch.Generator(device=dev).manual_seed(W)
keys = torch.randint(0, 1 << 30, (n,), generator=g, device=dev, dtype=torch.int64).to(torch.int32)
tags = torch.arange(n, device=dev, dtype=torch.int64)
bounds = [n * i // W for i in range(W + 1)]
for i in range(W):
    keys[bounds[i]:bounds[i + 1]] = torch.sort(keys[bounds[i]:bounds[i + 1]]).values
shards = [kway.Shard(keys.data_ptr(), tags.data_ptr(), bounds[i], bounds[i + 1]) for i in range(W)]
out = torch.empty_like(keys)
tout = torch.empty_like(tags)
ws = None
for _ in range(2):
    ws = kway.kway_merge(shards, out, tout, workspace=ws)
torch.cuda.synchronize()
print("sorted", bool(torch.all(out[1:] >= out[:-1]).item()))
