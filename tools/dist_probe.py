import os, sys, time
sys.path.insert(0, '.')
os.environ.setdefault('MASTER_ADDR', '127.0.0.1'); os.environ.setdefault('MASTER_PORT', '29561')
import torch, torch.distributed as dist
import numpy as np
from paper_1805_04154_b200 import dist as rsd, workloads
dist.init_process_group('nccl', rank=0, world_size=1)
k, _ = workloads.generate(2)
src = torch.from_numpy(k).cuda()
for it in range(6):
    w = src.clone(); torch.cuda.synchronize()
    t = [time.perf_counter()]
    m = rsd._default_local_sort(w, None); torch.cuda.synchronize(); t.append(time.perf_counter())
    sp = rsd.compute_splits(w); torch.cuda.synchronize(); t.append(time.perf_counter())
    out, tout, recv = rsd.exchange(w, sp); torch.cuda.synchronize(); t.append(time.perf_counter())
    m2 = rsd._default_local_sort(out, None); torch.cuda.synchronize(); t.append(time.perf_counter())
    print('ms', [round((t[i+1]-t[i])*1e3, 3) for i in range(4)], m2.runs_detected, m2.merge_cost)
