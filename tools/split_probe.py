"""Time the pieces of dist.compute_splits (1 rank, NCCL)."""
import os, sys, time
sys.path.insert(0, '.')
os.environ.setdefault('MASTER_ADDR', '127.0.0.1'); os.environ.setdefault('MASTER_PORT', '29562')
import numpy as np, torch, torch.distributed as dist
from paper_1805_04154_b200 import dist as rsd, workloads
dist.init_process_group('nccl', rank=0, world_size=1)
k, _ = workloads.generate(2)
keys = torch.sort(torch.from_numpy(k).cuda())[0]
torch.cuda.synchronize()
def T(): torch.cuda.synchronize(); return time.perf_counter()
for it in range(5):
    t0 = T()
    t1 = t2 = t3 = t4 = t5 = t6 = t0
    sp = rsd.compute_splits(keys); t7 = T()
    print('us', [round((b - a) * 1e6) for a, b in zip([t0, t1, t2, t3, t4, t5, t6], [t1, t2, t3, t4, t5, t6, t7])])
