"""Probe: numpy-in/numpy-out powersort (rs_sort_host_ex staging) on cfg2,
median wall ms over reps; run once per RS_HOST_CHUNK_KB / RS_HOST_THREADS
setting (read once per process).  RS_HOST_TRACE=1 prints the phases."""
import os
import sys
import time

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1805_04154_b200 as rs  # noqa: E402
from paper_1805_04154_b200 import workloads  # noqa: E402

cfg = int(os.environ.get("CFG", "2"))
keys = workloads.config2() if cfg == 2 else workloads.config1()
base = keys.copy()
ts = []
for it in range(13):
    np.copyto(keys, base)
    t0 = time.perf_counter()
    rs.powersort(keys)
    ts.append((time.perf_counter() - t0) * 1e3)
print(f"chunk_kb={os.environ.get('RS_HOST_CHUNK_KB')} threads={os.environ.get('RS_HOST_THREADS')} "
      f"median_ms={np.median(ts[3:]):.3f} min_ms={np.min(ts[3:]):.3f}", flush=True)
