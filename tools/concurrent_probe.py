"""Throughput of the public API with T host threads sorting independent arrays
concurrently (the shape of the reference arm: one sort per host thread), for
pinned CPU tensors and numpy arrays, config 2.  Prints keys/s per (path, T)."""
import sys
import threading
import time

sys.path.insert(0, ".")
import numpy as np
import torch

import paper_1805_04154_b200 as rs
from paper_1805_04154_b200 import workloads

cfg = int(sys.argv[1]) if len(sys.argv) > 1 else 2
K = int(sys.argv[2]) if len(sys.argv) > 2 else 12
keys, tags = workloads.generate(cfg)
n = len(keys)
ref = np.sort(keys, kind="stable")


def run(path, T):
    bar = threading.Barrier(T + 1)
    errs = []
    done = [0] * T
    t_end = [0.0] * T

    def worker(i):
        try:
            s = torch.cuda.Stream()
            base = torch.from_numpy(keys)
            # K fresh inputs per thread, prepared before the timed region
            bufs = [base.pin_memory() if path == "pinned" else keys.copy() for _ in range(K + 2)]
            with torch.cuda.stream(s):
                for it in range(2):  # warm-up (allocations, staging sessions)
                    rs.powersort(bufs[K + it])
                    s.synchronize()
                bar.wait()
                for it in range(K):
                    rs.powersort(bufs[it])  # synchronous: returns with the result in the host buffer
                    done[i] += 1
                t_end[i] = time.perf_counter()
                for b in bufs[:K]:
                    out = b.numpy() if path == "pinned" else b
                    if not np.array_equal(out, ref):
                        errs.append(f"thread {i}: wrong output")
                        break
        except Exception as ex:  # noqa: BLE001
            errs.append(repr(ex))
            try:
                bar.abort()
            except Exception:
                pass

    th = [threading.Thread(target=worker, args=(i,)) for i in range(T)]
    for t in th:
        t.start()
    bar.wait()
    t0 = time.perf_counter()
    for t in th:
        t.join()
    dt = max(t_end) - t0
    tot = sum(done)
    print(f"cfg{cfg} path={path:6s} T={T} sorts={tot} wall={dt*1e3:8.2f} ms  per-sort={dt*1e3/tot:6.3f} ms  "
          f"{tot*n/dt/1e9:6.2f} G keys/s  errs={errs}", flush=True)


for path in ("pinned", "numpy"):
    for T in (1, 2, 3, 4):
        run(path, T)
