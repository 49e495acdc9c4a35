"""Where the end-to-end time goes: pinned H2D alone, D2H alone, the device sort
alone, and the public-API call (H2D + sort + D2H + Metrics), config 2."""
import sys
import time

sys.path.insert(0, ".")
import numpy as np
import torch

import paper_1805_04154_b200 as rs
from paper_1805_04154_b200 import workloads

keys, _ = workloads.generate(2)
n = len(keys)
hk = torch.from_numpy(keys).pin_memory()
dk = torch.empty(n, dtype=torch.int32, device="cuda")
st = torch.cuda.current_stream()


def timed(fn, reps=10):
    out = []
    for _ in range(reps + 3):
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(st)
        fn()
        e1.record(st)
        e1.synchronize()
        out.append(e0.elapsed_time(e1))
    return float(np.median(out[3:]))


d2h = timed(lambda: hk.copy_(dk, non_blocking=True))
h2d = timed(lambda: dk.copy_(hk, non_blocking=True))
h2d_to = timed(lambda: hk.to("cuda", non_blocking=True))
h2d_b = timed(lambda: dk.copy_(hk, non_blocking=True), reps=30)
streams = [torch.cuda.Stream() for _ in range(4)]


def h2d_split():
    ev = torch.cuda.Event()
    ev.record(st)
    q = n // 4
    for i, s2 in enumerate(streams):
        s2.wait_event(ev)
        with torch.cuda.stream(s2):
            dk[i * q:(i + 1) * q].copy_(hk[i * q:(i + 1) * q], non_blocking=True)
    for s2 in streams:
        e = torch.cuda.Event()
        e.record(s2)
        st.wait_event(e)


h2d_s = timed(h2d_split)
print(f"H2D variants: copy_ {h2d:.3f}  .to {h2d_to:.3f}  copy_ (30 reps) {h2d_b:.3f}  4 streams {h2d_s:.3f} ms")
src = torch.from_numpy(keys).cuda()


def dev_sort():
    dk.copy_(src)
    rs.powersort(dk)


dsort = timed(dev_sort)
cp = timed(lambda: dk.copy_(src))


def e2e():
    hk.copy_(torch.from_numpy(keys))
    rs.powersort(hk)


# host copy of the input is outside the device timing (host memcpy before e0)
res = []
for _ in range(13):
    hk.copy_(torch.from_numpy(keys))
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    t0 = time.perf_counter()
    e0.record(st)
    rs.powersort(hk)
    e1.record(st)
    e1.synchronize()
    res.append((e0.elapsed_time(e1), (time.perf_counter() - t0) * 1e3))
res = res[3:]
e2e_dev = float(np.median([r[0] for r in res]))
e2e_wall = float(np.median([r[1] for r in res]))
print(f"n={n} bytes={n * 4}")
print(f"H2D {h2d:.3f} ms ({n * 4 / h2d / 1e6:.1f} GB/s)  D2H {d2h:.3f} ms ({n * 4 / d2h / 1e6:.1f} GB/s)")
print(f"device sort via API on a CUDA tensor {dsort - cp:.3f} ms (incl. API overhead; d2d restore {cp:.3f} subtracted)")
print(f"e2e events {e2e_dev:.3f} ms, wall {e2e_wall:.3f} ms; overhead beyond H2D+D2H+sort "
      f"{e2e_dev - h2d - d2h - (dsort - cp):.3f} ms")

# device timeline of one public-API call (CUPTI via torch.profiler)
from torch.profiler import ProfilerActivity, profile

for _ in range(3):
    e2e()
torch.cuda.synchronize()
with profile(activities=[ProfilerActivity.CPU, ProfilerActivity.CUDA]) as prof:
    hk.copy_(torch.from_numpy(keys))
    torch.cuda.synchronize()
    rs.powersort(hk)
    torch.cuda.synchronize()
evs = [e for e in prof.events() if e.device_type.name == "CUDA"]
t0 = min(e.time_range.start for e in evs)
for e in sorted(evs, key=lambda e: e.time_range.start):
    print(f"{(e.time_range.start - t0):9.1f} {(e.time_range.end - t0):9.1f} us  {e.name[:70]}")
cpu = [e for e in prof.events() if e.device_type.name == "CPU"]
c0 = min(e.time_range.start for e in cpu)
for e in sorted(cpu, key=lambda e: e.time_range.start)[:60]:
    print(f"cpu {(e.time_range.start - c0):9.1f} {(e.time_range.end - c0):9.1f} us  {e.name[:70]}")
