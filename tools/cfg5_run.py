"""Time powersort on BASELINE config 5 (n = 2^31 int64) on one GPU."""
import ctypes, sys, time
sys.path.insert(0, '.')
import numpy as np, torch
from paper_1805_04154_b200 import _lib, workloads
L = _lib.lib()
n = workloads.CONFIG5_N
t0 = time.time()
src = workloads.config5_device(n, seed=1)
torch.cuda.synchronize()
print('gen s', round(time.time() - t0, 2))
work = torch.empty_like(src)
wsb = L.rs_workspace_bytes(0, _lib.RS_KEY_I64, 0, n, 24)
ws = torch.empty(wsb, dtype=torch.uint8, device='cuda')
print('workspace GB', wsb / 1e9)
st = torch.cuda.current_stream()
L.rs_profile(1)
for i in range(4):
    work.copy_(src)
    torch.cuda.synchronize()
    e0 = torch.cuda.Event(enable_timing=True); e1 = torch.cuda.Event(enable_timing=True)
    m = _lib.RsMetrics()
    e0.record()
    _lib.check(L.rs_sort(0, _lib.RS_KEY_I64, work.data_ptr(), 0, None, n, 24, 0, ws.data_ptr(), wsb, st.cuda_stream, None, None))
    e1.record(); e1.synchronize()
    buf = (ctypes.c_double * 4)(); L.rs_profile_read(buf, 4)
    _lib.check(L.rs_fetch_metrics(0, _lib.RS_KEY_I64, 0, n, 24, ws.data_ptr(), st.cuda_stream, ctypes.byref(m)))
    ms = e0.elapsed_time(e1)
    alg = 2 * 8 * buf[3]
    print(f"ms {ms:.2f} keys/s {n / ms * 1e3:.3e} phases {[round(x, 2) for x in buf[:3]]} merge frac {alg / (buf[2] / 1e3) / 6551.7e9:.3f}",
          'metrics', m.merge_cost, m.comparisons, m.runs_detected, m.max_stack_height)
print('sorted', bool((work[1:] >= work[:-1]).all().item()))
