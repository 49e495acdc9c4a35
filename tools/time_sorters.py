"""Device time per sort for every SORTERS entry on one BASELINE config (CUDA
events around rs_sort_ex, inputs resident, one warm-up)."""
import argparse, ctypes, sys
sys.path.insert(0, '.')
import torch
from paper_1805_04154_b200 import _lib, workloads

ap = argparse.ArgumentParser()
ap.add_argument('--config', type=int, default=2)
ap.add_argument('--reps', type=int, default=5)
a = ap.parse_args()
keys, tags = workloads.generate(a.config)
L = _lib.lib()
n = len(keys)
kc = _lib.RS_KEY_I32 if keys.itemsize == 4 else _lib.RS_KEY_I64
src = torch.from_numpy(keys).cuda()
st = torch.cuda.current_stream()
for name, code in [("powersort", 0), ("peeksort", 1), ("top-down", 2), ("bottom-up", 3), ("alpha-stack", 4),
                   ("alpha-merge", 5)]:
    wsb = L.rs_workspace_bytes(code, kc, 0, n, 24)
    ws = torch.empty(wsb, dtype=torch.uint8, device='cuda')
    ts = []
    for i in range(a.reps + 1):
        w = src.clone()
        torch.cuda.synchronize()
        e0 = torch.cuda.Event(enable_timing=True); e1 = torch.cuda.Event(enable_timing=True)
        e0.record(st)
        _lib.check(L.rs_sort_ex(code, kc, w.data_ptr(), 0, None, n, 24, 0, 2.0, ws.data_ptr(), wsb, st.cuda_stream,
                                None, None))
        e1.record(st); e1.synchronize()
        if i: ts.append(e0.elapsed_time(e1))
    ts.sort()
    print(f"cfg{a.config} {name:12s} {ts[len(ts) // 2]:.3f} ms  ({n / ts[len(ts) // 2] / 1e6:.2f} G keys/s)")
    del ws
