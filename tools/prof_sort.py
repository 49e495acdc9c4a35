"""Run a few powersorts of one BASELINE config (device-resident) -- for ncu / nsight runs."""
import argparse, ctypes, sys
sys.path.insert(0, '.')
import torch
from paper_1805_04154_b200 import _lib, workloads

ap = argparse.ArgumentParser()
ap.add_argument('--config', type=int, default=2)
ap.add_argument('--n', type=int, default=None)
ap.add_argument('--reps', type=int, default=3)
ap.add_argument('--w', type=int, default=24)
ap.add_argument('--algo', type=int, default=0)
a = ap.parse_args()
keys, tags = workloads.generate(a.config, a.n)
L = _lib.lib()
dev = torch.device('cuda')
src = torch.from_numpy(keys).to(dev); work = torch.empty_like(src)
tsrc = torch.from_numpy(tags).to(dev) if tags is not None else None
twork = torch.empty_like(tsrc) if tsrc is not None else None
kc = _lib.RS_KEY_I32 if keys.itemsize == 4 else _lib.RS_KEY_I64
tb = tags.itemsize if tags is not None else 0
n = len(keys)
wsb = L.rs_workspace_bytes(a.algo, kc, tb, n, a.w)
ws = torch.empty(wsb, dtype=torch.uint8, device=dev)
st = torch.cuda.current_stream()
for i in range(a.reps):
    work.copy_(src)
    if twork is not None: twork.copy_(tsrc)
    m = _lib.RsMetrics()
    _lib.check(L.rs_sort(a.algo, kc, work.data_ptr(), tb, twork.data_ptr() if twork is not None else None, n, a.w, 0,
                         ws.data_ptr(), wsb, st.cuda_stream, ctypes.byref(m), None))
torch.cuda.synchronize()
print('ok', m.merge_cost, m.runs_detected)
if __import__('os').environ.get('RS_LIB'):
    buf = (ctypes.c_uint64 * 210)()
    k = L.rs_debug_counters(kc, tb, n, a.w, ws.data_ptr(), buf, 210)
    ts = list(buf[138:154]); print('prep phase us', [round((ts[i] - ts[i-1]) / 1e3, 1) for i in range(1, 12) if ts[i] and ts[i-1]])
    arr = list(buf[154:170]); print('phase work (latest arrival - prev exit) / barrier (exit - latest arrival) us', [(i, round((arr[i] - ts[i-1]) / 1e3, 1), round((ts[i] - arr[i]) / 1e3, 1)) for i in range(1, 10) if arr[i] and ts[i] and ts[i-1]])
    dbg = list(buf[170:202]); t4 = min([x for x in dbg if x] or [0]); print('dbg us after first dbg', [(i, round((dbg[i] - t4) / 1e3, 1)) for i in range(32) if dbg[i]])
    if ts[8]: print('small-path dbg[0..4] us after ts8', [round((dbg[i] - ts[8]) / 1e3, 2) for i in range(5) if dbg[i]], 'ts9', round((ts[9] - ts[8]) / 1e3, 2))
    print('ts us after ts4', [(i, round((ts[i] - t4) / 1e3, 1)) for i in range(4, 12) if ts[i]])
    print('phase-1 max-warp cycles wait/bits/bwords/walk', ts[12:16])
    dw = list(buf[10:74]); dt = list(buf[74:138])
    print('depth: wait_cycles(M) tasks', [(d, round(dw[d] / 1e6, 1), dt[d]) for d in range(64) if dt[d]])
    names = ['prod_dep_wait', 'prod_search', 'prod_stage_wait', 'cons_full_wait', 'cons_tile_work', 'prod_ready', 'prod_pfence', 'prod_issue', 'n_tasks', 'phaseA']
    print({nm: buf[i] for i, nm in enumerate(names[:k])})
    dur_max, dur_sum, ntask = buf[170 + 25], buf[170 + 26], buf[170 + 27]
    if ntask:
        print('phaseA tasks', ntask, 'max cycles', dur_max, 'mean', dur_sum // ntask,
              'max-task span', buf[170 + 28] & 0xffffff, 'leaves-1', buf[170 + 29] & 0xffffff, 'kind', buf[170 + 30] & 0xffffff)
    print('slowest fused task: total/tables+span/leaves/levels cycles, levels:', list(buf[202:207]) if len(buf) > 206 else 'n/a')
    if a.algo == 1:
        print('peeksort replay levels', buf[154 + 15])
