"""Run the same powersort twice on identically poisoned workspaces and report
which workspace arrays differ (nondeterminism hunting).  Layout replica of
make_layout (csrc/runsort_b200.cu) for powersort, int32 keys, no tags."""
import ctypes, sys
sys.path.insert(0, '.')
import numpy as np
import torch
from paper_1805_04154_b200 import workloads, _lib

cfg = int(sys.argv[1]) if len(sys.argv) > 1 else 2
reps = int(sys.argv[2]) if len(sys.argv) > 2 else 4
keys, _ = workloads.generate(cfg)
n, w, kb, tb = len(keys), 24, 4, 0
L = _lib.lib()
wsb = L.rs_workspace_bytes(0, _lib.RS_KEY_I32, 0, n, w)

def layout():
    au = lambda x: (x + 255) // 256 * 256
    words = (n + 31) // 32 + 2
    ntiles = (n + 2047) // 2048
    ngroups = (ntiles + 63) // 64
    r_max = n // max(w, 2) + 2
    nchunks = (r_max + 255) // 256 + 1
    tile, fcap = 256 * 15, 4096
    levels = 2 + n.bit_length()
    max_tasks = levels * (n // tile + n // fcap + 2) + 3 * r_max + 2 * (n // tile) + 16
    items = [("key1", n * kb + 64), ("tag1", n * tb + 64), ("key2", n * kb + 64), ("tag2", n * tb + 64),
             ("ascw", words * 4), ("tables", ntiles * (w + 1) * 8), ("gtab", ngroups * (w + 1) * 8),
             ("gentry", ngroups * 4), ("goff", ngroups * 8), ("tentry", ntiles * 4), ("toff", ntiles * 8),
             ("leaf_start", (r_max + 1) * 8), ("leaf_info", r_max * 4), ("leaf_depth", r_max), ("K", r_max * 8),
             ("P", r_max), ("la", r_max), ("ra", r_max), ("depth", r_max), ("node_a", r_max * 4),
             ("node_b", r_max * 4), ("node_s", r_max * 8), ("node_e", r_max * 8), ("parent", (2 * r_max + 2) * 4),
             ("child", (2 * r_max + 2) * 4), ("need", (2 * r_max + 2) * 4), ("done", (2 * r_max + 2) * 4),
             ("agg", 2 * nchunks * 16), ("tasks", max_tasks * 8), ("chunkdep", ((r_max + 255) // 256 + 1) * 64 * 4),
             ("cls", 2 * r_max + 2), ("met", 1 << 20)]
    off, out = 0, []
    for name, b in items:
        out.append((name, off, b))
        off = au(off + b)
    return out

lay = layout()
src = torch.from_numpy(keys).cuda()
ws = torch.empty(wsb, dtype=torch.uint8, device='cuda')
st = torch.cuda.current_stream()
snaps, outs = [], []
for i in range(reps):
    ws.fill_(0x5A)
    wk = src.clone()
    m = _lib.RsMetrics()
    _lib.check(L.rs_sort(0, _lib.RS_KEY_I32, wk.data_ptr(), 0, None, n, w, 0, ws.data_ptr(), wsb, st.cuda_stream,
                         ctypes.byref(m), None))
    torch.cuda.synchronize()
    snaps.append(ws.cpu().numpy())
    outs.append(wk.cpu().numpy())
for i in range(1, reps):
    d = np.nonzero(snaps[i] != snaps[0])[0]
    od = np.nonzero(outs[i] != outs[0])[0]
    names = {}
    for x in d[:: max(1, len(d) // 2000)] if len(d) else []:
        for name, o, b in lay:
            if o <= x < o + b:
                names[name] = names.get(name, 0) + 1
                break
    print(f"run {i} vs 0: {len(d)} workspace bytes differ {names}; output elems differ {len(od)}")
