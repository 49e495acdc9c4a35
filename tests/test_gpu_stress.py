"""GPU repeatability: the same sort repeated on a poisoned workspace.

The executors are dataflow kernels whose schedule changes from run to run
(task claiming, per-node completion counters, bulk copies); a synchronization
bug shows up as a rare wrong result, not a deterministic one.  Every repetition
poisons the whole workspace (scratch key/tag buffers included, so a missing
write cannot be masked by the previous run's data) and must reproduce the C
oracle bit for bit.
"""
import ctypes

import numpy as np
import pytest

from oracle import oracle
from paper_1805_04154_b200 import _lib, workloads

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("algo,cfg,reps", [("powersort", 2, 40), ("peeksort", 2, 15), ("powersort", 3, 10)])
def test_repeated_sorts_poisoned_workspace(algo, cfg, reps):
    import torch

    keys, _ = workloads.generate(cfg)
    ref = keys.copy()
    getattr(oracle, algo)(ref, 24, "bitonic")
    L = _lib.lib()
    code = _lib.RS_ALGO_PEEKSORT if algo == "peeksort" else _lib.RS_ALGO_POWERSORT
    n = len(keys)
    wsb = L.rs_workspace_bytes(code, _lib.RS_KEY_I32, 0, n, 24)
    ws = torch.empty(wsb, dtype=torch.uint8, device="cuda")
    src = torch.from_numpy(keys).cuda()
    st = torch.cuda.current_stream()
    bad = []
    for i in range(reps):
        ws.fill_(0xA5 if i % 2 else 0x3C)
        w = src.clone()
        m = _lib.RsMetrics()
        _lib.check(L.rs_sort(code, _lib.RS_KEY_I32, w.data_ptr(), 0, None, n, 24, 0, ws.data_ptr(), wsb,
                             st.cuda_stream, ctypes.byref(m), None))
        torch.cuda.synchronize()
        got = w.cpu().numpy()
        if not np.array_equal(got, ref):
            bad.append((i, int(np.count_nonzero(got != ref))))
    assert not bad, f"{len(bad)}/{reps} repetitions differ from the oracle: {bad[:5]}"
