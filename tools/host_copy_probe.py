"""Probe: host<->device copy paths for a 40 MB array (numpy pageable, pinned,
cudaHostRegister), to choose the numpy staging path of the public API."""
import time

import numpy as np
import torch

n = 10**7
dev = torch.device("cuda", 0)
cr = torch.cuda.cudart()
a = np.random.default_rng(1).integers(0, 1 << 31, n, dtype=np.int64).astype(np.int32)
d = torch.empty(n, dtype=torch.int32, device=dev)
st = torch.cuda.current_stream()


def timeit(f, reps=10):
    for _ in range(2):
        f()
    torch.cuda.synchronize()
    ts = []
    for _ in range(reps):
        t0 = time.perf_counter()
        f()
        torch.cuda.synchronize()
        ts.append(time.perf_counter() - t0)
    return 1e3 * float(np.median(ts))


pinned = torch.empty(n, dtype=torch.int32, pin_memory=True)
pinned.numpy()[:] = a
print("pinned H2D ms", timeit(lambda: d.copy_(pinned, non_blocking=True)))
print("pinned D2H ms", timeit(lambda: pinned.copy_(d, non_blocking=True)))
ta = torch.from_numpy(a)
print("pageable H2D (torch) ms", timeit(lambda: d.copy_(ta)))
print("pageable D2H (torch .cpu()) ms", timeit(lambda: d.cpu()))
out = np.empty_like(a)
tout = torch.from_numpy(out)
print("pageable D2H into existing (torch copy_) ms", timeit(lambda: tout.copy_(d)))
print("numpy memcpy 40MB ms", timeit(lambda: np.copyto(out, a)))


def reg():
    r = cr.cudaHostRegister(a.ctypes.data, a.nbytes, 0)
    assert int(r) == 0, r
    d.copy_(ta, non_blocking=True)
    torch.cuda.synchronize()
    cr.cudaHostUnregister(a.ctypes.data)


print("register+H2D+unregister ms", timeit(reg))


def reg_only():
    cr.cudaHostRegister(a.ctypes.data, a.nbytes, 0)
    cr.cudaHostUnregister(a.ctypes.data)


print("register+unregister only ms", timeit(reg_only))
cr.cudaHostRegister(a.ctypes.data, a.nbytes, 0)
print("registered H2D ms", timeit(lambda: d.copy_(ta, non_blocking=True)))
print("registered D2H ms", timeit(lambda: ta.copy_(d, non_blocking=True)))
cr.cudaHostUnregister(a.ctypes.data)
# freshly-written source (what a caller that just produced its data has)
def fresh_h2d():
    np.copyto(a, out)
    d.copy_(ta)
print("fresh write + pageable H2D ms", timeit(fresh_h2d))
