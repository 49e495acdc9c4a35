"""Seeded synthetic inputs for the five BASELINE configs (BASELINE.json).

The reference's own generators (reference ``gen.py:68-101``) emit permutations
of 1..n; BASELINE asks for other shapes, so these follow SURVEY.md Appendix B.
Every generator uses ``np.random.Generator(np.random.PCG64(seed))`` (the
reference's convention, ``gen.py:64-65``), one generator per array.  Config 5
is generated on the device in segment-aligned chunks (a 16 GiB host array is
not needed); it is identical for any GPU count.

Input synthesis is not part of the sort path: these may use numpy/torch freely.
"""

from __future__ import annotations

import math
from dataclasses import dataclass
from typing import Optional, Tuple

import numpy as np


def _rng(seed: int) -> np.random.Generator:
    return np.random.Generator(np.random.PCG64(seed))


def _geometric_bounds(rng: np.random.Generator, n: int, mean: float) -> np.ndarray:
    """Segment boundaries [0, b1, ..., n] with i.i.d. geometric lengths."""
    p = 1.0 / mean
    bounds = [0]
    pos = 0
    while pos < n:
        batch = rng.geometric(p, size=max(16, int(n / mean) + 16))
        cs = pos + np.cumsum(batch, dtype=np.int64)
        cut = np.searchsorted(cs, n, side="left")
        bounds.extend(cs[: cut].tolist())
        if cut < len(cs):
            bounds.append(n)
            pos = n
        else:
            pos = int(cs[-1])
    if bounds[-1] != n:
        bounds.append(n)
    return np.asarray(bounds, dtype=np.int64)


def config1(n: int = 1 << 20, seed: int = 1) -> np.ndarray:
    """Random permutation of 0..n-1 as int32: reference ``gen.random_permutation``
    (gen.py:68-73) shifted down by one."""
    return _rng(seed).permutation(n).astype(np.int32)


def config2(n: int = 10**7, seed: int = 1, mean: Optional[float] = None) -> np.ndarray:
    """Random runs: uniform int32 in [0, 2^31), geometric segments of mean
    sqrt(n), each sorted ascending (the last one truncated)."""
    rng = _rng(seed)
    keys = rng.integers(0, 1 << 31, size=n, dtype=np.int64).astype(np.int32)
    mean = float(round(math.sqrt(n))) if mean is None else float(mean)
    b = _geometric_bounds(rng, n, max(mean, 1.0))
    for s, e in zip(b[:-1], b[1:]):
        keys[s:e].sort()
    return keys


def config3(n: int = 1 << 24, seed: int = 1) -> np.ndarray:
    """Mixed-direction Zipf(1.2) segments capped at n/4: even segments sorted
    ascending, odd segments strictly descending (duplicates re-drawn)."""
    rng = _rng(seed)
    cap = max(1, n // 4)
    lens = []
    pos = 0
    while pos < n:  # lengths first, in batches
        z = np.minimum(rng.zipf(1.2, size=4096), cap)
        cs = pos + np.cumsum(z)
        cut = int(np.searchsorted(cs, n, side="left"))
        lens.extend(z[: cut].tolist())
        if cut < len(cs):
            lens.append(n - (int(cs[cut - 1]) if cut else pos))
            pos = n
        else:
            pos = int(cs[-1])
    lens = np.asarray(lens, dtype=np.int64)
    seg = np.repeat(np.arange(len(lens), dtype=np.int64), lens)
    desc = (seg & 1) == 1
    keys = rng.integers(0, 1 << 31, size=n, dtype=np.int64)
    # re-draw duplicates inside descending segments until they are distinct
    didx = np.nonzero(desc)[0]
    while len(didx):
        comp = (seg[didx] << 31) | keys[didx]
        order = np.argsort(comp)
        sc = comp[order]
        dup = np.zeros(len(didx), dtype=bool)
        dup[order[1:]] = (sc[1:] == sc[:-1])
        if not dup.any():
            break
        keys[didx[dup]] = rng.integers(0, 1 << 31, size=int(dup.sum()), dtype=np.int64)
    # ascending segments sort by key, descending ones by (2^31-1-key)
    mask = (1 << 31) - 1
    sc = np.sort((seg << 31) | np.where(desc, mask - keys, keys))
    low = sc & mask
    return np.where(((sc >> 31) & 1) == 1, mask - low, low).astype(np.int32)


def config4(n: int = 10**8, seed: int = 1, mean: float = 1024.0) -> Tuple[np.ndarray, np.ndarray]:
    """Stability stress: int32 keys over 16 values, int32 payload = arange(n),
    geometric(mean 1024) segments each sorted stably by key with the payload."""
    rng = _rng(seed)
    keys = rng.integers(0, 16, size=n, dtype=np.int64).astype(np.int32)
    payload = np.arange(n, dtype=np.int32)
    b = _geometric_bounds(rng, n, mean)
    for s, e in zip(b[:-1], b[1:]):
        seg = keys[s:e]
        order = np.argsort(seg, kind="stable")
        keys[s:e] = seg[order]
        payload[s:e] = payload[s:e][order]
    return keys, payload


CONFIG5_N = 1 << 31
CONFIG5_CHUNK = 1 << 24


def config5_bounds(n: int = CONFIG5_N, seed: int = 1, mean: float = float(1 << 16)) -> np.ndarray:
    """Segment boundaries of config 5 (host, small: ~n/mean entries)."""
    return _geometric_bounds(_rng(seed), n, mean)


def _config5_raw(lo: int, hi: int, n: int, seed: int, device, out):
    """Raw (unsorted) values of positions [lo, hi): per-chunk PCG64-seeded torch
    generators over fixed 2^24-element chunks, so any range of the array is the
    same bytes whatever range or GPU count it is generated for."""
    import torch

    g = torch.Generator(device=device)
    c = (lo // CONFIG5_CHUNK) * CONFIG5_CHUNK
    while c < hi:
        c1 = min(n, c + CONFIG5_CHUNK)
        g.manual_seed(int(_rng(seed * 1_000_003 + c // CONFIG5_CHUNK).integers(0, 1 << 62)))
        vals = torch.randint(0, (1 << 63) - 1, (c1 - c,), generator=g, device=device, dtype=torch.int64)
        a0, a1 = max(lo, c), min(hi, c1)
        out[a0 - lo: a1 - lo] = vals[a0 - c: a1 - c]
        c = c1
    return out


def _sort_segments(buf, b: np.ndarray, base: int):
    """Sort every segment [b[i], b[i+1]) of buf (positions offset by base) in
    windows of ~one chunk (two stable sorts: by value, then by segment)."""
    import torch

    device = buf.device
    bt = torch.as_tensor(b, device=device)
    i, nb = 0, len(b) - 1
    while i < nb:
        j = i + 1
        while j < nb and b[j + 1] - b[i] <= CONFIG5_CHUNK:
            j += 1
        s, e = int(b[i]), int(b[j])
        seg_id = torch.bucketize(torch.arange(s, e, device=device), bt[i + 1: j + 1], right=True)
        vals, idx = torch.sort(buf[s - base: e - base], stable=True)
        _, order = torch.sort(seg_id[idx], stable=True)
        buf[s - base: e - base] = vals[order]
        i = j


def config5_range(lo: int, hi: int, n: int = CONFIG5_N, seed: int = 1, device="cuda", out=None,
                  mean: float = float(1 << 16), bounds: Optional[np.ndarray] = None):
    """Positions [lo, hi) of the config-5 array on the device: uniform int64 in
    [0, 2^63), geometric segments of mean 2^16, each sorted ascending.  The
    segments overlapping the range are generated whole and sorted, then the
    range is cut out: shards of any GPU count concatenate to the same array."""
    import torch

    b = config5_bounds(n, seed, mean) if bounds is None else bounds
    i0 = int(np.searchsorted(b, lo, side="right")) - 1
    j1 = int(np.searchsorted(b, hi, side="left"))
    s0, e1 = int(b[i0]), int(b[j1])
    if out is None:
        out = torch.empty(hi - lo, dtype=torch.int64, device=device)
    whole = (s0, e1) == (lo, hi)
    buf = out if whole else torch.empty(e1 - s0, dtype=torch.int64, device=device)
    _config5_raw(s0, e1, n, seed, device, buf)
    _sort_segments(buf, b[i0: j1 + 1], s0)
    if not whole:
        out.copy_(buf[lo - s0: hi - s0])
    return out


def config5_device(n: int = CONFIG5_N, seed: int = 1, device="cuda", out=None,
                   mean: float = float(1 << 16)):
    """The whole config-5 array on the device (config5_range(0, n))."""
    return config5_range(0, n, n, seed, device, out, mean)


@dataclass(frozen=True)
class Workload:
    name: str
    n: int
    key_dtype: str
    tag_dtype: Optional[str]
    description: str


WORKLOADS = {
    1: Workload("cfg1-perm-2^20-int32", 1 << 20, "int32", None,
                "random permutation of 0..n-1 (Fisher-Yates, PCG64 seed)"),
    2: Workload("cfg2-random-runs-1e7-int32", 10**7, "int32", None,
                "uniform int32 keys, geometric segments of mean sqrt(n), sorted ascending"),
    3: Workload("cfg3-zipf-mixed-2^24-int32", 1 << 24, "int32", None,
                "Zipf(1.2) segments capped at n/4, alternating ascending / strictly descending"),
    4: Workload("cfg4-stability-1e8-int32+int32", 10**8, "int32", "int32",
                "16-valued int32 keys + int32 index payload, geometric mean-1024 stable runs"),
    5: Workload("cfg5-int64-2^31", 1 << 31, "int64", None,
                "uniform int64 in [0,2^63), geometric segments of mean 2^16"),
}


def generate(cfg: int, n: Optional[int] = None, seed: int = 1):
    """Host arrays (keys, tags-or-None) for configs 1-4 at size n."""
    if cfg == 1:
        return config1(n or (1 << 20), seed), None
    if cfg == 2:
        return config2(n or 10**7, seed), None
    if cfg == 3:
        return config3(n or (1 << 24), seed), None
    if cfg == 4:
        return config4(n or 10**8, seed)
    raise ValueError("config 5 is generated on the device (config5_device)")
