"""Pure-Python model of the CUDA powersort pipeline -- TEST INFRASTRUCTURE.

Restates, step by step, what the kernels in paper_1805_04154_b200/csrc compute
(pair-type bits -> min-run chain via per-tile candidate tables -> midpoint keys
and node powers -> trie ranges -> depth via (mask, const) scans -> depth-parity
ping-pong merge schedule -> closed-form Metrics).  tests/test_device_model.py
checks it against the C oracle, which validates the *algorithm* of the device
path independently of CUDA.  Small inputs only.
"""

from __future__ import annotations

import numpy as np


def asc_bits(a):
    n = len(a)
    return (a[:-1] <= a[1:]) if n > 1 else np.zeros(0, dtype=bool)


def b_set(asc, n):
    """B = {k in [1, n-2] : asc_k != asc_{k-1}} U {n-1} (as a boolean array)."""
    B = np.zeros(n, dtype=bool)
    if n >= 3:
        B[1:n - 1] = asc[1:] != asc[:-1]
    if n >= 1:
        B[n - 1] = True
    return B


def nat_end(B, p):
    n = len(B)
    if p >= n - 1:
        return n - 1
    k = p + 1
    while not B[k]:
        k += 1
    return k


def chain_direct(B, n, w):
    starts = []
    p = 0
    while p < n:
        starts.append(p)
        p = max(nat_end(B, p) + 1, min(p + w, n))
    return starts


def chain_tiled(B, n, w, T):
    """Per-tile candidate tables + sequential composition (kernels K12a/K2b-e)."""
    ntiles = (n + T - 1) // T
    tables = []
    for t in range(ntiles):
        t0, t1 = t * T, min(n, (t + 1) * T)
        cands = [t0 + c for c in range(w)]
        cands.append(nat_end(B, t0 - 1) + 1 if t0 > 0 else t0)
        tab = []
        for q in cands:
            p, cnt = q, 0
            while p < t1:
                cnt += 1
                p = max(nat_end(B, p) + 1, min(p + w, n))
            if p - t1 < w:
                ex = p - t1
            else:
                assert p == nat_end(B, t1 - 1) + 1
                ex = w
            tab.append((ex, cnt, q))
        tables.append(tab)
    starts = []
    e = 0
    for t in range(ntiles):
        t1 = min(n, (t + 1) * T)
        p = tables[t][e][2]
        while p < t1:
            starts.append(p)
            p = max(nat_end(B, p) + 1, min(p + w, n))
        e = tables[t][e][0]
    return starts


def mid_keys(starts, n):
    s = list(starts) + [n]
    return [((s[i] + s[i + 1]) << 32) // (2 * n) for i in range(len(starts))]


def bitlen(x):
    return int(x).bit_length()


def powers_from_keys(K):
    return [33 - bitlen(K[j - 1] ^ K[j]) for j in range(1, len(K))]


def depth_by_scans(P):
    """la/ra via the (mask, const) scan; returns depth[j] (j=1..r-1), max stack."""
    m = len(P)
    bit = lambda p: 1 << (p - 1)
    la = [0] * (m + 1)
    ra = [0] * (m + 1)
    M = 0
    best = 0
    for j in range(1, m + 1):
        p = P[j - 1]
        la[j] = bin(M & (bit(p) - 1)).count("1")
        best = max(best, 1 + la[j])
        M = bit(p) | (M & (bit(p) - 1))
    M = 0
    for j in range(m, 0, -1):
        p = P[j - 1]
        ra[j] = bin(M & (bit(p) - 1)).count("1")
        M = bit(p) | (M & (bit(p) - 1))
    depth = [None] + [la[j] + ra[j] for j in range(1, m + 1)]
    return depth, best


def node_ranges(K, P):
    """Leaves [a, b] under boundary j: all leaves sharing K_j's (P_j - 1)-bit prefix."""
    r = len(K)
    rng = [None]
    for j in range(1, r):
        p = P[j - 1]
        shift = 32 - (p - 1)
        pre = K[j] >> shift
        a = j - 1
        while a - 1 >= 0 and (K[a - 1] >> shift) == pre:
            a -= 1
        b = j
        while b + 1 < r and (K[b + 1] >> shift) == pre:
            b += 1
        rng.append((a, b))
    return rng


def simulate(a, w=24, merge_kind="bitonic", tags=None, T=64):
    """Full model: returns (sorted keys, tags, metrics tuple, leaf starts, powers)."""
    a = np.array(a)
    n = len(a)
    if n <= 1:
        return a.copy(), None if tags is None else tags.copy(), (0, 0, n, 0), list(range(n)), []
    asc = asc_bits(a)
    B = b_set(asc, n)
    starts = chain_tiled(B, n, w, T)
    assert starts == chain_direct(B, n, w)
    r = len(starts)
    S = starts + [n]
    comps = 0
    buf = [a.copy(), a.copy()]
    tbuf = [tags.copy(), tags.copy()] if tags is not None else None
    # leaves: detection comparisons, reversal, insertion
    K = mid_keys(starts, n)
    P = powers_from_keys(K)
    depth, best = depth_by_scans(P) if r > 1 else ([None], 0)
    rngs = node_ranges(K, P) if r > 1 else [None]
    leaf_depth = []
    for i in range(r):
        if r == 1:
            leaf_depth.append(0)
            continue
        cand = []
        if i >= 1:
            cand.append((P[i - 1], depth[i]))
        if i + 1 <= r - 1:
            cand.append((P[i], depth[i + 1]))
        leaf_depth.append(max(cand)[1] + 1)
    for i in range(r):
        s, e = S[i], S[i + 1]
        ne = nat_end(B, s)
        L = ne - s + 1
        if s < n - 1:
            comps += (ne - s + 1) if ne < n - 1 else (ne - s)
        chunk = a[s:e].copy()
        tch = tags[s:e].copy() if tags is not None else None
        if s < n - 1 and not asc[s] and L >= 2:
            chunk[:L] = chunk[:L][::-1].copy()
            if tch is not None:
                tch[:L] = tch[:L][::-1].copy()
        if L < e - s:
            npre = max(1, L)
            for t in range(npre, e - s):
                g = int(np.count_nonzero(chunk[:t] > chunk[t]))
                comps += g + (1 if g < t else 0)
            order = np.argsort(chunk, kind="stable")
            chunk = chunk[order]
            if tch is not None:
                tch = tch[order]
        d = leaf_depth[i] % 2
        buf[d][s:e] = chunk
        if tbuf is not None:
            tbuf[d][s:e] = tch
    merge_cost = 0
    if r > 1:
        dmax = max(depth[1:])
        for d in range(dmax, -1, -1):
            for j in range(1, r):
                if depth[j] != d:
                    continue
                lo, hi = rngs[j]
                s, m, e = S[lo], S[j], S[hi + 1]
                src, dst = buf[(d + 1) % 2], buf[d % 2]
                L, R = src[s:m], src[m:e]
                merge_cost += e - s
                if merge_kind == "bitonic":
                    comps += e - s
                else:
                    pl = len(L) - 1 + int(np.count_nonzero(R < L[-1]))
                    pr = len(R) - 1 + int(np.count_nonzero(L <= R[-1]))
                    comps += min(pl, pr) + 1
                keys = np.concatenate([L, R])
                order = np.argsort(keys, kind="stable")
                dst[s:e] = keys[order]
                if tbuf is not None:
                    tt = np.concatenate([tbuf[(d + 1) % 2][s:m], tbuf[(d + 1) % 2][m:e]])
                    tbuf[d % 2][s:e] = tt[order]
    return buf[0], (tbuf[0] if tbuf else None), (merge_cost, comps, r, best), starts, P
