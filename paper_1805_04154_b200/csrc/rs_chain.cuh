// rs_chain.cuh -- run detection and the min-run leaf chain (powersort's detect()).
//
// Reference: sorters.py:462-470 (detect: natural run from `start`, extended to
// min_run_len by insertion sort), runcore.py:137-159 (find_run_right: maximal
// weakly-increasing or strictly-decreasing run).
//
// Closed form: with asc_k = a[k] <= a[k+1] and
// B = {k in [1,n-2] : asc_k != asc_{k-1}} U {n-1}, natEnd(p) = min{k in B, k > p},
// and the leaf chain is p_0 = 0, p_{i+1} = max(natEnd(p_i)+1, min(p_i+w, n)).
// The chain is sequential; we make it parallel with per-tile candidate tables:
// the first chain position >= a tile start t0 is one of {t0..t0+w-1} or
// natEnd(t0-1)+1 (candidate index w).  Each tile maps candidate -> (exit
// candidate of the next tile, #leaves in this tile); tables are composed per
// group, then sequentially across groups, then leaves are emitted per tile.
#pragma once
#include "rs_common.cuh"

namespace rs {

// Build the B-words (run-boundary bits), zero word 0 when it holds only
// positions before the window of interest, and the next-nonzero index array.
// Executed by one warp over nwords words.  asc[] must hold the window's asc words
// and `prev0` the asc word just before the window (0 when none).
__device__ inline void build_bwords_warp(const uint32_t* asc, uint32_t prev0, uint32_t* bw,
                                         uint16_t* nz, int nwords, pos_t base, pos_t n,
                                         bool zero_first) {
  int lane = threadIdx.x & 31;
  for (int q = lane; q < nwords; q += 32) {
    uint32_t x = asc[q];
    uint32_t prev = q > 0 ? asc[q - 1] : prev0;
    uint32_t b = x ^ ((x << 1) | (prev >> 31));
    pos_t p0 = base + 32 * pos_t(q);
    if (p0 == 0) b &= ~1u;  // B_0 undefined (k >= 1)
    // positions >= n-1: B_{n-1} = 1, beyond: 0
    pos_t last = n - 1;
    if (last < p0) b = 0;
    else if (last < p0 + 32) {
      int bit = int(last - p0);
      b &= (bit == 31) ? 0xffffffffu : ((1u << (bit + 1)) - 1);
      b |= 1u << bit;
    }
    if (q == 0 && zero_first) b = 0;
    bw[q] = b;
  }
  __syncwarp();
  // next-nonzero word index, scanning chunks of 32 from the end
  int carry = nwords;
  int nchunks = (nwords + 31) >> 5;
  for (int c = nchunks - 1; c >= 0; --c) {
    int q = c * 32 + lane;
    bool nzb = (q < nwords) && bw[q] != 0;
    uint32_t bal = __ballot_sync(0xffffffffu, nzb);
    uint32_t m = bal & (0xffffffffu << lane);
    if (q < nwords) nz[q] = (uint16_t)(m ? c * 32 + __ffs(m) - 1 : carry);
    if (bal) carry = c * 32 + __ffs(bal) - 1;
  }
  __syncwarp();
}

// natEnd(p) within the window; kInf when beyond it.
__device__ __forceinline__ pos_t nat_end_win(const uint32_t* bw, const uint16_t* nz, int nwords,
                                             pos_t base, pos_t n, pos_t p) {
  if (p >= n - 1) return n - 1;
  return next_set_bit(bw, nz, nwords, base, p + 1);
}

__device__ __forceinline__ pos_t chain_next(pos_t p, pos_t ne, int w, pos_t n) {
  pos_t b = p + w < n ? p + w : n;
  pos_t a = ne + 1;
  return a > b ? a : b;
}

// Window of words [q0, q1) for chain tile `tile`.
__device__ __forceinline__ void chain_window(int64_t tile, pos_t n, int w, int64_t* q0, int64_t* q1,
                                             pos_t* t0, pos_t* t1, int ct = kChainT) {
  *t0 = tile * (pos_t)ct;
  *t1 = (*t0 + ct < n) ? *t0 + ct : n;
  int64_t total_words = (n + 31) >> 5;
  *q0 = *t0 == 0 ? 0 : ((*t0 - 1) >> 5);
  int64_t e = ((*t1 + w + 64) >> 5) + 1;
  *q1 = e < total_words ? e : total_words;
}

__host__ __device__ constexpr int kMaxWinWords(int w, int ct = kChainT) { return (ct + w + 96) / 32 + 4; }

// K1+K2a: pair-type bits for this tile (written to ascw) and the tile's
// candidate table.  One CTA per chain tile.
template <typename K>
__device__ void d_scan_table_tile(const K* __restrict__ a, pos_t n, int w, uint32_t* __restrict__ ascw,
                                  uint2* __restrict__ tables, int64_t tile) {
  extern __shared__ uint32_t smem_u32[];
  pos_t t0, t1;
  int64_t q0, q1;
  chain_window(tile, n, w, &q0, &q1, &t0, &t1);
  int nwords = int(q1 - q0);
  uint32_t* asc = smem_u32;
  uint32_t* bw = asc + nwords;
  uint16_t* nz = reinterpret_cast<uint16_t*>(bw + nwords);
  int lane = threadIdx.x & 31, wid = threadIdx.x >> 5, nw = blockDim.x >> 5;
  int64_t own0 = t0 >> 5, own1 = (t1 + 31) >> 5;
  // each warp handles runs of 8 consecutive words: 8 independent loads per lane
  constexpr int U = 8;
  for (int qb = wid * U; qb < nwords; qb += nw * U) {
    K v[U + 1];
#pragma unroll
    for (int u = 0; u <= U; ++u) {
      pos_t k = 32 * (q0 + qb + u) + lane;
      v[u] = (qb + u <= nwords && k < n && (u < U || lane == 0)) ? __ldcg(a + k) : K(0);
    }
#pragma unroll
    for (int u = 0; u < U; ++u) {
      int qi = qb + u;
      K nx = __shfl_down_sync(0xffffffffu, v[u], 1);
      K first_next = __shfl_sync(0xffffffffu, v[u + 1], 0);
      if (lane == 31) nx = first_next;
      pos_t k = 32 * (q0 + qi) + lane;
      bool bit = qi < nwords && (k < n - 1) && (v[u] <= nx);
      uint32_t word = __ballot_sync(0xffffffffu, bit);
      if (lane == 0 && qi < nwords) {
        int64_t q = q0 + qi;
        asc[qi] = word;
        if (q >= own0 && q < own1) ascw[q] = word;
      }
    }
  }
  __syncthreads();
  pos_t base = 32 * q0;
  if (wid == 0) build_bwords_warp(asc, 0u, bw, nz, nwords, base, n, q0 > 0 || t0 > 0);
  __syncthreads();
  // candidates
  for (int c = threadIdx.x; c <= w; c += blockDim.x) {
    pos_t p;
    if (c < w) p = t0 + c;
    else if (t0 == 0) p = 0;
    else {
      pos_t ne = nat_end_win(bw, nz, nwords, base, n, t0 - 1);
      p = ne >= kInf ? kInf : ne + 1;
    }
    uint32_t cnt = 0;
    while (p < t1) {
      ++cnt;
      pos_t ne = nat_end_win(bw, nz, nwords, base, n, p);
      if (ne >= kInf) { p = kInf; break; }
      p = chain_next(p, ne, w, n);
    }
    uint32_t ex;
    if (p >= kInf) ex = (uint32_t)w;
    else ex = (p - t1 < w) ? (uint32_t)(p - t1) : (uint32_t)w;
    tables[tile * (w + 1) + c] = make_uint2(ex, cnt);
  }
}

// K1+K2a with TMA, one chain tile per warp: the warp stages its key window in
// a warp-private shared-memory slice with one 1D bulk copy (mbarrier
// completion), derives the pair-type bits and B-words there, and its lanes
// walk the w+1 candidates.  16+ tiles are in flight per SM.
__host__ __device__ inline int chain_win_bytes(int w, int kb, int ct = kChainT) {
  return ((ct + w + 192) * kb + 16 + 127) / 128 * 128;
}
__host__ __device__ inline int chain_warp_bytes(int w, int kb, int ct = kChainT) {
  int maxw = kMaxWinWords(w, ct);
  return chain_win_bytes(w, kb, ct) + ((maxw * 8 + maxw * 2 + 127) / 128) * 128;
}

#ifndef RS_BITS_LPW
#define RS_BITS_LPW 1
#endif
template <typename K>
__device__ __forceinline__ void d_scan_tables_tma(const K* __restrict__ a, pos_t n, int w, uint32_t* __restrict__ ascw,
                                  uint2* __restrict__ tables, int64_t ntiles, int ct, DevMetrics* imet = nullptr) {
  extern __shared__ __align__(128) unsigned char smem_tab[];
  __shared__ __align__(8) uint64_t kbar[32];
  int lane = threadIdx.x & 31, wid = threadIdx.x >> 5, nw = blockDim.x >> 5;
  int maxw = kMaxWinWords(w, ct);
  unsigned char* kbuf = smem_tab + (size_t)wid * chain_warp_bytes(w, sizeof(K), ct);
  uint32_t* asc = reinterpret_cast<uint32_t*>(kbuf + chain_win_bytes(w, sizeof(K), ct));
  uint32_t* bw = asc + maxw;
  uint16_t* nz = reinterpret_cast<uint16_t*>(bw + maxw);
  if (lane == 0) {
    mbar_init(&kbar[wid], 1);
    mbar_fence_init();
  }
  __syncwarp();
  uint32_t ph = 0;
#ifdef RS_INSTR
  unsigned long long c_wait = 0, c_bits = 0, c_bw = 0, c_walk = 0;
#endif
  // The key window is only read by the pair-bit step: the next tile's bulk
  // copy is issued right after it, overlapping the B-words and the walks.
  auto issue = [&](int64_t tl) -> int32_t {
    pos_t u0, u1;
    int64_t r0, r1;
    chain_window(tl, n, w, &r0, &r1, &u0, &u1, ct);
    pos_t e0 = 32 * r0, e1 = 32 * r1 + 1 < n ? 32 * r1 + 1 : n;
    int32_t ko = 0;
    if (lane == 0) {
      uintptr_t a0 = reinterpret_cast<uintptr_t>(a + e0), a1 = reinterpret_cast<uintptr_t>(a + e1);
      uint32_t bytes = (uint32_t)(((a1 + 15) & ~(uintptr_t)15) - (a0 & ~(uintptr_t)15));
      fence_proxy_async_smem();
      mbar_arrive_tx(&kbar[wid], bytes);
      tma_window(kbuf, a, e0, e1, sizeof(K), &kbar[wid], &ko);
    }
    return __shfl_sync(0xffffffffu, ko, 0);
  };
  const int64_t tstride = (int64_t)gridDim.x * nw;
  int32_t koff_next = 0;
  if ((int64_t)blockIdx.x * nw + wid < ntiles) koff_next = issue((int64_t)blockIdx.x * nw + wid);
  for (int64_t tile = (int64_t)blockIdx.x * nw + wid; tile < ntiles; tile += tstride) {
#ifdef RS_INSTR
    unsigned long long c0 = clock64();
#endif
    pos_t t0, t1;
    int64_t q0, q1;
    chain_window(tile, n, w, &q0, &q1, &t0, &t1, ct);
    int nwords = int(q1 - q0);
    const int32_t koff = koff_next;
    mbar_wait(&kbar[wid], ph);
    ph ^= 1u;
#ifdef RS_INSTR
    unsigned long long c1 = clock64();
    c_wait += c1 - c0;
#endif
    const K* sk = reinterpret_cast<const K*>(kbuf) + koff;  // element 32*q0
    int64_t own0 = t0 >> 5, own1 = (t1 + 31) >> 5;
#if RS_BITS_LPW
    // one pair-type word per lane: lane l builds word wb+l from its 33 keys,
    // visiting them in the rotated order j = (l + k) mod 32 so the 32 lanes
    // hit 32 different banks; no shuffles, 32 independent compares per lane
    for (int wb = 0; wb < nwords; wb += 32) {
      const int wi = wb + lane;
      if (wi < nwords) {
        const K* p = sk + 32 * wi;
        const pos_t p0 = 32 * (q0 + wi);
        uint32_t w4[4] = {0u, 0u, 0u, 0u};  // independent accumulators: no 32-long OR chain
#pragma unroll
        for (int k = 0; k < 32; ++k) {
          const int j = (lane + k) & 31;
          w4[k & 3] |= (uint32_t)(p[j] <= p[j + 1]) << j;
        }
        uint32_t word = (w4[0] | w4[1]) | (w4[2] | w4[3]);
        const pos_t rem = (n - 1) - p0;  // pairs p0 + j with j < rem lie before n - 1
        if (rem < 32) word &= rem <= 0 ? 0u : ((1u << rem) - 1u);
        asc[wi] = word;
        const int64_t q = q0 + wi;
        if (q >= own0 && q < own1) ascw[q] = word;
      }
    }
#else
    constexpr int VEC = 16 / sizeof(K);  // elements per 16B lane load = words per warp load
    constexpr int LPW = 32 / VEC;        // lanes per word
    if (koff % VEC == 0) {
      // vector path: one LDS.128 per lane covers VEC words per warp step;
      // steps are independent, unrolled so their shuffle chains overlap
#pragma unroll 4
      for (int vb = 0; vb < nwords; vb += VEC) {
        const uint4 raw = reinterpret_cast<const uint4*>(sk + 32 * vb)[lane];
        const K* x = reinterpret_cast<const K*>(&raw);
        K first = x[0];
        K nxt = __shfl_down_sync(0xffffffffu, first, 1);
        if (lane == 31) nxt = sk[32 * vb + 32 * VEC];
        // pairs k0 + i (i < lim) lie before n - 1: one 64-bit clamp instead of VEC compares
        pos_t rem = (n - 1) - (32 * (q0 + vb) + (pos_t)lane * VEC);
        int lim = rem <= 0 ? 0 : (rem >= VEC ? VEC : (int)rem);
        uint32_t nib = 0;
#pragma unroll
        for (int i = 0; i < VEC; ++i) {
          K cur = x[i];
          K nx = i + 1 < VEC ? x[i + 1] : nxt;
          nib |= (uint32_t)(i < lim && cur <= nx) << i;
        }
        uint32_t word = nib << ((lane % LPW) * VEC);
#pragma unroll
        for (int o = 1; o < LPW; o <<= 1) word |= __shfl_xor_sync(0xffffffffu, word, o);
        int wi = vb + lane / LPW;
        if ((lane % LPW) == 0 && wi < nwords) {
          int64_t q = q0 + wi;
          asc[wi] = word;
          if (q >= own0 && q < own1) ascw[q] = word;
        }
      }
    } else
    for (int qi = 0; qi < nwords; ++qi) {
      pos_t k = 32 * (q0 + qi) + lane;
      int rel = 32 * qi + lane;
      bool bit = false;
      if (k < n - 1) bit = sk[rel] <= sk[rel + 1];
      uint32_t word = __ballot_sync(0xffffffffu, bit);
      if (lane == 0) {
        int64_t q = q0 + qi;
        asc[qi] = word;
        if (q >= own0 && q < own1) ascw[q] = word;
      }
    }
#endif
    __syncwarp();
    if (tile + tstride < ntiles) koff_next = issue(tile + tstride);  // the window has been read
#ifdef RS_INSTR
    unsigned long long c2 = clock64();
    c_bits += c2 - c1;
#endif
    pos_t base = 32 * q0;
    build_bwords_warp(asc, 0u, bw, nz, nwords, base, n, t0 > 0);
#ifdef RS_INSTR
    unsigned long long c3 = clock64();
    c_bw += c3 - c2;
#endif
    for (int c = lane; c <= w; c += 32) {
      pos_t p;
      if (c < w) p = t0 + c;
      else if (t0 == 0) p = 0;
      else {
        pos_t ne = nat_end_win(bw, nz, nwords, base, n, t0 - 1);
        p = ne >= kInf ? kInf : ne + 1;
      }
      uint32_t cnt = 0;
      while (p < t1) {
        ++cnt;
        pos_t ne = nat_end_win(bw, nz, nwords, base, n, p);
        if (ne >= kInf) { p = kInf; break; }
        p = chain_next(p, ne, w, n);
      }
      uint32_t ex;
      if (p >= kInf) ex = (uint32_t)w;
      else ex = (p - t1 < w) ? (uint32_t)(p - t1) : (uint32_t)w;
      tables[tile * (w + 1) + c] = make_uint2(ex, cnt);
    }
    __syncwarp();
#ifdef RS_INSTR
    c_walk += clock64() - c3;
#endif
  }
#ifdef RS_INSTR
  if (lane == 0 && imet) {  // max over warps of the per-part cycle sums
    atomicMax(&imet->prep_ts[12], c_wait);
    atomicMax(&imet->prep_ts[13], c_bits);
    atomicMax(&imet->prep_ts[14], c_bw);
    atomicMax(&imet->prep_ts[15], c_walk);
  }
#endif
}

// K2b: compose the tables of each group of kChainGroup tiles.
// out[g*(w+1)+c] = (exit candidate after the group, #leaves) starting at candidate c.
__device__ void d_group_compose(const uint2* __restrict__ tables, int64_t ntiles, int w, int batch,
                                uint2* __restrict__ gtab, int64_t g) {
  extern __shared__ uint2 stab[];
  int W1 = w + 1;
  uint32_t* cur = reinterpret_cast<uint32_t*>(stab + (size_t)batch * W1);
  uint32_t* cnt = cur + W1;
  int64_t k0 = g * kChainGroup, k1 = k0 + kChainGroup < ntiles ? k0 + kChainGroup : ntiles;
  for (int c = threadIdx.x; c < W1; c += blockDim.x) { cur[c] = c; cnt[c] = 0; }
  for (int64_t kb = k0; kb < k1; kb += batch) {
    int nb = int((k1 - kb) < batch ? (k1 - kb) : batch);
    __syncthreads();
    copy_g2s(stab, tables + kb * W1, nb * W1, threadIdx.x, blockDim.x);
    __syncthreads();
    for (int c = threadIdx.x; c < W1; c += blockDim.x) {
      uint32_t e = cur[c], s = cnt[c];
      for (int k = 0; k < nb; ++k) {
        uint2 t = stab[k * W1 + e];
        s += t.y;
        e = t.x;
      }
      cur[c] = e;
      cnt[c] = s;
    }
  }
  __syncthreads();
  for (int c = threadIdx.x; c < W1; c += blockDim.x) gtab[g * W1 + c] = make_uint2(cur[c], cnt[c]);
}

// K2c: one CTA walks the group tables from candidate 0 of tile 0, recording each
// group's entry candidate and leaf offset; writes r and the start sentinel.
__device__ void d_group_entries(const uint2* __restrict__ gtab, int64_t ngroups, int w, int batch,
                                uint32_t* __restrict__ gentry, uint64_t* __restrict__ goff,
                                pos_t* __restrict__ leaf_start, pos_t n, int64_t r_max,
                                DevMetrics* __restrict__ met) {
  extern __shared__ uint2 stab[];
  int W1 = w + 1;
  __shared__ uint32_t s_e;
  __shared__ unsigned long long s_off;
  if (threadIdx.x == 0) { s_e = 0; s_off = 0; }
  for (int64_t gb = 0; gb < ngroups; gb += batch) {
    int nb = int((ngroups - gb) < batch ? (ngroups - gb) : batch);
    __syncthreads();
    copy_g2s(stab, gtab + gb * W1, nb * W1, threadIdx.x, blockDim.x);
    __syncthreads();
    if (threadIdx.x == 0) {
      uint32_t e = s_e;
      unsigned long long off = s_off;
      for (int k = 0; k < nb; ++k) {
        gentry[gb + k] = e;
        goff[gb + k] = off;
        uint2 t = stab[k * W1 + e];
        off += t.y;
        e = t.x;
      }
      s_e = e;
      s_off = off;
    }
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    unsigned long long r = s_off;
    if ((int64_t)r > r_max) { met->error = 1; r = r_max; }
    met->n_leaves = r;
    met->runs_detected = r;
    leaf_start[r] = n;
  }
}

// K2d: per group, walk the tile tables to get each tile's entry and leaf offset
// (tables staged through shared memory in batches).
__device__ void d_tile_entries(const uint2* __restrict__ tables, int64_t ntiles, int w, int batch,
                               const uint32_t* __restrict__ gentry, const uint64_t* __restrict__ goff,
                               uint32_t* __restrict__ tentry, uint64_t* __restrict__ toff, int64_t g) {
  extern __shared__ uint2 stab[];
  __shared__ uint32_t s_e2;
  __shared__ unsigned long long s_off2;
  int W1 = w + 1;
  int64_t k0 = g * kChainGroup, k1 = k0 + kChainGroup < ntiles ? k0 + kChainGroup : ntiles;
  if (threadIdx.x == 0) { s_e2 = gentry[g]; s_off2 = goff[g]; }
  for (int64_t kb = k0; kb < k1; kb += batch) {
    int nb = int((k1 - kb) < batch ? (k1 - kb) : batch);
    __syncthreads();
    copy_g2s(stab, tables + kb * W1, nb * W1, threadIdx.x, blockDim.x);
    __syncthreads();
    if (threadIdx.x == 0) {
      uint32_t e = s_e2;
      unsigned long long off = s_off2;
      for (int k = 0; k < nb; ++k) {
        tentry[kb + k] = e;
        toff[kb + k] = off;
        uint2 t = stab[k * W1 + e];
        off += t.y;
        e = t.x;
      }
      s_e2 = e;
      s_off2 = off;
    }
  }
}

// K2e: one warp per tile re-walks the chain from the tile's true entry and emits
// leaves: start position and info = min(natural run length, w) | desc << 31.
__device__ __forceinline__ void d_emit_tile(const uint32_t* __restrict__ ascw, pos_t n, int w, const uint32_t* __restrict__ tentry,
                            const uint64_t* __restrict__ toff, int64_t r_max, pos_t* __restrict__ leaf_start,
                            uint32_t* __restrict__ leaf_info, int64_t tile, int ct) {
  extern __shared__ uint32_t smem_u32[];
  int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  int maxw = kMaxWinWords(w, ct);
  uint32_t* asc = smem_u32 + (size_t)wid * (maxw * 2 + (maxw + 1) / 2 + 1);
  uint32_t* bw = asc + maxw;
  uint16_t* nz = reinterpret_cast<uint16_t*>(bw + maxw);
  pos_t t0, t1;
  int64_t q0, q1;
  chain_window(tile, n, w, &q0, &q1, &t0, &t1, ct);
  int nwords = int(q1 - q0);
  {
    uint32_t v[4];
#pragma unroll
    for (int u = 0; u < 4; ++u) {
      int q = lane + 32 * u;
      v[u] = q < nwords ? __ldcg(ascw + q0 + q) : 0u;
    }
    for (int q = lane + 128; q < nwords; q += 32) asc[q] = __ldcg(ascw + q0 + q);
#pragma unroll
    for (int u = 0; u < 4; ++u) {
      int q = lane + 32 * u;
      if (q < nwords) asc[q] = v[u];
    }
  }
  uint32_t prev0 = q0 > 0 ? __ldcg(ascw + q0 - 1) : 0u;
  __syncwarp();
  pos_t base = 32 * q0;
  build_bwords_warp(asc, prev0, bw, nz, nwords, base, n, false);
  if (lane == 0) {
    uint32_t e = tentry[tile];
    uint64_t off = toff[tile];
    pos_t p;
    if (e < (uint32_t)w) p = t0 + e;
    else if (t0 == 0) p = 0;
    else {
      pos_t ne = nat_end_win(bw, nz, nwords, base, n, t0 - 1);
      p = ne >= kInf ? kInf : ne + 1;
    }
    while (p < t1) {
      pos_t ne = nat_end_win(bw, nz, nwords, base, n, p);
      uint32_t nl;
      if (ne >= kInf) nl = (uint32_t)w;
      else {
        pos_t L = ne - p + 1;
        nl = L < w ? (uint32_t)L : (uint32_t)w;
      }
      uint32_t desc = 0;
      if (p < n - 1) {
        pos_t rel = p - base;
        desc = ((asc[rel >> 5] >> (rel & 31)) & 1u) ? 0u : 1u;
      }
      if ((int64_t)off < r_max) {
        leaf_start[off] = p;
        leaf_info[off] = nl | (desc << 31);
      }
      ++off;
      if (ne >= kInf) break;
      p = chain_next(p, ne, w, n);
    }
  }
  __syncwarp();  // the warp's smem window is reused for its next tile
}

}  // namespace rs
