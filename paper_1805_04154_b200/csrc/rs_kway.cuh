// rs_kway.cuh -- the cross-GPU stable merge of sharded powersort.
//
// An array sharded contiguously over W ranks is sorted shard by shard; the
// global order the reference defines for the concatenation is (key, shard,
// position in shard), because the reference's merges send ties to the left
// run (runcore.py:262-263) and the shards are the concatenation's left-to-right
// pieces.  Rank g owns output positions [t_g, t_{g+1}) of that order.
//
// Three kernels, all reading the W sorted shards through plain device
// pointers -- local buffers, or peer shards mapped over NVLink (CUDA IPC), in
// which case the exchange IS the merge's input stream (no staging copy):
//
//  k_corank    exact multi-sequence selection: for a global rank t, the split
//              vector c with sum(c) = t and shard i contributing its first c_i
//              elements.  Per-shard brackets [L_i, H_i] shrink by evaluating
//              pivots p = (key, shard j, position q) inside them: with
//              cnt_i(p) = #elements of shard i preceding p (upper_bound for
//              i < j, lower_bound for i > j, q for i = j) and C = sum cnt_i,
//              C < t  => p is among the first t:  L_i >= cnt_i (+1 for i = j);
//              C >= t => the first t precede p:   H_i <= cnt_i.
//              Every bracket shrinks by the pivot density each round.
//  k_kway_pivots  every S-th element of each shard's range becomes a pivot; its
//              split vector (one warp per pivot, lane = shard) cuts the rank's
//              output into work items of at most W*S elements, ordered by the
//              pivots' global positions (no sort needed: a pivot's index is the
//              number of pivots preceding it, read off its own counts).
//  k_kway_merge   persistent CTAs claim work items and stream a W-way merge of
//              them: per step, the next K outputs are the first K of a pairwise
//              merge tree over per-shard shared-memory windows (ties to the
//              lower shard at every level => the (key, shard, position) order),
//              with the windows refilled by cp.async one step ahead.
#pragma once
#include "rs_common.cuh"

namespace rs {

constexpr int kKwayMaxW = 8;  // ranks of one NVSwitch node

struct KwayShards {
  const void* keys[kKwayMaxW];
  const void* tags[kKwayMaxW];
  int64_t lo[kKwayMaxW];  // range [lo, hi) of each shard taking part
  int64_t hi[kKwayMaxW];
  int w;
};

// #elements of `a[lo..hi)` that precede pivot key `kp` of shard j, for shard i:
// i < j -> elements <= kp, i > j -> elements < kp.
template <typename K>
__device__ __forceinline__ int64_t count_before(const K* a, int64_t lo, int64_t hi, K kp, bool le) {
  while (lo < hi) {
    int64_t mid = lo + ((hi - lo) >> 1);
    K v = a[mid];
    bool prec = le ? (v <= kp) : (v < kp);
    if (prec) lo = mid + 1;
    else hi = mid;
  }
  return lo;
}

// One block (kCorankThreads) per target; out[b * w + i] = c_i(targets[b]).
constexpr int kCorankThreads = 1024;
// With `dlens` (device, W shard lengths): shard i is [0, dlens[i]) and block
// b in {0, 1} computes target sum(dlens[0..g+b)) -- rank g's output range,
// entirely on the device (no host round trip between the local sorts and the
// merge).
template <typename K>
__global__ void __launch_bounds__(kCorankThreads) k_corank(KwayShards S, const int64_t* __restrict__ targets,
                                                           int64_t* __restrict__ out, const int64_t* __restrict__ dlens,
                                                           int g) {
  const int W = S.w;
  __shared__ int64_t sL[kKwayMaxW], sH[kKwayMaxW];
  __shared__ int64_t s_t;
  if (dlens) {
    if (threadIdx.x == 0) {
      int64_t t = 0;
      for (int i = 0; i < g + (int)blockIdx.x; ++i) t += dlens[i];
      s_t = t;
    }
  } else if (threadIdx.x == 0) {
    s_t = targets[blockIdx.x];
  }
  __syncthreads();
  if (dlens) {  // every thread's copy of the range table
    for (int i = 0; i < W; ++i) {
      S.lo[i] = 0;
      S.hi[i] = dlens[i];
    }
  }
  __shared__ int64_t s_cnt[kCorankThreads];
  __shared__ uint8_t s_flag[kCorankThreads];  // 1: below bracket (p in prefix), 2: above (p not in prefix)
  __shared__ int8_t s_cls[kCorankThreads];    // per pivot: +1 in prefix, -1 not, 0 exact, 2 inactive
  __shared__ int s_active;
  const int tid = threadIdx.x;
  const int64_t t = s_t;
  if (tid == 0) {
    int64_t total = 0;
    for (int i = 0; i < W; ++i) total += S.hi[i] - S.lo[i];
    for (int i = 0; i < W; ++i) {
      int64_t len = S.hi[i] - S.lo[i];
      int64_t l = t - (total - len);
      sL[i] = l > 0 ? l : 0;
      sH[i] = t < len ? t : len;
    }
  }
  int P = kCorankThreads / (W * W);  // pivots per shard per round
  if (P < 1) P = 1;
  const int V = P * W;  // pivots per round
  for (int round = 0; round < 128; ++round) {
    __syncthreads();
    if (tid == 0) {
      int act = 0;
      for (int i = 0; i < W; ++i) act |= sH[i] > sL[i];
      s_active = act;
    }
    __syncthreads();
    if (!s_active) break;
    const int v = tid / W, i = tid % W;
    bool live = v < V;
    int j = live ? v / P : 0, m = live ? v % P : 0;
    int64_t Lj = sL[j], Hj = sH[j];
    live = live && Hj > Lj;
    if (live) {
      const K* kj = reinterpret_cast<const K*>(S.keys[j]);
      int64_t q = Lj + ((int64_t)(m + 1) * (Hj - Lj)) / (P + 1);
      if (q >= Hj) q = Hj - 1;
      K kp = kj[S.lo[j] + q];
      int64_t c;
      uint8_t fl = 0;
      if (i == j) {
        c = q;
      } else {
        const K* ki = reinterpret_cast<const K*>(S.keys[i]);
        bool le = i < j;
        int64_t base = S.lo[i];
        c = count_before(ki, base + sL[i], base + sH[i], kp, le) - base;
        if (c == sL[i] && sL[i] > 0) {
          K x = ki[base + sL[i] - 1];
          if (!(le ? (x <= kp) : (x < kp))) fl = 1;
        }
        if (c == sH[i] && sH[i] < S.hi[i] - S.lo[i]) {
          K x = ki[base + sH[i]];
          if (le ? (x <= kp) : (x < kp)) fl = 2;
        }
      }
      s_cnt[tid] = c;
      s_flag[tid] = fl;
      if (i == 0) s_cls[v] = 0;
    } else if (v < V && i == 0) {
      s_cls[v] = 2;
    }
    __syncthreads();
    if (tid < V && s_cls[tid] != 2) {
      int64_t C = 0;
      int below = 0, above = 0;
      for (int k = 0; k < W; ++k) {
        C += s_cnt[tid * W + k];
        below |= s_flag[tid * W + k] == 1;
        above |= s_flag[tid * W + k] == 2;
      }
      int8_t cls;
      if (below) cls = 1;
      else if (above) cls = -1;
      else cls = C < t ? 1 : (C > t ? -1 : 0);
      s_cls[tid] = cls;
    }
    __syncthreads();
    if (tid < W) {
      int64_t l = sL[tid], h = sH[tid];
      for (int vv = 0; vv < V; ++vv) {
        int8_t cls = s_cls[vv];
        if (cls == 2) continue;
        int64_t c = s_cnt[vv * W + tid];
        if (cls >= 0) {  // in the prefix (or exact)
          int64_t nl = c + (cls == 1 && vv / P == tid ? 1 : 0);
          if (nl > l) l = nl;
        }
        if (cls <= 0 && c < h) h = c;
      }
      sL[tid] = l;
      sH[tid] = h;
    }
  }
  __syncthreads();
  if (tid < W) out[(int64_t)blockIdx.x * W + tid] = S.lo[tid] + sL[tid];
}

// Work-item boundaries.  Pivots: shard k's positions lo_k + m*S, m < npiv_k.
// bounds[(1 + index) * W + i] = split vector of pivot `index` (global order);
// bounds[0] = lo, bounds[(npiv + 1) * W] = hi.  One warp per pivot.
struct KwayPiv {
  int64_t off[kKwayMaxW + 1];  // prefix of per-shard pivot counts
};

// With `dsplit` (device, 2 x W: lo row, hi row) the ranges come from the
// co-rank kernel instead of S.lo / S.hi; the pivot table and its count are
// then derived here (npiv_cap bounds the grid-stride loop).  The number of
// work items (npiv + 1) goes to *nitems for the merge kernel.
template <typename K>
__global__ void __launch_bounds__(256) k_kway_pivots(KwayShards S, int64_t spacing, KwayPiv piv_off,
                                                     int64_t npiv, int64_t* __restrict__ bounds,
                                                     const int64_t* __restrict__ dsplit, int64_t* __restrict__ nitems) {
  const int W = S.w;
  const int lane = threadIdx.x & 31;
  if (dsplit) {
    npiv = 0;
    piv_off.off[0] = 0;
    for (int i = 0; i < W; ++i) {
      S.lo[i] = dsplit[i];
      S.hi[i] = dsplit[W + i];
      piv_off.off[i + 1] = piv_off.off[i] + (S.hi[i] - S.lo[i] + spacing - 1) / spacing;
    }
    npiv = piv_off.off[W];
  }
  if (blockIdx.x == 0 && threadIdx.x == 0) *nitems = npiv + 1;
  const int64_t warp = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int64_t nwarps = ((int64_t)gridDim.x * blockDim.x) >> 5;
  if (warp == 0 && lane < W) {
    bounds[lane] = S.lo[lane];
    bounds[(npiv + 1) * W + lane] = S.hi[lane];
  }
  for (int64_t p = warp; p < npiv; p += nwarps) {
    int k = 0;
    while (k + 1 < W && piv_off.off[k + 1] <= p) ++k;
    int64_t m = p - piv_off.off[k];
    int64_t q = S.lo[k] + m * spacing;
    K kp = reinterpret_cast<const K*>(S.keys[k])[q];
    int64_t c = 0, before = 0;
    if (lane < W) {
      if (lane == k) {
        c = q;
        before = m;
      } else {
        c = count_before(reinterpret_cast<const K*>(S.keys[lane]), S.lo[lane], S.hi[lane], kp, lane < k);
        before = (c - S.lo[lane] + spacing - 1) / spacing;
      }
    }
    int64_t idx = before;
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) idx += __shfl_xor_sync(0xffffffffu, idx, o);
    if (lane < W) bounds[(1 + idx) * W + lane] = c;
  }
}

template <typename K, int TB>
struct KwayCfg {
  static constexpr int THREADS = 512;
  static constexpr int kb = sizeof(K);
  // outputs per step: windows hold 2K elements per shard (K in use, K in flight)
  static constexpr int KS = (kb + TB) <= 8 ? 1024 : 512;
  static constexpr int WIN = 2 * KS;
  // level entries: key + 16-bit window slot (shard * WIN + index)
  __host__ __device__ static constexpr size_t win_bytes(int wp) { return (size_t)wp * WIN * (kb + TB); }
  __host__ __device__ static constexpr size_t lvl_bytes(int wp) {
    return (size_t)((wp / 2 > 1 ? wp / 2 : 1) + (wp / 4 > 1 ? wp / 4 : 1)) * KS * (kb + 2);
  }
  __host__ __device__ static constexpr size_t smem(int wp) { return win_bytes(wp) + lvl_bytes(wp) + 256; }
};

__device__ __forceinline__ void cp_async4(void* s, const void* g) {
  asm volatile("cp.async.ca.shared.global [%0], [%1], 4;" ::"r"(smem_addr(s)), "l"(g) : "memory");
}
__device__ __forceinline__ void cp_async8(void* s, const void* g) {
  asm volatile("cp.async.ca.shared.global [%0], [%1], 8;" ::"r"(smem_addr(s)), "l"(g) : "memory");
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;" ::: "memory"); }
__device__ __forceinline__ void cp_async_wait1() { asm volatile("cp.async.wait_group 1;" ::: "memory"); }
__device__ __forceinline__ void cp_async_wait0() { asm volatile("cp.async.wait_group 0;" ::: "memory"); }

template <int B>
__device__ __forceinline__ void cp_async_elem(void* s, const void* g) {
  if (B == 4) cp_async4(s, g);
  else cp_async8(s, g);
}

struct KwayMergeArgs {
  KwayShards S;
  const int64_t* bounds;  // (nitems + 1) x W split vectors; row 0 = the ranges' starts
  const int64_t* nitems;  // written by k_kway_pivots
  void* out_keys;
  void* out_tags;
  unsigned long long* claim;  // zeroed before launch
};

// Stable merge of two sorted sequences a (len na) and b (len nb), producing
// outputs [d0, d1) of their merge (ties to a).  Accessors return (key, slot).
template <typename K, typename FA, typename FB, typename FO>
__device__ __forceinline__ void merge_range(FA fa, int na, FB fb, int nb, int d0, int d1, FO emit) {
  // merge path: i = #a among the first d0 outputs
  int lo = d0 - nb > 0 ? d0 - nb : 0, hi = d0 < na ? d0 : na;
  while (lo < hi) {
    int i = (lo + hi) >> 1;  // take a[i] before b[d0-1-i]?  a[i] <= b[d0-1-i] (ties to a)
    K ai, bj;
    uint16_t s;
    fa(i, ai, s);
    fb(d0 - 1 - i, bj, s);
    if (ai <= bj) lo = i + 1;
    else hi = i;
  }
  int i = lo, j = d0 - lo;
  for (int d = d0; d < d1; ++d) {
    K ka = K(), kb2 = K();
    uint16_t sa = 0, sb = 0;
    if (i < na) fa(i, ka, sa);
    if (j < nb) fb(j, kb2, sb);
    bool ta = j >= nb || (i < na && ka <= kb2);
    if (ta) {
      emit(d, ka, sa);
      ++i;
    } else {
      emit(d, kb2, sb);
      ++j;
    }
  }
}

template <typename K, int TB>
__global__ void __launch_bounds__(512, 1) k_kway_merge(KwayMergeArgs A) {
  using C = KwayCfg<K, TB>;
  constexpr int KS = C::KS, WIN = C::WIN, T = C::THREADS;
  extern __shared__ __align__(16) unsigned char smem_kw[];
  const int W = A.S.w;
  int wp = 1;
  while (wp < W) wp <<= 1;
  K* wk = reinterpret_cast<K*>(smem_kw);                                   // [wp][WIN]
  unsigned char* wt = smem_kw + (size_t)wp * WIN * sizeof(K);               // [wp][WIN] tags
  unsigned char* lv = smem_kw + C::win_bytes(wp);                           // level buffers
  // level l (1..levels) list p: entries at lvl_off(l) + p*KS; keys then slots
  __shared__ int64_t s_cur[kKwayMaxW], s_loaded[kKwayMaxW], s_hi[kKwayMaxW];
  __shared__ int s_len[2 * kKwayMaxW];  // current level's list lengths (read side)
  __shared__ int s_cons[kKwayMaxW];
  __shared__ int64_t s_item, s_out;
  const int tid = threadIdx.x;
  int levels = 0;
  while ((1 << levels) < wp) ++levels;
  // level buffers: ping = wp/2 lists, pong = wp/4 lists (+1 for the wp = 2 case)
  K* lk[2];
  uint16_t* ls[2];
  {
    size_t n0 = (size_t)(wp / 2 > 0 ? wp / 2 : 1) * KS, n1 = (size_t)(wp / 4 > 0 ? wp / 4 : 1) * KS;
    lk[0] = reinterpret_cast<K*>(lv);
    lk[1] = lk[0] + n0;
    ls[0] = reinterpret_cast<uint16_t*>(lk[1] + n1);
    ls[1] = ls[0] + n0;
  }
  K* okeys = reinterpret_cast<K*>(A.out_keys);
  const int64_t nitems = *A.nitems;
  for (;;) {
    __syncthreads();
    if (tid == 0) s_item = (int64_t)atomicAdd(A.claim, 1ull);
    __syncthreads();
    const int64_t item = s_item;
    if (item >= nitems) break;
    if (tid < W) {
      int64_t lo = A.bounds[item * W + tid], hi = A.bounds[(item + 1) * W + tid];
      s_cur[tid] = lo;
      s_loaded[tid] = lo;
      s_hi[tid] = hi;
    }
    if (tid == 0) {
      int64_t o = 0;
      for (int i = 0; i < W; ++i) o += A.bounds[item * W + i] - A.bounds[i];
      s_out = o;
    }
    __syncthreads();
    int64_t remaining = 0;
    for (int i = 0; i < W; ++i) remaining += s_hi[i] - s_cur[i];
    // initial fill: two groups (the first K and the next K of every shard)
    for (int g = 0; g < 2; ++g) {
      for (int i = 0; i < W; ++i) {
        int64_t p0 = s_cur[i] + (int64_t)g * KS, p1 = p0 + KS;
        if (p1 > s_hi[i]) p1 = s_hi[i];
        const K* gk = reinterpret_cast<const K*>(A.S.keys[i]);
        for (int64_t p = p0 + tid; p < p1; p += T) {
          int sl = (int)(p & (WIN - 1));
          cp_async_elem<sizeof(K)>(&wk[i * WIN + sl], gk + p);
          if (TB) cp_async_elem<(TB ? TB : 4)>(wt + ((size_t)i * WIN + sl) * TB, (const unsigned char*)A.S.tags[i] + p * TB);
        }
      }
      cp_async_commit();
    }
    __syncthreads();
    if (tid < W) {
      int64_t e = s_cur[tid] + 2 * KS;
      s_loaded[tid] = e < s_hi[tid] ? e : s_hi[tid];
    }
    while (remaining > 0) {
      cp_async_wait1();  // every group but the latest has landed (this thread's)
      __syncthreads();
      const int nout = remaining < KS ? (int)remaining : KS;
      // level 1..levels: pairwise merges truncated to nout outputs
      for (int l = 1; l <= levels; ++l) {
        const int npairs = wp >> l;
        const int tpp = T / npairs;  // threads per pair
        const int pair = tid / tpp, r = tid % tpp;
        const int out_buf = (l - 1) & 1, in_buf = (l - 2) & 1;
        int la, lb;
        if (l == 1) {
          int a = 2 * pair, b = 2 * pair + 1;
          la = a < W ? (int)min((int64_t)KS, s_hi[a] - s_cur[a]) : 0;
          lb = b < W ? (int)min((int64_t)KS, s_hi[b] - s_cur[b]) : 0;
        } else {
          la = s_len[2 * pair];
          lb = s_len[2 * pair + 1];
        }
        int tot = la + lb < nout ? la + lb : nout;
        int per = (tot + tpp - 1) / tpp;
        int d0 = r * per, d1 = d0 + per < tot ? d0 + per : tot;
        K* ok = lk[out_buf] + (size_t)pair * KS;
        uint16_t* os = ls[out_buf] + (size_t)pair * KS;
        auto emit = [&](int d, K k, uint16_t s) {
          ok[d] = k;
          os[d] = s;
        };
        if (d0 < d1) {
          if (l == 1) {
            int a = 2 * pair, b = 2 * pair + 1;
            int64_t ca = a < W ? s_cur[a] : 0, cb = b < W ? s_cur[b] : 0;
            auto fa = [&](int x, K& k, uint16_t& s) {
              int sl = (int)((ca + x) & (WIN - 1));
              k = wk[a * WIN + sl];
              s = (uint16_t)(a * WIN + sl);
            };
            auto fb = [&](int x, K& k, uint16_t& s) {
              int sl = (int)((cb + x) & (WIN - 1));
              k = wk[b * WIN + sl];
              s = (uint16_t)(b * WIN + sl);
            };
            merge_range<K>(fa, la, fb, lb, d0, d1, emit);
          } else {
            const K* ak = lk[in_buf] + (size_t)(2 * pair) * KS;
            const uint16_t* as = ls[in_buf] + (size_t)(2 * pair) * KS;
            const K* bk = lk[in_buf] + (size_t)(2 * pair + 1) * KS;
            const uint16_t* bs = ls[in_buf] + (size_t)(2 * pair + 1) * KS;
            auto fa = [&](int x, K& k, uint16_t& s) { k = ak[x]; s = as[x]; };
            auto fb = [&](int x, K& k, uint16_t& s) { k = bk[x]; s = bs[x]; };
            merge_range<K>(fa, la, fb, lb, d0, d1, emit);
          }
        }
        __syncthreads();
        if (r == 0) s_len[pair] = tot;  // read side of the next level
        __syncthreads();
      }
      // wp == 1: the single shard's window is the output
      const K* fk = lk[(levels - 1) & 1];
      const uint16_t* fs = ls[(levels - 1) & 1];
      if (tid < W) s_cons[tid] = 0;
      __syncthreads();
      const int64_t ob = s_out;
      for (int d = tid; d < nout; d += T) {
        K k;
        uint16_t s;
        if (levels == 0) {
          int sl = (int)((s_cur[0] + d) & (WIN - 1));
          k = wk[sl];
          s = (uint16_t)sl;
        } else {
          k = fk[d];
          s = fs[d];
        }
        okeys[ob + d] = k;
        if (TB == 4)
          reinterpret_cast<uint32_t*>(A.out_tags)[ob + d] = *reinterpret_cast<const uint32_t*>(wt + (size_t)s * 4);
        else if (TB == 8)
          reinterpret_cast<uint64_t*>(A.out_tags)[ob + d] = *reinterpret_cast<const uint64_t*>(wt + (size_t)s * 8);
        atomicAdd(&s_cons[s / WIN], 1);
      }
      __syncthreads();
      if (tid < W) s_cur[tid] += s_cons[tid];
      if (tid == 0) s_out = ob + nout;
      remaining -= nout;
      __syncthreads();
      // refill: [loaded, min(cur + 2K, hi)) into the slots just consumed
      for (int i = 0; i < W; ++i) {
        int64_t p0 = s_loaded[i], p1 = s_cur[i] + 2 * KS;
        if (p1 > s_hi[i]) p1 = s_hi[i];
        const K* gk = reinterpret_cast<const K*>(A.S.keys[i]);
        for (int64_t p = p0 + tid; p < p1; p += T) {
          int sl = (int)(p & (WIN - 1));
          cp_async_elem<sizeof(K)>(&wk[i * WIN + sl], gk + p);
          if (TB) cp_async_elem<(TB ? TB : 4)>(wt + ((size_t)i * WIN + sl) * TB, (const unsigned char*)A.S.tags[i] + p * TB);
        }
      }
      cp_async_commit();
      __syncthreads();
      if (tid < W) {
        int64_t e = s_cur[tid] + 2 * KS;
        s_loaded[tid] = e < s_hi[tid] ? e : s_hi[tid];
      }
    }
    cp_async_wait0();
  }
}

}  // namespace rs
