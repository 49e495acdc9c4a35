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
#include "rs_exec.cuh"

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

// W = 1: the merge is a copy of the one range (from S.lo / S.hi, or from the
// device split rows).  Coalesced, 16 bytes per thread when both sides allow.
template <typename K, int TB>
__global__ void __launch_bounds__(256) k_kway_copy1(KwayShards S, const int64_t* __restrict__ dsplit, void* out_keys,
                                                    void* out_tags) {
  using T = typename TagT<TB>::type;
  const int64_t lo = dsplit ? dsplit[0] : S.lo[0], hi = dsplit ? dsplit[1] : S.hi[0];
  const int64_t len = hi - lo;
  const int64_t tid = (int64_t)blockIdx.x * blockDim.x + threadIdx.x, nt = (int64_t)gridDim.x * blockDim.x;
  const K* sk = reinterpret_cast<const K*>(S.keys[0]) + lo;
  K* dk = reinterpret_cast<K*>(out_keys);
  constexpr int VK = 16 / sizeof(K);
  if (((reinterpret_cast<uintptr_t>(sk) | reinterpret_cast<uintptr_t>(dk)) & 15) == 0) {
    const int64_t nv = len / VK;
    for (int64_t i = tid; i < nv; i += nt) reinterpret_cast<uint4*>(dk)[i] = reinterpret_cast<const uint4*>(sk)[i];
    for (int64_t i = nv * VK + tid; i < len; i += nt) dk[i] = sk[i];
  } else {
    for (int64_t i = tid; i < len; i += nt) dk[i] = sk[i];
  }
  if (TB) {
    const T* st = reinterpret_cast<const T*>(S.tags[0]) + lo;
    T* dt = reinterpret_cast<T*>(out_tags);
    for (int64_t i = tid; i < len; i += nt) dt[i] = st[i];
  }
}

// Item boundaries: item k starts at the first pivot row whose global rank is
// >= k * group (rank(q) = sum_i bounds[q][i] - bounds[0][i], monotone in q;
// rows 0 .. nrows-1 with nrows = *npiv_items + 1).  item_rows[nitems] = the
// last row; *nitems_out = the item count.
__global__ void __launch_bounds__(256) k_kway_items(const int64_t* __restrict__ bounds, int w,
                                                    const int64_t* __restrict__ npiv_items, int64_t group,
                                                    int64_t kmax, int64_t* __restrict__ item_rows,
                                                    int64_t* __restrict__ nitems_out) {
  const int64_t last = *npiv_items;  // row index of the ends
  int64_t total = 0;
  for (int i = 0; i < w; ++i) total += bounds[last * w + i] - bounds[i];
  const int64_t K = total > 0 ? (total + group - 1) / group : 0;
  if (blockIdx.x == 0 && threadIdx.x == 0) {
    *nitems_out = K;
    item_rows[K] = last;
  }
  for (int64_t k = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; k < K && k < kmax;
       k += (int64_t)gridDim.x * blockDim.x) {
    const int64_t t = k * group;
    int64_t lo = 0, hi = last;  // smallest row with rank >= t
    while (lo < hi) {
      const int64_t mid = (lo + hi) >> 1;
      int64_t r = 0;
      for (int i = 0; i < w; ++i) r += bounds[mid * w + i] - bounds[i];
      if (r >= t) hi = mid;
      else lo = mid + 1;
    }
    item_rows[k] = lo;
  }
}

// k_kway_merge: persistent CTAs claim work items (the intervals between
// consecutive pivots in global order: at most `spacing` elements of each
// shard, so at most ITEM in all).  An item's W windows arrive in shared memory
// by 1D bulk copies (TMA, local or peer memory alike) while the previous item
// is merged: a pairwise merge tree inside shared memory, every level's
// outputs split evenly over the CTA's threads by merge-path searches (ties to
// the lower shard at every level => the (key, shard, position) order), keys
// and tags moved together; the last level lands in shared memory and the CTA
// writes it out with coalesced stores.
template <typename K, int TB>
struct KwayCfg {
  static constexpr int THREADS = 256;
  static constexpr int kb = sizeof(K);
  static constexpr int eb = kb + TB;
  static constexpr int ITEM = eb <= 4 ? 8192 : (eb <= 8 ? 4096 : (eb <= 12 ? 2688 : 2048));  // elements per item
  static constexpr int PAD = 16 * kKwayMaxW;  // per-window 16-byte phase slack (elements)
  static constexpr int CAP = ITEM + PAD;
  static constexpr size_t KBUF = ((size_t)CAP * kb + 127) / 128 * 128;
  static constexpr size_t TBUF = TB ? ((size_t)CAP * (TB ? TB : 1) + 127) / 128 * 128 : 0;
  static constexpr size_t BUF = KBUF + TBUF;
  static constexpr size_t SMEM = 3 * BUF + 256;  // two load buffers + one merge buffer
  // Items are cut where the pivots' global ranks cross multiples of GROUP, and
  // consecutive pivots are at most W * spacing apart, so an item holds fewer
  // than GROUP + W * spacing <= ITEM elements (about GROUP on average).
  static constexpr int GROUP = ITEM / 2;
  static int64_t spacing(int w) { return GROUP / (w > 0 ? w : 1); }
};

__device__ __forceinline__ void cp_async16(void* s, const void* g) {
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(smem_addr(s)), "l"(g) : "memory");
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;" ::: "memory"); }
__device__ __forceinline__ void cp_async_wait1() { asm volatile("cp.async.wait_group 1;" ::: "memory"); }
__device__ __forceinline__ void cp_async_wait0() { asm volatile("cp.async.wait_group 0;" ::: "memory"); }

struct KwayMergeArgs {
  KwayShards S;
  const int64_t* bounds;  // (nitems + 1) x W split vectors; row 0 = the ranges' starts
  const int64_t* nitems;     // written by k_kway_items
  const int64_t* item_rows;  // item k = pivot rows [item_rows[k], item_rows[k + 1])
  void* out_keys;
  void* out_tags;
  unsigned long long* claim;  // zeroed before launch
};

template <typename K, int TB>
__global__ void __launch_bounds__(256, 2) k_kway_merge(KwayMergeArgs A) {
  using C = KwayCfg<K, TB>;
  using T = typename TagT<TB>::type;
  constexpr bool HT = TB != 0;
  constexpr int NT = C::THREADS;
  constexpr int kHalf = kKwayMaxW / 2 + 1;
  extern __shared__ __align__(128) unsigned char smem_kw[];
  __shared__ int64_t s_item[2], s_out[2];
  __shared__ int s_kseg[2][kKwayMaxW], s_tseg[2][kKwayMaxW], s_len[2][kKwayMaxW];  // per load buffer
  const int W = A.S.w;
  const int tid = threadIdx.x;
  auto kbuf = [&](int b) { return reinterpret_cast<K*>(smem_kw + (size_t)b * C::BUF); };
  auto tbuf = [&](int b) { return reinterpret_cast<T*>(smem_kw + (size_t)b * C::BUF + C::KBUF); };
  const int64_t nitems = *A.nitems;
  // Collective: claim an item and stream its windows into load buffer b with
  // 16-byte cp.async copies spread over all threads (one commit group per call,
  // empty when no item is left).  Windows are copied as their 16-byte covers;
  // s_kseg / s_tseg = where each window's first element lands.  (Whole-window
  // 1D bulk copies cost ~1 us each for the few-hundred-byte windows of an
  // 8-way item; the W bounds are read by W threads at once.)
  __shared__ int64_t s_lo[kKwayMaxW], s_base[kKwayMaxW];
  __shared__ uint32_t s_kc[kKwayMaxW + 1], s_tc[kKwayMaxW + 1];  // chunk prefix (16-byte units)
  __shared__ uintptr_t s_ka[kKwayMaxW], s_ta[kKwayMaxW];            // aligned source addresses
  auto fetch = [&](int b) {
    if (tid == 0) s_item[b] = (int64_t)atomicAdd(A.claim, 1ull);
    __syncthreads();
    const int64_t item = s_item[b];
    if (item < nitems) {
      if (tid < W) {
        const int64_t r0 = A.item_rows[item], r1 = A.item_rows[item + 1];
        const int64_t lo = A.bounds[r0 * W + tid], hi = A.bounds[r1 * W + tid], base = A.bounds[tid];
        s_lo[tid] = lo;
        s_base[tid] = base;
        s_len[b][tid] = (int)(hi - lo);
        uint32_t kc = 0, tc = 0;
        if (hi > lo) {
          uintptr_t a0 = reinterpret_cast<uintptr_t>(reinterpret_cast<const K*>(A.S.keys[tid]) + lo);
          uintptr_t a1 = reinterpret_cast<uintptr_t>(reinterpret_cast<const K*>(A.S.keys[tid]) + hi);
          s_ka[tid] = a0 & ~(uintptr_t)15;
          kc = (uint32_t)((((a1 + 15) & ~(uintptr_t)15) - s_ka[tid]) / 16);
          s_kseg[b][tid] = (int)((a0 & 15) / sizeof(K));  // + the window's base, below
          if (HT) {
            uintptr_t t0 = reinterpret_cast<uintptr_t>(reinterpret_cast<const T*>(A.S.tags[tid]) + lo);
            uintptr_t t1 = reinterpret_cast<uintptr_t>(reinterpret_cast<const T*>(A.S.tags[tid]) + hi);
            s_ta[tid] = t0 & ~(uintptr_t)15;
            tc = (uint32_t)((((t1 + 15) & ~(uintptr_t)15) - s_ta[tid]) / 16);
            s_tseg[b][tid] = (int)((t0 & 15) / (HT ? TB : 1));
          }
        } else {
          s_kseg[b][tid] = 0;
          s_tseg[b][tid] = 0;
        }
        s_kc[tid + 1] = kc;
        s_tc[tid + 1] = tc;
      }
      __syncthreads();
      if (tid == 0) {
        int64_t o = 0;
        s_kc[0] = 0;
        s_tc[0] = 0;
        for (int i = 0; i < W; ++i) {
          o += s_lo[i] - s_base[i];
          s_kseg[b][i] += (int)(s_kc[i] * 16 / sizeof(K));
          if (HT) s_tseg[b][i] += (int)(s_tc[i] * 16 / (HT ? TB : 1));
          s_kc[i + 1] += s_kc[i];
          s_tc[i + 1] += s_tc[i];
        }
        s_out[b] = o;
      }
      __syncthreads();
      unsigned char* kd = reinterpret_cast<unsigned char*>(kbuf(b));
      for (uint32_t c = tid; c < s_kc[W]; c += NT) {
        int i = 0;
        while (s_kc[i + 1] <= c) ++i;
        const uint32_t r = c - s_kc[i];
        cp_async16(kd + (size_t)c * 16, reinterpret_cast<const void*>(s_ka[i] + (uintptr_t)r * 16));
      }
      if (HT) {
        unsigned char* td = reinterpret_cast<unsigned char*>(tbuf(b));
        for (uint32_t c = tid; c < s_tc[W]; c += NT) {
          int i = 0;
          while (s_tc[i + 1] <= c) ++i;
          const uint32_t r = c - s_tc[i];
          cp_async16(td + (size_t)c * 16, reinterpret_cast<const void*>(s_ta[i] + (uintptr_t)r * 16));
        }
      }
    }
    cp_async_commit();
  };
  fetch(0);
  int cur = 0;
  for (;;) {
    __syncthreads();  // s_item / segment tables visible; the last item's buffers are read
    if (s_item[cur] >= nitems) break;
    fetch(cur ^ 1);  // the next item's windows stream in while this one merges
    cp_async_wait1();  // this thread's copies of the current item have landed
    __syncthreads();   // ... and everyone's
    int N = 0;
    for (int i = 0; i < W; ++i) N += s_len[cur][i];
    // segments of the current level: key / tag starts and lengths (registers, uniform)
    int kst[kKwayMaxW], tst[kKwayMaxW], len[kKwayMaxW];
    for (int i = 0; i < W; ++i) {
      kst[i] = s_kseg[cur][i];
      tst[i] = s_tseg[cur][i];
      len[i] = s_len[cur][i];
    }
    int nseg = W, src = cur, dst = 2;
    while (nseg > 1) {
      const int npairs = (nseg + 1) / 2;
      int ost[kHalf + 1];
      ost[0] = 0;
      for (int p = 0; p < npairs; ++p) ost[p + 1] = ost[p] + len[2 * p] + (2 * p + 1 < nseg ? len[2 * p + 1] : 0);
      const K* sk = kbuf(src);
      const T* stg = HT ? tbuf(src) : nullptr;
      K* dk = kbuf(dst);
      T* dtg = HT ? tbuf(dst) : nullptr;
      const int per = (N + NT - 1) / NT;
      const int d0 = tid * per < N ? tid * per : N, d1 = d0 + per < N ? d0 + per : N;
      for (int p = 0; p < npairs; ++p) {
        const int s0 = d0 > ost[p] ? d0 : ost[p], s1 = d1 < ost[p + 1] ? d1 : ost[p + 1];
        if (s0 >= s1) continue;
        const int ia_ = 2 * p, ib_ = 2 * p + 1;
        const K* Ak = sk + kst[ia_];
        const int la = len[ia_];
        const K* Bk = ib_ < nseg ? sk + kst[ib_] : Ak;
        const int lb = ib_ < nseg ? len[ib_] : 0;
        const T* At = HT ? stg + tst[ia_] : nullptr;
        const T* Bt = HT ? (ib_ < nseg ? stg + tst[ib_] : At) : nullptr;
        const int x0 = s0 - ost[p];
        int lo = x0 - lb > 0 ? x0 - lb : 0, hi = x0 < la ? x0 : la;  // #A among the first x0 outputs
        while (lo < hi) {
          int mid = (lo + hi) >> 1;
          if (Ak[mid] <= Bk[x0 - 1 - mid]) lo = mid + 1;
          else hi = mid;
        }
        int ia = lo, ib = x0 - lo;
        for (int d = s0; d < s1; ++d) {
          const bool ta = ib >= lb || (ia < la && Ak[ia] <= Bk[ib]);  // ties: the lower shard
          if (ta) {
            dk[d] = Ak[ia];
            if (HT) dtg[d] = At[ia];
            ++ia;
          } else {
            dk[d] = Bk[ib];
            if (HT) dtg[d] = Bt[ib];
            ++ib;
          }
        }
      }
      __syncthreads();  // the level is complete
      for (int p = 0; p < npairs; ++p) {
        kst[p] = ost[p];
        tst[p] = ost[p];
        len[p] = ost[p + 1] - ost[p];
      }
      nseg = npairs;
      const int t = src;  // ping-pong: the merge buffer and this item's own load buffer
      src = dst;
      dst = t;
    }
    // coalesced write-out of the single remaining segment
    {
      const K* fk = kbuf(src) + kst[0];
      const T* ft = HT ? tbuf(src) + tst[0] : nullptr;
      const int64_t ob = s_out[cur];
      K* ok = reinterpret_cast<K*>(A.out_keys) + ob;
      T* ot = HT ? reinterpret_cast<T*>(A.out_tags) + ob : nullptr;
      for (int d = tid; d < N; d += NT) {
        ok[d] = fk[d];
        if (HT) ot[d] = ft[d];
      }
    }
    cur ^= 1;
  }
  cp_async_wait0();
}

}  // namespace rs
