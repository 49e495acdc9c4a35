// rs_tree.cuh -- node powers, the powersort merge tree, and the executor's task list.
//
// Reference: sorters.py:414-423 (_node_power0), sorters.py:455-516 (the
// power-indexed run stack, whose merge order is the min-Cartesian tree of the
// boundary powers, opttree.py:308-336).
//
// Device formulation (validated in tests/device_model.py):
//  * K_i = floor((s_i + s_{i+1}) * 2^F / (2n)) is leaf i's midpoint in F-bit fixed
//    point (F = 32 for n <= 2^31, else 63); P_j = F + 1 - bitlen(K_{j-1} ^ K_j).
//  * node j (boundary between leaves j-1 and j) covers exactly the leaves whose K
//    shares K_j's top P_j - 1 bits (a compressed binary trie) -> [a_j, b_j].
//  * depth_j = #left ancestors + #right ancestors; both are prefix scans of the
//    maps x -> (x & (bit(P)-1)) | bit(P) over 64-bit power masks.
//  * max_stack_height = max_j (1 + #left ancestors of j)   (sorters.py:500-502).
#pragma once
#include "rs_common.cuh"

namespace rs {

struct MC {
  uint64_t m, c;
};
__device__ __forceinline__ MC mc_identity() { return MC{~0ull, 0ull}; }
__device__ __forceinline__ MC mc_of_power(int p) {
  uint64_t b = 1ull << (p - 1);
  return MC{b - 1, b};
}
// apply `first`, then `then`
__device__ __forceinline__ MC mc_compose(MC first, MC then) {
  return MC{first.m & then.m, (first.c & then.m) | then.c};
}
__device__ __forceinline__ MC shfl_mc_up(MC v, int o) {
  return MC{__shfl_up_sync(0xffffffffu, v.m, o), __shfl_up_sync(0xffffffffu, v.c, o)};
}

// midpoint key of leaf [s0, s1)
__device__ __noinline__ uint64_t mid_key63(uint64_t l2, pos_t n) {  // n > 2^31 only
  unsigned __int128 num = (unsigned __int128)l2 << 63;
  return (uint64_t)(num / (unsigned __int128)(2 * (uint64_t)n));
}
__device__ __forceinline__ uint64_t mid_key(pos_t s0, pos_t s1, pos_t n, int F) {
  uint64_t l2 = (uint64_t)(s0 + s1);
  if (F == 32) return udiv64(l2 << 32, 2 * (uint64_t)n);
  return mid_key63(l2, n);
}

// T1: midpoint keys and boundary powers.
__device__ void d_keys_powers(const pos_t* __restrict__ leaf_start, pos_t n, int F,
                              const DevMetrics* __restrict__ met, uint64_t* __restrict__ K,
                              uint8_t* __restrict__ P) {
  int64_t r = (int64_t)met->n_leaves;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < r; i += (int64_t)gridDim.x * blockDim.x) {
    pos_t s0 = leaf_start[i], s1 = leaf_start[i + 1];
    uint64_t k = mid_key(s0, s1, n, F);
    K[i] = k;
    if (i >= 1) {
      uint64_t kp = mid_key(leaf_start[i - 1], s0, n, F);
      P[i] = (uint8_t)(F + 1 - bitlen64(kp ^ k));
    }
  }
}

// ---- T2: (mask, const) scans for left / right ancestor counts ----
#ifndef RS_SCAN_ITEMS
#define RS_SCAN_ITEMS 2
#endif
constexpr int kScanItems = RS_SCAN_ITEMS;  // max items per thread (unrolled: code size)
constexpr int kScanThreads = 256;
constexpr int kScanChunk = kScanItems * kScanThreads;
// Items per thread adapt to r so that small trees still spread over many blocks.
__device__ __forceinline__ int scan_items(int64_t m) {
  int64_t per = (m + (int64_t)gridDim.x * kScanThreads - 1) / ((int64_t)gridDim.x * kScanThreads);
  return per < 1 ? 1 : (per > kScanItems ? kScanItems : (int)per);
}

// boundary for scan position x in direction dir (m = r-1 boundaries)
__device__ __forceinline__ int64_t scan_j(int64_t x, int64_t m, int dir) { return dir == 0 ? 1 + x : m - x; }

// Ordered block reduction (thread order = sequence order).  Result valid in thread 0.
__device__ inline MC block_reduce_mc(MC v, MC* sm) {
  int lane = threadIdx.x & 31, wid = threadIdx.x >> 5, nw = blockDim.x >> 5;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    MC hi{__shfl_down_sync(0xffffffffu, v.m, o), __shfl_down_sync(0xffffffffu, v.c, o)};
    if (lane + o < 32 && (lane & (2 * o - 1)) == 0) v = mc_compose(v, hi);
  }
  __syncthreads();
  if (lane == 0) sm[wid] = v;
  __syncthreads();
  MC acc = mc_identity();
  if (threadIdx.x == 0)
    for (int i = 0; i < nw; ++i) acc = mc_compose(acc, sm[i]);
  return acc;
}

// Exclusive block scan (thread order = sequence order); returns prefix of threads < t.
__device__ inline MC block_excl_scan_mc(MC v, MC* sm, MC* total) {
  int lane = threadIdx.x & 31, wid = threadIdx.x >> 5, nw = blockDim.x >> 5;
  MC x = v;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    MC y = shfl_mc_up(x, o);
    if (lane >= o) x = mc_compose(y, x);
  }
  __syncthreads();
  if (lane == 31) sm[wid] = x;
  __syncthreads();
  if (threadIdx.x == 0) {
    MC acc = mc_identity();
    for (int i = 0; i < nw; ++i) {
      MC t = sm[i];
      sm[i] = acc;
      acc = mc_compose(acc, t);
    }
    sm[nw] = acc;
  }
  __syncthreads();
  MC excl_w = sm[wid];
  MC ex_lane = shfl_mc_up(x, 1);
  if (lane == 0) ex_lane = mc_identity();
  MC r = mc_compose(excl_w, ex_lane);
  *total = sm[nw];
  __syncthreads();
  return r;
}

__device__ void d_scan_top(const DevMetrics* __restrict__ met, MC* __restrict__ agg, int64_t nchunks_max, int dir);

// Also computes the node powers (dir 0 writes K and P): P_j from leaf starts
// s_{j-1}, s_j, s_{j+1} (sorters.py:414-423).  The block that completes a
// direction's last chunk aggregate scans that direction's aggregates
// (d_scan_top), so the two directions' top scans run concurrently.
// dir_ctr: two zeroed counters.
__device__ void d_scan_reduce(const pos_t* __restrict__ leaf_start, pos_t n, int F, uint64_t* __restrict__ Kk,
                              uint8_t* __restrict__ P, const DevMetrics* __restrict__ met,
                              MC* __restrict__ agg /* [2][nchunks_max] */, int64_t nchunks_max,
                              unsigned int* __restrict__ dir_ctr) {
  __shared__ MC sm[33];
  __shared__ bool s_top;
  int64_t r = (int64_t)met->n_leaves;
  int64_t m = r - 1;
  if (m <= 0) {
    if (m == 0 && blockIdx.x == 0 && threadIdx.x == 0) Kk[0] = mid_key(leaf_start[0], leaf_start[1], n, F);
    return;
  }
  const int items = scan_items(m);
  const int64_t chunk = (int64_t)items * kScanThreads;
  int64_t nch = (m + chunk - 1) / chunk;
  for (int64_t w = blockIdx.x; w < 2 * nch; w += gridDim.x) {
    int dir = int(w / nch);
    int64_t ch = w % nch;
    int64_t x0 = ch * chunk + (int64_t)threadIdx.x * items;
    MC v = mc_identity();
    if (dir == 0) {
      uint64_t kprev = 0;
      if (x0 < m) kprev = mid_key(leaf_start[x0], leaf_start[x0 + 1], n, F);
      if (x0 == 0) Kk[0] = kprev;
      for (int k = 0; k < items; ++k) {
        int64_t x = x0 + k;
        if (x < m) {
          int64_t j = x + 1;
          uint64_t kj = mid_key(leaf_start[j], leaf_start[j + 1], n, F);
          int p = F + 1 - bitlen64(kprev ^ kj);
          Kk[j] = kj;
          P[j] = (uint8_t)p;
          kprev = kj;
          v = mc_compose(v, mc_of_power(p));
        }
      }
    } else {
      for (int k = 0; k < items; ++k) {
        int64_t x = x0 + k;
        if (x < m) {
          int64_t j = scan_j(x, m, 1);
          uint64_t ka = mid_key(leaf_start[j - 1], leaf_start[j], n, F);
          uint64_t kb = mid_key(leaf_start[j], leaf_start[j + 1], n, F);
          v = mc_compose(v, mc_of_power(F + 1 - bitlen64(ka ^ kb)));
        }
      }
    }
    MC t = block_reduce_mc(v, sm);
    if (threadIdx.x == 0) {
      agg[dir * nchunks_max + ch] = t;
      __threadfence();
      s_top = atomicAdd(&dir_ctr[dir], 1u) == (unsigned)(nch - 1);
      if (s_top) __threadfence();
    }
    __syncthreads();
    if (s_top) d_scan_top(met, agg, nchunks_max, dir);
    __syncthreads();
  }
}

// Exclusive scan of chunk aggregates, per direction (one CTA per direction).
__device__ void d_scan_top(const DevMetrics* __restrict__ met, MC* __restrict__ agg,
                           int64_t nchunks_max, int dir) {
  __shared__ MC sm[33];
  int64_t m = (int64_t)met->n_leaves - 1;
  if (m <= 0) return;
  const int64_t chunk = (int64_t)scan_items(m) * kScanThreads;
  int64_t nch = (m + chunk - 1) / chunk;
  MC carry = mc_identity();
  for (int64_t b = 0; b < nch; b += blockDim.x) {
    int64_t i = b + threadIdx.x;
    MC v = i < nch ? agg[dir * nchunks_max + i] : mc_identity();
    MC tot;
    MC ex = block_excl_scan_mc(v, sm, &tot);
    if (i < nch) agg[dir * nchunks_max + i] = mc_compose(carry, ex);
    carry = mc_compose(carry, tot);
  }
}

// Blocks that d_scan_down keeps busy (2 directions x chunks), capped so the
// trie items keep at least half of the grid.
__device__ __forceinline__ int scan_down_blocks(int64_t r) {
  int64_t m = r - 1;
  if (m <= 0) return 0;
  const int64_t chunk = (int64_t)scan_items(m) * kScanThreads;
  int64_t b = 2 * ((m + chunk - 1) / chunk);
  return b > (int64_t)gridDim.x / 2 ? 0 : (int)b;
}

__device__ void d_scan_down(const uint8_t* __restrict__ P,
                                                            DevMetrics* __restrict__ met,
                                                            const MC* __restrict__ agg, int64_t nchunks_max,
                                                            uint8_t* __restrict__ la, uint8_t* __restrict__ ra) {
  __shared__ MC sm[33];
  __shared__ unsigned long long smax[32];
  int64_t m = (int64_t)met->n_leaves - 1;
  if (m <= 0) return;
  const int items = scan_items(m);
  const int64_t chunk = (int64_t)items * kScanThreads;
  int64_t nch = (m + chunk - 1) / chunk;
  unsigned long long best = 0;
  for (int64_t w = blockIdx.x; w < 2 * nch; w += gridDim.x) {
    int dir = int(w / nch);
    int64_t ch = w % nch;
    int64_t x0 = ch * chunk + (int64_t)threadIdx.x * items;
    uint8_t pw[kScanItems];
    MC v = mc_identity();
#pragma unroll
    for (int k = 0; k < kScanItems; ++k) {
      int64_t x = x0 + k;
      pw[k] = (k < items && x < m) ? P[scan_j(x, m, dir)] : 1;
      if (k < items && x < m) v = mc_compose(v, mc_of_power(pw[k]));
    }
    MC tot;
    MC ex = block_excl_scan_mc(v, sm, &tot);
    MC st = mc_compose(agg[dir * nchunks_max + ch], ex);
    uint64_t M = st.c;  // state applied to 0
#pragma unroll
    for (int k = 0; k < kScanItems; ++k) {
      int64_t x = x0 + k;
      if (k < items && x < m) {
        int p = pw[k];
        uint64_t low = (1ull << (p - 1)) - 1;
        int cntv = __popcll(M & low);
        int64_t j = scan_j(x, m, dir);
        if (dir == 0) {
          la[j] = (uint8_t)cntv;
          if ((unsigned long long)(cntv + 1) > best) best = cntv + 1;
        } else {
          ra[j] = (uint8_t)cntv;
        }
        M = (1ull << (p - 1)) | (M & low);
      }
    }
  }
  best = warp_max(best);
  if ((threadIdx.x & 31) == 0) smax[threadIdx.x >> 5] = best;
  __syncthreads();
  if (threadIdx.x == 0) {
    unsigned long long b = 0;
    for (int i = 0; i < (int)(blockDim.x >> 5); ++i) b = smax[i] > b ? smax[i] : b;
    if (b) atomicMax(&met->max_stack_height, b);
  }
}

// ---- T3: trie ranges, parents, children, depths ----
// Unified node ids: internal node j in [1, r-1] -> j; leaf i -> leaf_base + i.
struct TreeArrays {
  const pos_t* leaf_start;
  const uint32_t* leaf_info;
  const uint64_t* K;
  const uint8_t* P;
  const uint8_t* la;
  const uint8_t* ra;
  uint8_t* depth;       // [j] internal node depth
  uint8_t* leaf_depth;  // [i]
  int32_t* node_a;      // [j] first leaf under j
  int32_t* node_b;      // [j] last leaf under j
  int32_t* parent;      // unified id -> unified parent id (-1 root)
  uint32_t* child;      // [2*j + side] unified child ids
  pos_t* node_s;        // [j] span start
  pos_t* node_e;        // [j] span end (exclusive)
  uint32_t leaf_base;
};

// Blocks [b0, gridDim.x) take the items (the first b0 blocks run the ancestor
// scans of the same phase).  Depths are not written here: classification
// derives them from the ancestor counts (ClassifyArgs::la / ra).
__device__ void d_tree(TreeArrays T, int F, const DevMetrics* __restrict__ met, int b0 = 0) {
  int64_t r = (int64_t)met->n_leaves;
  if ((int)blockIdx.x < b0) return;
  const int64_t nb = (int64_t)gridDim.x - b0;
  for (int64_t i = ((int64_t)blockIdx.x - b0) * blockDim.x + threadIdx.x; i < r; i += nb * blockDim.x) {
    // leaf i
    {
      int64_t par = -1;
      int side = 0;
      bool hasL = i >= 1, hasR = i + 1 <= r - 1;
      if (hasL && hasR) {
        if (T.P[i] > T.P[i + 1]) { par = i; side = 1; } else { par = i + 1; side = 0; }
      } else if (hasL) { par = i; side = 1; }
      else if (hasR) { par = i + 1; side = 0; }
      uint32_t lid = T.leaf_base + (uint32_t)i;
      T.parent[lid] = (int32_t)par;
      if (par >= 0) T.child[2 * par + side] = lid;
    }
    if (i >= 1) {
      int64_t j = i;
      int p = T.P[j];
      int sh = F - (p - 1);
      uint64_t kj = T.K[j];
      uint64_t pre = sh >= 64 ? 0 : (kj >> sh);
      uint64_t lo_key = sh >= 64 ? 0 : (pre << sh);
      // left end: smallest a in [0, j-1] with K[a] >= lo_key (gallop from j-1)
      int64_t hi = j - 1, step = 1, x = j - 1 - step;
      while (x >= 0 && T.K[x] >= lo_key) { hi = x; step <<= 1; x = j - 1 - step; }
      int64_t lo = x < 0 ? 0 : x + 1;  // answer in [lo, hi]
      while (lo < hi) {
        int64_t md = lo + (hi - lo) / 2;
        if (T.K[md] >= lo_key) hi = md; else lo = md + 1;
      }
      int64_t a = lo;
      // right end: largest b in [j, r-1] with (K[b] >> sh) == pre
      int64_t b;
      if (sh >= 64) b = r - 1;
      else {
        uint64_t hi_key = (pre + 1) << sh;  // exclusive (wraps to 0 only if pre+1 == 2^(64-sh), F < 64 so never)
        int64_t lo2 = j;
        step = 1;
        x = j + step;
        while (x <= r - 1 && T.K[x] < hi_key) { lo2 = x; step <<= 1; x = j + step; }
        int64_t hi2 = x > r - 1 ? r - 1 : x - 1;  // answer in [lo2, hi2]
        while (lo2 < hi2) {
          int64_t md = lo2 + (hi2 - lo2 + 1) / 2;
          if (T.K[md] < hi_key) lo2 = md; else hi2 = md - 1;
        }
        b = lo2;
      }
      T.node_a[j] = (int32_t)a;
      T.node_b[j] = (int32_t)b;
      T.node_s[j] = T.leaf_start[a];
      T.node_e[j] = T.leaf_start[b + 1];
      int64_t par = -1;
      int side = 0;
      bool hasL = a >= 1, hasR = b + 1 <= r - 1;
      if (hasL && hasR) {
        if (T.P[a] > T.P[b + 1]) { par = a; side = 1; } else { par = b + 1; side = 0; }
      } else if (hasL) { par = a; side = 1; }
      else if (hasR) { par = b + 1; side = 0; }
      T.parent[j] = (int32_t)par;
      if (par >= 0) T.child[2 * par + side] = (uint32_t)j;
    }
  }
}

}  // namespace rs
