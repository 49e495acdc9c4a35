// rs_small.cuh -- the tree half of the prep (node powers, ancestor scans, trie
// ranges, classification, ordered task list) for trees of at most kSmallR
// leaves (n < 2^31): the tree in ONE CTA working out of shared memory, the
// task records written by the whole grid.
//
// Same outputs as k_prep's phases 5-9 (rs_tree.cuh, rs_exec.cuh: d_scan_reduce,
// d_scan_down, d_tree, d_classify, d_task_offsets/d_order_scan, d_task_fill),
// with the merge tasks ordered by estimated ready time instead of (depth desc,
// position) -- any topological order gives the same output.  With few
// leaves those phases are pure latency: each is a chain of L2 round trips plus
// a grid barrier over hundreds of mostly idle CTAs.  Here the chains run at
// shared-memory latency behind __syncthreads (block 0, small_tree), which
// leaves a compact job list -- {first task slot, id, task count | kind} per
// phase-A item and per merge node, merge jobs with their node's 48-byte
// descriptor -- and after one grid barrier every thread of the grid writes
// task records (small_fill: one task per thread, its job found by a binary
// search over the job slots staged in shared memory).  A single CTA writing
// the records (16K merge tasks on config 2) was the old bottleneck.
#pragma once
#include "rs_exec.cuh"
#include "rs_tree.cuh"

namespace rs {

// Per-item loops stay rolled (per-item state in local memory): the block runs
// this code once per sort from a cold instruction cache, so code bytes cost
// more than the extra local-memory traffic.
#ifndef RS_SMALL_UNROLL_N
#define RS_SMALL_UNROLL_N 1
#endif
constexpr int kSmallUnroll = RS_SMALL_UNROLL_N;
#ifndef RS_SMALL_R
#define RS_SMALL_R 2048
#endif
constexpr int kSmallR = RS_SMALL_R;  // above this the grid-wide phases of k_prep are faster
constexpr int kJobCap = 2 * kSmallR + 2;  // <= one job per leaf and one per boundary

// 32-bit shared-memory arrays (positions and midpoint keys fit: n < 2^31, F = 32)
__host__ __device__ constexpr size_t small_arrays_bytes() {
  return (size_t)(kSmallR + 1) * 4      // Ls: leaf starts
         + (size_t)kSmallR * 4 * 4      // Ks: midpoint keys; spans | no-fuse bit 31; phase-A / merge task counts
         + (size_t)2 * kSmallR * 2      // par: parents of leaves [0, r) and nodes [r, 2r)
         + (size_t)(kSmallR + 1) * 5    // Ps, las, ras, dep, ldep
         + (size_t)kSmallR * 2;         // leaf / node classes
}
__host__ __device__ constexpr size_t small_smem_bytes() {
  return small_arrays_bytes() > (size_t)kJobCap * 4 ? small_arrays_bytes() : (size_t)kJobCap * 4;
}
// Global job list (workspace): slots, ids, counts | kind << 30, and the merge
// descriptors indexed by node id (a merge job's id).
__host__ __device__ constexpr size_t small_jobs_bytes() { return (size_t)kJobCap * (12 + sizeof(MDesc)) + 64; }
struct SmallJobs {
  uint32_t* slot;
  uint32_t* id;
  uint32_t* cnt;
  MDesc* md;
  __host__ __device__ static SmallJobs at(unsigned char* base) {
    SmallJobs J;
    J.md = reinterpret_cast<MDesc*>(base);  // 16-byte aligned first
    J.slot = reinterpret_cast<uint32_t*>(base + (size_t)kJobCap * sizeof(MDesc));
    J.id = J.slot + kJobCap;
    J.cnt = J.id + kJobCap;
    return J;
  }
};

__device__ __forceinline__ unsigned long long block_excl_scan_u64(unsigned long long v, unsigned long long* smem,
                                                                  unsigned long long* total) {
  int lane = threadIdx.x & 31, wid = threadIdx.x >> 5, nw = blockDim.x >> 5;
  unsigned long long x = v;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    unsigned long long y = __shfl_up_sync(0xffffffffu, x, o);
    if (lane >= o) x += y;
  }
  __syncthreads();
  if (lane == 31) smem[wid] = x;
  __syncthreads();
  if (wid == 0) {
    unsigned long long s = lane < nw ? smem[lane] : 0, t = s;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      unsigned long long y = __shfl_up_sync(0xffffffffu, t, o);
      if (lane >= o) t += y;
    }
    if (lane < nw) smem[lane] = t - s;
    if (lane == 31) smem[32] = t;
  }
  __syncthreads();
  unsigned long long r = smem[wid] + x - v;
  *total = smem[32];
  __syncthreads();
  return r;
}

// Run by one CTA of NT threads (block 0 of k_prep after its leaf phase);
// smem_small: small_smem_bytes() of dynamic shared memory.  Requires n < 2^31.
template <int NT>
__device__ void small_tree(const TreeArrays& T, ClassifyArgs A, unsigned char* smem_small, SmallJobs J) {
  constexpr int kSmallPer = (kSmallR + NT - 1) / NT;  // items per thread
  constexpr int F = 32;
  DevMetrics* met = A.met;
  const int64_t r = (int64_t)met->n_leaves;
  if (r > kSmallR || r < 1) return;
  // Fuse policy.  Short leaves on average: every subtree that fits (as in the
  // grid path).  Long leaves: the grid path fuses nothing (pairs of ~1K-element
  // runs merge faster in the executor); a small tree is latency-bound instead
  // -- every executor level under a big node costs a full tile latency (~10 us)
  // on its critical path -- so subtrees of >= 3 leaves that fit are still fused
  // (config 3: the chain of nine small levels below a 4M-element merge loses three).
  int min_nodes = 0;  // 2: see the demotion pass after the trie phase
  if (A.n >= (pos_t)A.fuse_avg * r) {
    if (A.small_fuse) min_nodes = 2;
    else A.fcap = 0;
  }
  RS_TS(met, 5);
  uint32_t* Ls = reinterpret_cast<uint32_t*>(smem_small);
  uint32_t* Ks = Ls + kSmallR + 1;
  // per-item state lives in shared memory, indexed by item: local arrays
  // indexed by a rolled loop spill to local memory, whose loads missed L1
  // (measured: 14.6 us for config 3's 50-leaf per-depth loop)
  uint32_t* spans = Ks + kSmallR;     // node span | kNoFuse (bit 31)
  uint32_t* s_aof = spans + kSmallR;  // phase-A tasks of item i (its leaf, its fused node)
  uint32_t* s_tk = s_aof + kSmallR;   // merge tasks of node i (0 unless big)
  int16_t* par = reinterpret_cast<int16_t*>(s_tk + kSmallR);
  uint8_t* Ps = reinterpret_cast<uint8_t*>(par + 2 * kSmallR);
  uint8_t* las = Ps + kSmallR + 1;
  uint8_t* ras = las + kSmallR + 1;
  uint8_t* dep = ras + kSmallR + 1;
  uint8_t* ldep = dep + kSmallR + 1;
  uint8_t* s_lc = ldep + kSmallR + 1;  // leaf classes
  uint8_t* s_nc = s_lc + kSmallR;       // node classes
  __shared__ MC smc[33];
  __shared__ unsigned long long sred[33];
  __shared__ unsigned s_maxd;

  const int tid = threadIdx.x, nt = blockDim.x;
  const pos_t n = A.n;
  const int64_t m = r - 1;  // boundaries 1..m
  uint64_t* Kg = const_cast<uint64_t*>(T.K);
  uint8_t* Pg = const_cast<uint8_t*>(T.P);
  uint8_t* lag = const_cast<uint8_t*>(T.la);
  uint8_t* rag = const_cast<uint8_t*>(T.ra);

  for (int64_t i = tid; i <= r; i += nt) Ls[i] = (uint32_t)T.leaf_start[i];
  if (tid == 0) s_maxd = 0;
  __syncthreads();
  // ---- keys and powers (sorters.py:414-423 via the midpoint-key closed form)
  for (int64_t i = tid; i < r; i += nt) {
    uint64_t k = mid_key(Ls[i], Ls[i + 1], n, F);
    Ks[i] = (uint32_t)k;
    Kg[i] = k;
  }
  __syncthreads();
  for (int64_t j = 1 + tid; j < r; j += nt) {
    int p = F + 1 - bitlen64((uint64_t)(Ks[j - 1] ^ Ks[j]));
    Ps[j] = (uint8_t)p;
    Pg[j] = (uint8_t)p;
  }
  __syncthreads();
  // ---- left / right ancestor counts: (mask, const) scans, contiguous items per thread
  unsigned long long best = 0;
  if (m > 0) {
    const int64_t per = (m + nt - 1) / nt;
    const int64_t x0 = (int64_t)tid * per;
    for (int dir = 0; dir < 2; ++dir) {
      MC v = mc_identity();
      for (int64_t k = 0; k < per; ++k) {
        int64_t x = x0 + k;
        if (x < m) v = mc_compose(v, mc_of_power(Ps[scan_j(x, m, dir)]));
      }
      MC tot;
      MC ex = block_excl_scan_mc(v, smc, &tot);
      uint64_t M = ex.c;
      for (int64_t k = 0; k < per; ++k) {
        int64_t x = x0 + k;
        if (x >= m) break;
        int64_t j = scan_j(x, m, dir);
        int p = Ps[j];
        uint64_t low = (1ull << (p - 1)) - 1;
        int cnt = __popcll(M & low);
        if (dir == 0) {
          las[j] = (uint8_t)cnt;
          lag[j] = (uint8_t)cnt;
          if ((unsigned long long)(cnt + 1) > best) best = cnt + 1;
        } else {
          ras[j] = (uint8_t)cnt;
          rag[j] = (uint8_t)cnt;
        }
        M = (1ull << (p - 1)) | (M & low);
      }
    }
  }
  best = warp_max(best);
  if ((tid & 31) == 0) sred[tid >> 5] = best;
  __syncthreads();
  if (tid == 0 && m > 0) {
    unsigned long long b = 0;
    for (int i = 0; i < (nt >> 5); ++i) b = sred[i] > b ? sred[i] : b;
    met->max_stack_height = b;  // sorters.py:500-502
  }
  RS_TS(met, 6);
  // ---- trie ranges, parents, children, spans (d_tree)
  if (tid == 0) spans[0] = 0;
#pragma unroll kSmallUnroll
  for (int q = 0; q < kSmallPer; ++q) {
    int64_t i = tid + (int64_t)q * nt;
    if (i >= r) continue;
    {
      int64_t p = -1;
      int side = 0;
      bool hasL = i >= 1, hasR = i + 1 <= r - 1;
      if (hasL && hasR) {
        if (Ps[i] > Ps[i + 1]) { p = i; side = 1; } else { p = i + 1; side = 0; }
      } else if (hasL) { p = i; side = 1; }
      else if (hasR) { p = i + 1; side = 0; }
      uint32_t lid = T.leaf_base + (uint32_t)i;
      T.parent[lid] = (int32_t)p;
      par[i] = (int16_t)p;
      uint8_t ld = 0;
      if (p >= 0) {
        T.child[2 * p + side] = lid;
        ld = (uint8_t)(las[p] + ras[p] + 1);
      }
      T.leaf_depth[i] = ld;
      ldep[i] = ld;
    }
    if (i >= 1) {
      int64_t j = i;
      int p = Ps[j];
      int sh = F - (p - 1);
      uint64_t kj = Ks[j];
      uint64_t pre = sh >= 64 ? 0 : (kj >> sh);
      uint64_t lo_key = sh >= 64 ? 0 : (pre << sh);
      int64_t hi = j - 1, step = 1, x = j - 1 - step;
      while (x >= 0 && (uint64_t)Ks[x] >= lo_key) { hi = x; step <<= 1; x = j - 1 - step; }
      int64_t lo = x < 0 ? 0 : x + 1;
      while (lo < hi) {
        int64_t md = lo + (hi - lo) / 2;
        if ((uint64_t)Ks[md] >= lo_key) hi = md; else lo = md + 1;
      }
      int64_t a = lo, b;
      if (sh >= 64) b = r - 1;
      else {
        uint64_t hi_key = (pre + 1) << sh;
        int64_t lo2 = j;
        step = 1;
        x = j + step;
        while (x <= r - 1 && (uint64_t)Ks[x] < hi_key) { lo2 = x; step <<= 1; x = j + step; }
        int64_t hi2 = x > r - 1 ? r - 1 : x - 1;
        while (lo2 < hi2) {
          int64_t md = lo2 + (hi2 - lo2 + 1) / 2;
          if ((uint64_t)Ks[md] < hi_key) lo2 = md; else hi2 = md - 1;
        }
        b = lo2;
      }
      T.node_a[j] = (int32_t)a;
      T.node_b[j] = (int32_t)b;
      pos_t s0 = Ls[a], e0 = Ls[b + 1];
      T.node_s[j] = s0;
      T.node_e[j] = e0;
      // bit 31: not fusable (fusable_span: node table, average leaf length)
      spans[j] = (uint32_t)(e0 - s0) | (fusable_span(A, e0 - s0, b - a) ? 0u : 0x80000000u);
      uint8_t dd = (uint8_t)(las[j] + ras[j]);
      T.depth[j] = dd;
      dep[j] = dd;
      int64_t pp = -1;
      int side = 0;
      bool hasL = a >= 1, hasR = b + 1 <= r - 1;
      if (hasL && hasR) {
        if (Ps[a] > Ps[b + 1]) { pp = a; side = 1; } else { pp = b + 1; side = 0; }
      } else if (hasL) { pp = a; side = 1; }
      else if (hasR) { pp = b + 1; side = 0; }
      T.parent[j] = (int32_t)pp;
      par[r + j] = (int16_t)pp;
      if (pp >= 0) T.child[2 * pp + side] = (uint32_t)j;
    }
  }
  __syncthreads();
  // long leaves: a fusable subtree of only two leaves whose parent is not
  // fusable stays with the executor (marked not fusable; nothing reads the
  // entries written here in this pass: such a node has no node child, and its
  // parent, having one, is not rewritten)
  if (min_nodes) {
    for (int64_t j = 1 + tid; j < r; j += nt) {
      const int pp = par[r + j];
      if ((pos_t)spans[j] <= (pos_t)A.fcap && par[j - 1] == (int16_t)j && par[j] == (int16_t)j &&
          !(pp >= 0 && (pos_t)spans[pp] <= (pos_t)A.fcap))
        spans[j] |= 0x80000000u;
    }
    __syncthreads();
  }
  RS_TS(met, 7);
  // ---- classification (d_classify), contiguous items per thread
  const int64_t per = (r + nt - 1) / nt;
  const int64_t i0 = (int64_t)tid * per;
  constexpr uint32_t kNoFuse = 0x80000000u;
  auto fusable_s = [&](int64_t j) { return (pos_t)spans[j] <= (pos_t)A.fcap; };  // kNoFuse set -> > fcap
  auto parent_small_s = [&](int32_t p) { return p >= 0 && fusable_s(p); };
  unsigned long long comps = 0, mcost = 0, mbig = 0;
  unsigned maxd = 0;
  for (int q = 0; q < per; ++q) {
    int64_t i = i0 + q;
    if (i >= r) break;
    uint32_t tk_i = 0, a_i = 0;
    uint8_t nc_i = 0;
    pos_t s0 = Ls[i], len = (pos_t)Ls[i + 1] - s0;
    uint32_t info = A.leaf_info[i];
    uint32_t nl = info & 0x7fffffffu;
    if (!A.peek && s0 < n - 1) {
      pos_t L = (nl >= (uint32_t)A.w) ? len : (pos_t)nl;
      pos_t ne = s0 + L - 1;
      comps += (unsigned long long)((ne < n - 1) ? L : L - 1);
    }
    // leaf (classify_leaf)
    uint32_t lid = A.leaf_base + (uint32_t)i;
    int c = 0;
    int64_t tl = 0;
    if (!(len <= A.fcap && parent_small_s(par[i]))) {
      if (nl < (uint32_t)A.w && (pos_t)nl < len) c = 1;
      else {
        int mode = leaf_mode((info >> 31) != 0, ldep[i]);
        tl = leaf_tiles(len, mode, A.tile);
        c = tl > 0 ? 2 : 0;
      }
    }
    A.need[lid] = c == 1 ? 1u : (uint32_t)tl;
    A.cls[lid] = (uint8_t)c;
    s_lc[i] = (uint8_t)c;
    a_i = c == 1 ? 1u : (uint32_t)tl;
    if (i >= 1) {
      bool fz = fusable_s(i);
      pos_t span = (pos_t)(spans[i] & ~kNoFuse);
      mcost += span;
      if (!A.classic) comps += span;  // runcore.py:299-301
      int cn;
      if (fz) cn = parent_small_s(par[r + i]) ? 0 : 1;
      else cn = 2;
      A.cls[i] = (uint8_t)cn;
      nc_i = (uint8_t)cn;
      if (cn == 1) {
        A.need[i] = 1;
        a_i += 1;
      } else if (cn == 2) {
        int64_t tn = ceil_div64(span, A.mtile);
        A.need[i] = (uint32_t)tn;
        tk_i = (uint32_t)ceil_div64(tn, A.msuper);
        mbig += span;
        maxd = dep[i] > maxd ? dep[i] : maxd;
      } else A.need[i] = 0;
    }
    s_nc[i] = nc_i;
    s_tk[i] = tk_i;
    s_aof[i] = a_i;
  }
  unsigned long long sc = block_sum(comps, sred);
  if (tid == 0) met->comparisons += sc;
  sc = block_sum(mcost, sred);
  if (tid == 0) met->merge_cost += sc;
  sc = block_sum(mbig, sred);
  if (tid == 0) met->merge_cost_exec += sc;
  maxd = warp_max(maxd);
  if ((tid & 31) == 0 && maxd) atomicMax(&s_maxd, maxd);
  RS_TS(met, 8);
  __syncthreads();  // A.need / A.cls / T.child of every item written (descriptors read them)
  // ---- job list: phase-A jobs -- the fused ones first (a fused subtree runs for
  // tens of thousands of cycles, a leaf tile for ~6K: claimed last it would end
  // the phase), then the leaf tiles, each group by position -- then merge jobs.
  // Each job's first task slot and its own index come from one packed scan
  // (fused jobs << 45 | leaf jobs << 32 | leaf tasks; a fused job is one task);
  // merge jobs carry their node's descriptor.
  unsigned long long vA = 0;
  for (int q = 0; q < per; ++q) {
    const int64_t i = i0 + q;
    if (i >= r) break;
    const uint32_t tl = s_aof[i] - (s_nc[i] == 1 ? 1u : 0u);  // the leaf's own tasks
    const unsigned long long jf = (s_lc[i] == 1 ? 1u : 0u) + (s_nc[i] == 1 ? 1u : 0u);
    const unsigned long long jl = (s_lc[i] == 2 && tl > 0) ? 1u : 0u;
    vA += (jf << 45) | (jl << 32) | (jl ? tl : 0u);
  }
  unsigned long long totv;
  RS_TSD(met, 0);
  unsigned long long ex = block_excl_scan_u64(vA, sred, &totv);
  RS_TSD(met, 1);
  const uint32_t totF = (uint32_t)(totv >> 45), totJL = (uint32_t)(totv >> 32) & 0x1fffu;
  const uint32_t totA = totF + (uint32_t)totv;
  {
    uint32_t jf = (uint32_t)(ex >> 45);                       // fused job index = its slot
    uint32_t jl = totF + ((uint32_t)(ex >> 32) & 0x1fffu);    // leaf job index
    uint32_t slot = totF + (uint32_t)ex;                      // leaf job's first slot
    for (int q = 0; q < per; ++q) {
      int64_t i = i0 + q;
      if (i >= r) break;
      uint32_t lid = A.leaf_base + (uint32_t)i;
      const uint8_t lc = s_lc[i], nc = s_nc[i];
      uint32_t tl = s_aof[i] - (nc == 1 ? 1u : 0u);
      if (lc == 1) {
        J.slot[jf] = jf;
        J.id[jf] = lid;
        J.cnt[jf] = 1u | ((uint32_t)kTaskFuse << 30);
        ++jf;
      } else if (lc == 2 && tl > 0) {
        J.slot[jl] = slot;
        J.id[jl] = lid;
        J.cnt[jl] = tl | ((uint32_t)kTaskLeaf << 30);
        ++jl;
        slot += tl;
      }
      if (nc == 1) {
        J.slot[jf] = jf;
        J.id[jf] = (uint32_t)i;
        J.cnt[jf] = 1u | ((uint32_t)kTaskFuse << 30);
        ++jf;
      }
    }
  }
  // merge descriptors, node-indexed, all at once: one strided pass of
  // independent round trips instead of one dependent chain per depth
  for (int64_t i = 1 + tid; i < r; i += nt)
    if (A.cls[i] == 2) J.md[i] = load_mdesc(A, (uint32_t)i);
  RS_TSD(met, 2);
  uint32_t jbase = totF + totJL;
  uint64_t base = totA;
  const int dmax = (int)s_maxd;
  RS_TSD(met, 3);
  // ---- merge jobs in the order of their estimated ready times.  The executor
  // claims tasks strictly in list order and a producer that claimed a task
  // waits for the node's children, so a (depth desc, position) list lets one
  // node with a deep subtree below it hold every producer while its ready
  // siblings' tiles sit behind it (config 3: three 4M-element depth-2 nodes
  // queued behind the fourth, which waits for a chain of nine small levels).
  // ready(node) = max over its executor children of ready + c0 + c1 * tasks
  // (c0: one tile's latency through the executor, c1: a tile's service time
  // over the whole grid), 0 below phase-A children.  ready(parent) > ready(child),
  // so the list stays a topological order (every wait is on an earlier task).
  uint32_t* ready = spans;  // spans are dead after classification
  unsigned long long* skey = reinterpret_cast<unsigned long long*>(smem_small);  // over Ls + Ks (dead)
  for (int64_t i = tid; i < r; i += nt) ready[i] = 0;
  __syncthreads();
  for (int d = dmax; d >= 1; --d) {
    for (int q = 0; q < per; ++q) {
      const int64_t i = i0 + q;
      if (i >= r) break;
      if (s_nc[i] == 2 && dep[i] == d) {
        const int p = par[r + i];
        if (p >= 0) atomicMax(&ready[p], ready[i] + (uint32_t)A.est_c0 + (uint32_t)A.est_c1 * s_tk[i]);
      }
    }
    __syncthreads();
  }
  // compact the big nodes' sort keys: ready << 32 | min(tasks, 2^20 - 1) << 12 | node
  unsigned long long vb = 0;
  for (int q = 0; q < per; ++q) {
    const int64_t i = i0 + q;
    if (i >= r) break;
    if (s_nc[i] == 2) vb += 1;
  }
  unsigned long long totb;
  const unsigned long long exb = block_excl_scan_u64(vb, sred, &totb);
  const int m2 = (int)totb;
  int P2 = 1;
  while (P2 < m2) P2 <<= 1;
  {
    int k = (int)exb;
    for (int q = 0; q < per; ++q) {
      const int64_t i = i0 + q;
      if (i >= r) break;
      if (s_nc[i] == 2) {
        const uint32_t tk = s_tk[i] < 0xfffffu ? s_tk[i] : 0xfffffu;
        skey[k++] = ((unsigned long long)ready[i] << 32) | ((unsigned long long)tk << 12) | (unsigned long long)i;
      }
    }
    for (int x = m2 + tid; x < P2; x += nt) skey[x] = ~0ull;
  }
  __syncthreads();
  // bitonic sort of P2 <= 2048 keys (all distinct: the node id is in the key)
  for (int k = 2; k <= P2; k <<= 1) {
    for (int j = k >> 1; j > 0; j >>= 1) {
      for (int t = tid; t < (P2 >> 1); t += nt) {
        const int lo = ((t & ~(j - 1)) << 1) | (t & (j - 1));
        const int hi = lo | j;
        const unsigned long long a = skey[lo], b = skey[hi];
        const bool up = (lo & k) == 0;
        if ((a > b) == up) { skey[lo] = b; skey[hi] = a; }
      }
      __syncthreads();
    }
  }
  // first task slot of every job: scan of the task counts in sorted order
  {
    const int per2 = (m2 + nt - 1) / nt;
    const int x0 = tid * per2;
    unsigned long long v = 0;
    for (int q = 0; q < per2; ++q) {
      const int x = x0 + q;
      if (x < m2) v += s_tk[(uint32_t)skey[x] & 0xfffu];
    }
    unsigned long long tot;
    const unsigned long long e = block_excl_scan_u64(v, sred, &tot);
    uint32_t slot = (uint32_t)(base + e);
    for (int q = 0; q < per2; ++q) {
      const int x = x0 + q;
      if (x >= m2) break;
      const uint32_t i = (uint32_t)skey[x] & 0xfffu;
      J.slot[jbase + x] = slot;
      J.id[jbase + x] = i;
      J.cnt[jbase + x] = s_tk[i] | ((uint32_t)kTaskMerge << 30);
      slot += s_tk[i];
    }
    base += tot;
    jbase += (uint32_t)m2;
  }
  if (tid == 0) {
    met->phaseA = totA;
    met->max_depth = (unsigned long long)dmax;
    met->n_tasks = base;
    met->n_jobs = jbase;
    met->cursorA = totA;
    met->task_ctr = totA;
    met->task_ctr_A = 0;
  }
  RS_TSD(met, 4);
  RS_TS(met, 9);
}

// All blocks, after the grid barrier that follows small_tree: one task per
// thread, grid-stride; the job is the last one whose first slot is <= the task.
__device__ void small_fill(const ClassifyArgs& A, SmallJobs J, unsigned char* smem_small) {
  const DevMetrics* met = A.met;
  const uint32_t nj = (uint32_t)met->n_jobs;
  const unsigned long long ntask = met->n_tasks;
  const uint32_t mbase = (uint32_t)met->phaseA;
  uint32_t* sslot = reinterpret_cast<uint32_t*>(smem_small);
  copy_g2s(sslot, J.slot, (int)nj, threadIdx.x, blockDim.x);
  __syncthreads();
  for (unsigned long long q = blockIdx.x * (unsigned long long)blockDim.x + threadIdx.x; q < ntask;
       q += (unsigned long long)gridDim.x * blockDim.x) {
    uint32_t lo = 0, hi = nj - 1;  // last job k with sslot[k] <= q
    while (lo < hi) {
      uint32_t md = (lo + hi + 1) >> 1;
      if (sslot[md] <= (uint32_t)q) lo = md; else hi = md - 1;
    }
    const uint32_t c = J.cnt[lo], id = J.id[lo];
    const uint32_t kind = c >> 30, k = (uint32_t)q - sslot[lo];
    if (kind == kTaskMerge) store_merge_task(A, (uint32_t)q, mbase, J.md[id], k);
    else A.tasks[q] = make_task(kind, kind == kTaskFuse ? 0u : k, id);
  }
}

}  // namespace rs
