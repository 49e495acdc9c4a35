// rs_small.cuh -- the tree half of the prep (node powers, ancestor scans, trie
// ranges, classification, ordered task list) for trees of at most kSmallR
// leaves, in ONE 1024-thread CTA working out of shared memory.
//
// Same outputs as k_prep's phases 5-9 (rs_tree.cuh, rs_exec.cuh: d_scan_reduce,
// d_scan_down, d_tree, d_classify, d_task_offsets/d_order_scan, d_task_fill),
// with the merge tasks in the identical (depth desc, position) order.  With few
// leaves those phases are pure latency: each is a chain of L2 round trips plus
// a grid barrier over hundreds of mostly idle CTAs.  Here the chains run at
// shared-memory latency behind __syncthreads.  k_prep runs this in block 0
// (the other blocks exit) when n_leaves <= kSmallR.
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
constexpr int kSmallR = 2048;  // above this the grid-wide phases of k_prep are faster

__host__ __device__ constexpr size_t small_arrays_bytes() {
  return (size_t)(kSmallR + 1) * 8      // Ls: leaf starts
         + (size_t)kSmallR * 8          // Ks: midpoint keys, later node spans
         + (size_t)2 * kSmallR * 4      // par: parents of leaves [0, r) and nodes [r, 2r)
         + (size_t)(kSmallR + 1) * 5;   // Ps, las, ras, dep, ldep
}
constexpr size_t kSmallMdOff = (small_arrays_bytes() + 15) / 16 * 16;  // + one round of merge descriptors
__host__ __device__ constexpr size_t small_smem_bytes() { return kSmallMdOff + 256 * 48; }

// Run by one CTA of NT threads (block 0 of k_prep after its leaf phase);
// smem_small: small_smem_bytes() of dynamic shared memory.
template <int NT>
__device__ void small_tree(const TreeArrays& T, ClassifyArgs A, int F, unsigned char* smem_small) {
  constexpr int kSmallPer = (kSmallR + NT - 1) / NT;  // items per thread
  DevMetrics* met = A.met;
  const int64_t r = (int64_t)met->n_leaves;
  if (r > kSmallR || r < 1) return;
  set_fuse_policy(A, r);
  RS_TS(met, 5);
  pos_t* Ls = reinterpret_cast<pos_t*>(smem_small);
  uint64_t* Ks = reinterpret_cast<uint64_t*>(Ls + kSmallR + 1);
  pos_t* spans = reinterpret_cast<pos_t*>(Ks);  // after the trie ranges
  int32_t* par = reinterpret_cast<int32_t*>(Ks + kSmallR);
  uint8_t* Ps = reinterpret_cast<uint8_t*>(par + 2 * kSmallR);
  uint8_t* las = Ps + kSmallR + 1;
  uint8_t* ras = las + kSmallR + 1;
  uint8_t* dep = ras + kSmallR + 1;
  uint8_t* ldep = dep + kSmallR + 1;
  __shared__ MC smc[33];
  __shared__ unsigned long long sred[32];
  __shared__ uint32_t sscan[40];
  __shared__ unsigned s_maxd;

  const int tid = threadIdx.x, nt = blockDim.x;
  const pos_t n = A.n;
  const int64_t m = r - 1;  // boundaries 1..m
  uint64_t* Kg = const_cast<uint64_t*>(T.K);
  uint8_t* Pg = const_cast<uint8_t*>(T.P);
  uint8_t* lag = const_cast<uint8_t*>(T.la);
  uint8_t* rag = const_cast<uint8_t*>(T.ra);

  for (int64_t i = tid; i <= r; i += nt) Ls[i] = T.leaf_start[i];
  if (tid == 0) s_maxd = 0;
  __syncthreads();
  // ---- keys and powers (sorters.py:414-423 via the midpoint-key closed form)
  for (int64_t i = tid; i < r; i += nt) {
    uint64_t k = mid_key(Ls[i], Ls[i + 1], n, F);
    Ks[i] = k;
    Kg[i] = k;
  }
  __syncthreads();
  for (int64_t j = 1 + tid; j < r; j += nt) {
    int p = F + 1 - bitlen64(Ks[j - 1] ^ Ks[j]);
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
  pos_t myspan[kSmallPer];
#pragma unroll kSmallUnroll
  for (int q = 0; q < kSmallPer; ++q) {
    int64_t i = tid + (int64_t)q * nt;
    myspan[q] = 0;
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
      par[i] = (int32_t)p;
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
      while (x >= 0 && Ks[x] >= lo_key) { hi = x; step <<= 1; x = j - 1 - step; }
      int64_t lo = x < 0 ? 0 : x + 1;
      while (lo < hi) {
        int64_t md = lo + (hi - lo) / 2;
        if (Ks[md] >= lo_key) hi = md; else lo = md + 1;
      }
      int64_t a = lo, b;
      if (sh >= 64) b = r - 1;
      else {
        uint64_t hi_key = (pre + 1) << sh;
        int64_t lo2 = j;
        step = 1;
        x = j + step;
        while (x <= r - 1 && Ks[x] < hi_key) { lo2 = x; step <<= 1; x = j + step; }
        int64_t hi2 = x > r - 1 ? r - 1 : x - 1;
        while (lo2 < hi2) {
          int64_t md = lo2 + (hi2 - lo2 + 1) / 2;
          if (Ks[md] < hi_key) lo2 = md; else hi2 = md - 1;
        }
        b = lo2;
      }
      T.node_a[j] = (int32_t)a;
      T.node_b[j] = (int32_t)b;
      pos_t s0 = Ls[a], e0 = Ls[b + 1];
      T.node_s[j] = s0;
      T.node_e[j] = e0;
      // bit 62: not fusable (fusable_span: node table, average leaf length)
      myspan[q] = (e0 - s0) | (fusable_span(A, e0 - s0, b - a) ? (pos_t)0 : ((pos_t)1 << 62));
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
      par[r + j] = (int32_t)pp;
      if (pp >= 0) T.child[2 * pp + side] = (uint32_t)j;
    }
  }
  __syncthreads();  // Ks dead from here: spans reuse it
#pragma unroll kSmallUnroll
  for (int q = 0; q < kSmallPer; ++q) {
    int64_t i = tid + (int64_t)q * nt;
    if (i < r) spans[i] = myspan[q];
  }
  __syncthreads();
  RS_TS(met, 7);
  // ---- classification (d_classify), contiguous items per thread
  const int64_t per = (r + nt - 1) / nt;
  const int64_t i0 = (int64_t)tid * per;
  constexpr pos_t kNoFuse = (pos_t)1 << 62;
  auto fusable_s = [&](int64_t j) { return spans[j] <= A.fcap; };  // kNoFuse set -> > fcap
  auto parent_small_s = [&](int32_t p) { return p >= 0 && fusable_s(p); };
  unsigned long long comps = 0, mcost = 0, mbig = 0;
  uint32_t cntA = 0;
  unsigned maxd = 0;
  uint32_t tk_of[kSmallPer];   // merge tasks of node i0+q (0 unless big)
  uint32_t a_of[kSmallPer];    // phase-A tasks of item i0+q
  uint8_t lcls[kSmallPer], ncls[kSmallPer];
#pragma unroll kSmallUnroll
  for (int q = 0; q < kSmallPer; ++q) {
    int64_t i = i0 + q;
    tk_of[q] = 0;
    a_of[q] = 0;
    lcls[q] = 0;
    ncls[q] = 0;
    if (q >= per || i >= r) continue;
    pos_t s0 = Ls[i], len = Ls[i + 1] - s0;
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
    lcls[q] = (uint8_t)c;
    a_of[q] = c == 1 ? 1u : (uint32_t)tl;
    if (i >= 1) {
      bool fz = fusable_s(i);
      pos_t span = spans[i] & (kNoFuse - 1);
      mcost += span;
      if (!A.classic) comps += span;  // runcore.py:299-301
      int cn;
      if (fz) cn = parent_small_s(par[r + i]) ? 0 : 1;
      else cn = 2;
      A.cls[i] = (uint8_t)cn;
      ncls[q] = (uint8_t)cn;
      if (cn == 1) {
        A.need[i] = 1;
        a_of[q] += 1;
      } else if (cn == 2) {
        int64_t tn = ceil_div64(span, A.mtile);
        A.need[i] = (uint32_t)tn;
        tk_of[q] = (uint32_t)ceil_div64(tn, A.msuper);
        mbig += span;
        maxd = dep[i] > maxd ? dep[i] : maxd;
      } else A.need[i] = 0;
    }
    cntA += a_of[q];
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
  // ---- task records.  Slots come from block scans; the records are written
  // from a job list {first slot, id, count | kind << 30} (in the dead Ks / par
  // regions) by whole warps, so a node with many tiles is not written by one thread.
  __syncthreads();  // classification reads of spans / par are over
  uint32_t* jslot = reinterpret_cast<uint32_t*>(Ks);
  uint32_t* jid = jslot + kSmallR;
  uint32_t* jcnt = reinterpret_cast<uint32_t*>(par);
  __shared__ uint32_t s_nj;
  const int wid = tid >> 5, lane = tid & 31, nw = nt >> 5;
  auto push = [&](uint32_t slot, uint32_t id, uint32_t cnt, uint32_t kind) {
    uint32_t e = atomicAdd(&s_nj, 1u);
    jslot[e] = slot;
    jid[e] = id;
    jcnt[e] = cnt | (kind << 30);
  };
  uint32_t s_mbase = 0;  // first merge-task slot (set once the phase-A count is known)
  auto drain = [&]() {
    __syncthreads();
    uint32_t nj = s_nj;
    MDesc* s_md = reinterpret_cast<MDesc*>(smem_small + kSmallMdOff);
    for (uint32_t g = 0; g < nj; g += nt) {
      // merge descriptors of this round's jobs: one thread per job, parallel round trips
      uint32_t e = g + tid;
      if (e < nj && (jcnt[e] >> 30) == kTaskMerge) s_md[tid] = load_mdesc(A, jid[e]);
      __syncthreads();
      uint32_t ny = nj - g < (uint32_t)nt ? nj - g : (uint32_t)nt;
      for (uint32_t y = wid; y < ny; y += nw) {
        uint32_t slot = jslot[g + y], id = jid[g + y], c = jcnt[g + y];
        uint32_t kind = c >> 30, cnt = c & 0x3fffffffu;
        if (kind == kTaskMerge) {
          const MDesc md = s_md[y];
          for (uint32_t k = lane; k < cnt; k += 32) store_merge_task(A, slot + k, s_mbase, md, k);
        } else {
          for (uint32_t k = lane; k < cnt; k += 32) A.tasks[slot + k] = make_task(kind, kind == kTaskFuse ? 0 : k, id);
        }
      }
      __syncthreads();
    }
    __syncthreads();
    if (tid == 0) s_nj = 0;
    __syncthreads();
  };
  if (tid == 0) s_nj = 0;
  // phase-A tasks (any order; here by position)
  uint32_t totA;
  uint32_t slotA = block_excl_scan_u32(cntA, sscan, &totA);
  s_mbase = totA;  // first merge-task slot
#pragma unroll kSmallUnroll
  for (int q = 0; q < kSmallPer; ++q) {
    int64_t i = i0 + q;
    if (q >= per || i >= r) continue;
    uint32_t lid = A.leaf_base + (uint32_t)i;
    if (lcls[q] == 1) push(slotA++, lid, 1u, kTaskFuse);
    else if (lcls[q] == 2) {
      uint32_t tl = a_of[q] - (ncls[q] == 1 ? 1u : 0u);
      push(slotA, lid, tl, kTaskLeaf);
      slotA += tl;
    }
    if (ncls[q] == 1) push(slotA++, (uint32_t)i, 1u, kTaskFuse);
  }
  drain();
  // merge tasks: depth desc, then position (d_task_offsets + d_task_fill)
  const int dmax = (int)s_maxd;
  uint64_t base = totA;
  for (int d = dmax; d >= 0; --d) {
    uint32_t mine = 0;
#pragma unroll kSmallUnroll
    for (int q = 0; q < kSmallPer; ++q)
      if (q < per && i0 + q < r && ncls[q] == 2 && dep[i0 + q] == d) mine += tk_of[q];
    uint32_t tot;
    uint32_t slot = block_excl_scan_u32(mine, sscan, &tot);
    if (tid == 0) {
      met->depth_tiles[d] = tot;
      met->depth_base[d] = base;
      met->depth_cursor[d] = base;
    }
    slot += (uint32_t)base;
#pragma unroll kSmallUnroll
    for (int q = 0; q < kSmallPer; ++q) {
      int64_t i = i0 + q;
      if (q < per && i < r && ncls[q] == 2 && dep[i] == d) {
        push(slot, (uint32_t)i, tk_of[q], kTaskMerge);
        slot += tk_of[q];
      }
    }
    base += tot;
  }
  drain();
  if (tid == 0) {
    met->phaseA = totA;
    met->max_depth = (unsigned long long)dmax;
    met->n_tasks = base;
    met->cursorA = totA;
    met->task_ctr = totA;
    met->task_ctr_A = 0;
  }
  RS_TS(met, 9);
}

}  // namespace rs
