// rs_exec.cuh -- leaf formation and dataflow execution of the merge tree.
//
// Reference: runcore.py:70-74 (reverse_range), runcore.py:215-248
// (insertionsort_presorted and its exact comparison count), runcore.py:251-326
// (stable two-run merge, ties to the left run; bitonic / classic comparison
// accounting), sorters.py:474-516 (every pending run merged exactly once).
//
// Layout: keys/tags live in three HBM buffers: buf[0] = the caller's array,
// buf[1], buf[2] = scratch.  Phase-A items (leaves, fused subtrees) are formed
// IN PLACE in buf[0], except at depth 1 where they go to buf[2]; a merge node
// at depth d >= 1 writes buf[1 + (d & 1)] and the root writes buf[0].  So a
// parent at depth d reads merge children from buf[node_buf(d + 1)], which it
// does not write, and phase-A children from buf[0] (d >= 1) or buf[2] (root);
// it overwrites only data of its grandchildren, already consumed by its
// (complete) children; and the root, which runs last, is the only writer of
// buf[0] after phase A.  Natural ascending leaves therefore cost nothing, and
// descending ones one in-place reversal.
//
// One persistent kernel claims tasks in list order: first the "phase A" tasks
// (fused subtrees whose span fits in shared memory -- leaves are formed and all
// their merges run in SMEM -- and tiles of large leaves), then merge tiles of
// large nodes, deepest first.  Every task's inputs come from earlier tasks, so
// waiting on per-node completion counters cannot deadlock while all CTAs are
// resident.
#pragma once
#include "rs_common.cuh"

namespace rs {

template <typename K, int TB>
struct ExecCfg {
  static constexpr int kb = sizeof(K);
  static constexpr int eb = kb + TB;
  static constexpr int IPT = (kb == 4) ? 15 : 11;  // odd: conflict-free blocked->smem writes
  static constexpr int TILE = kExecThreads * IPT;
  static constexpr int FCAP = (eb <= 8) ? 4096 : 2048;  // fused-subtree capacity (elements)
  static constexpr int MAXB = FCAP / 2 + 2;             // boundaries inside a fused subtree (any w)
};

template <int TB> struct TagT { using type = uint32_t; };
template <> struct TagT<8> { using type = uint64_t; };

struct ExecArgs {
  void* key[3];
  void* tag[3];
  pos_t n;
  int w;
  int classic;
  uint32_t leaf_base;
  const pos_t* leaf_start;
  const uint32_t* leaf_info;
  const uint8_t* leaf_depth;
  const uint8_t* depth;
  const int32_t* node_a;
  const int32_t* node_b;
  const pos_t* node_s;
  const pos_t* node_e;
  const uint32_t* child;
  const uint32_t* need;
  uint32_t* done;
  const uint64_t* tasks;
  DevMetrics* met;
  int maxb;  // node-table capacity of a fused subtree: FCAP / max(w, 2) + 2
};

// scratch buffer of a merge node at depth d (root: the caller's array)
__device__ __forceinline__ int node_buf(int d) { return d == 0 ? 0 : 1 + (d & 1); }
// where a phase-A item (leaf, fused subtree) at depth d leaves its sorted span
__device__ __forceinline__ int item_buf(int d) { return d == 1 ? 2 : 0; }
// big natural leaf at depth d: in place in buf[0], or (d == 1) copied to buf[2]
__device__ __forceinline__ int leaf_mode(bool desc, int d) {
  return d == 1 ? (desc ? kLeafRevCopy : kLeafCopy) : (desc ? kLeafSwap : kLeafNone);
}
__device__ __forceinline__ int64_t leaf_tiles(pos_t len, int mode, int tile) {
  if (mode == kLeafNone) return 0;
  if (mode == kLeafSwap) {
    int64_t half = tile / 2;
    return ceil_div64(len / 2, half);
  }
  return ceil_div64(len, tile);
}

// ---------------------------------------------------------------- T4: tasks
struct ClassifyArgs {
  pos_t n;
  int w;
  int classic;
  int fcap;
  int tile;   // leaf-tile granularity (phase A)
  int mtile;  // merge-tile granularity (merge executor)
  int msuper; // merge tiles per merge task
  int peek;   // no run-detection comparison term (peeksort counted its scans; top-down/bottom-up detect none)
  int runtime_merges;  // merges may be skipped at run time: merge_cost / merge comparisons counted by the executor
  uint32_t leaf_base;
  const pos_t* leaf_start;
  const uint32_t* leaf_info;
  const uint8_t* leaf_depth;
  const uint8_t* depth;
  const pos_t* node_s;
  const pos_t* node_e;
  const int32_t* parent;
  uint32_t* need;
  uint8_t* cls;  // unified id -> 0 none, 1 fused root, 2 big (tiles in need[])
  uint64_t* tasks;
  DevMetrics* met;
  const int32_t* node_a;
  const int32_t* node_b;
  int maxb;      // ExecArgs::maxb
  int fuse_avg;  // fused subtrees: average leaf length below this
  const uint32_t* child;
  MDesc* mdesc;      // per merge task, index = task slot - first merge slot (met->phaseA)
  int64_t mdesc_cap;
  // k_prep's grid path: the ancestor counts, from which classification derives
  // (and writes) depth / leaf_depth itself -- the trie phase then no longer
  // waits for the ancestor scans (null: depths are already in place)
  const uint8_t* la = nullptr;
  const uint8_t* ra = nullptr;
  // small-tree path: ready-time model of the merge-job order (ns; rs_small.cuh)
  int est_c0 = 6000;  // one tile's latency through the executor
  int est_c1 = 12;    // a tile's service time over the whole grid
  int small_fuse = 1; // small-tree path: fuse subtrees of >= 3 leaves even when the leaves are long on average
};

// Merge descriptor of node i (two dependent round trips: the node's fields,
// then its children's counts and classes).
__device__ __forceinline__ MDesc load_mdesc(const ClassifyArgs& A, uint32_t i) {
  MDesc md;
  pos_t s0 = A.node_s[i];
  md.e = A.node_e[i];
  pos_t m = A.leaf_start[i];
  md.c0 = A.child[2 * i];
  md.c1 = A.child[2 * i + 1];
  pos_t d = A.depth[i];
  md.nd0 = A.need[md.c0];
  md.nd1 = A.need[md.c1];
  uint8_t cl0 = md.c0 < A.leaf_base ? A.cls[md.c0] : 0, cl1 = md.c1 < A.leaf_base ? A.cls[md.c1] : 0;
  pos_t cl = (cl0 == 2 ? 1 : 0) | (cl1 == 2 ? 2 : 0);
  md.s_d = s0 | (d << 56);
  md.m_cl = m | (cl << 56);
  md.j = i;
  md.sk = 0;
  return md;
}

// Task record + descriptor of the k-th task of the node described by md
// (three 16-byte stores assembled in registers).
__device__ __forceinline__ void store_merge_task(const ClassifyArgs& A, uint32_t t, uint32_t mbase, const MDesc& md,
                                                 uint32_t k) {
  A.tasks[t] = make_task(kTaskMerge, k, md.j);
  if ((int64_t)(t - mbase) >= A.mdesc_cap) return;  // beyond the layout bound: the producer walks the node arrays
  uint4* d = reinterpret_cast<uint4*>(A.mdesc + (t - mbase));
  const uint64_t sd = (uint64_t)md.s_d, mc = (uint64_t)md.m_cl, e = (uint64_t)md.e;
  d[0] = make_uint4((uint32_t)sd, (uint32_t)(sd >> 32), (uint32_t)mc, (uint32_t)(mc >> 32));
  d[1] = make_uint4((uint32_t)e, (uint32_t)(e >> 32), md.c0, md.c1);
  d[2] = make_uint4(md.nd0, md.nd1, md.j, k);
}

// Node j can run as (part of) one fused phase-A task: its span fits the fused
// capacity and its internal nodes fit the task's node table (both monotone, so
// "parent fusable" decides membership).
__device__ __forceinline__ bool fusable_span(const ClassifyArgs& A, pos_t span, int64_t nodes) {
  return span <= A.fcap && nodes <= A.maxb - 2;
}
// Fused subtrees pay for short leaves (insertion sorts, several merge levels in
// SMEM); runs averaging >= fuse_avg elements merge faster in the pipelined
// executor, so then only insertion-sort leaves are phase-A tasks (fcap -> 0).
__device__ __forceinline__ void set_fuse_policy(ClassifyArgs& A, int64_t r) {
  if (A.n >= (pos_t)A.fuse_avg * r) A.fcap = 0;
}
__device__ __forceinline__ bool fusable(const ClassifyArgs& A, int32_t j) {
  return fusable_span(A, A.node_e[j] - A.node_s[j], A.node_b[j] - A.node_a[j]);
}
__device__ __forceinline__ bool parent_small(const ClassifyArgs& A, int32_t par) {
  return par >= 0 && fusable(A, par);
}

// Per element: 0 = nothing, 1 = fused root, 2 = big (tiles > 0).  *tiles out.
__device__ __forceinline__ int classify_leaf(const ClassifyArgs& A, int64_t i, int64_t* tiles) {
  pos_t len = A.leaf_start[i + 1] - A.leaf_start[i];
  uint32_t lid = A.leaf_base + (uint32_t)i;
  *tiles = 0;
  if (len <= A.fcap && parent_small(A, A.parent[lid])) return 0;  // inside a fused subtree
  uint32_t info = A.leaf_info[i];
  uint32_t nl = info & 0x7fffffffu;
  if (nl < (uint32_t)A.w && (pos_t)nl < len) return 1;  // extended by insertion sort: fused task
  bool desc = (info >> 31) != 0;
  int mode = leaf_mode(desc, A.leaf_depth[i]);
  *tiles = leaf_tiles(len, mode, A.tile);
  return *tiles > 0 ? 2 : 0;
}
// Big nodes: *tiles = merge tiles (the node's completion count), *tasks = super tasks.
__device__ __forceinline__ int classify_node(const ClassifyArgs& A, int64_t j, int64_t* tiles, int64_t* tasks) {
  pos_t span = A.node_e[j] - A.node_s[j];
  *tiles = 0;
  *tasks = 0;
  if (fusable(A, (int32_t)j)) return parent_small(A, A.parent[j]) ? 0 : 1;
  *tiles = ceil_div64(span, A.mtile);
  *tasks = ceil_div64(*tiles, A.msuper);
  return 2;
}

// Chunks of kOrdChunk elements (leaf i and boundary j = i).  Merge tasks are
// ordered by depth (deepest first) and, within a depth, by position, so a
// node's tasks are claimed after the wave of its children's tasks has passed.
constexpr int kOrdChunkMin = 256, kOrdChunkMax = 4096;
// d_task_fill's shared-memory staging: slots, tile counts, depths, then one round of merge descriptors
constexpr int kFillMdOff = (kOrdChunkMax * 9 + 15) / 16 * 16;
constexpr int kFillSmem = kFillMdOff + 256 * 48;
// Chunk of boundaries for the ordered fill: small trees -> many small chunks.
__host__ __device__ inline int64_t ord_chunk(int64_t r) {
  int64_t c = kOrdChunkMin;
  while (c < kOrdChunkMax && c * 512 < r) c <<= 1;
  return c;
}

// Element-parallel: leaf i and boundary j = i per thread.  Big nodes add their
// task count to their (chunk, depth) cell for the ordered fill.
__device__ void d_classify(ClassifyArgs A, uint32_t* __restrict__ chunk_depth) {
  __shared__ unsigned long long sred[32];
  __shared__ uint32_t s_cd[kMaxDepth];  // this iteration's per-depth task counts (one chunk)
  int64_t r = (int64_t)A.met->n_leaves;
  set_fuse_policy(A, r);
  const int64_t ochunk = ord_chunk(r);  // a multiple of blockDim: one chunk per block iteration
  unsigned long long comps = 0, mcost = 0, cntA = 0, mbig = 0;
  unsigned long long dtl = 0;  // thread d < kMaxDepth: tasks of depth d over all iterations
  unsigned maxd = 0;
  for (int64_t i0 = blockIdx.x * (int64_t)blockDim.x; i0 < r; i0 += (int64_t)gridDim.x * blockDim.x) {
    for (int d = threadIdx.x; d < kMaxDepth; d += blockDim.x) s_cd[d] = 0;
    __syncthreads();
    const int64_t i = i0 + threadIdx.x;
    if (i < r) {
    if (A.la) {  // depths from the ancestor counts (sorters.py:500-502: depth = left + right ancestors)
      int32_t pl = A.parent[A.leaf_base + (uint32_t)i];
      const_cast<uint8_t*>(A.leaf_depth)[i] = pl >= 0 ? (uint8_t)(A.la[pl] + A.ra[pl] + 1) : (uint8_t)0;
      if (i >= 1) const_cast<uint8_t*>(A.depth)[i] = (uint8_t)(A.la[i] + A.ra[i]);
    }
    // leaf: detection comparisons (runcore.py:154/157 closed form)
    pos_t s0 = A.leaf_start[i], len = A.leaf_start[i + 1] - s0;
    if (!A.peek && s0 < A.n - 1) {
      uint32_t nl = A.leaf_info[i] & 0x7fffffffu;
      pos_t L = (nl >= (uint32_t)A.w) ? len : (pos_t)nl;
      pos_t ne = s0 + L - 1;
      comps += (unsigned long long)((ne < A.n - 1) ? L : L - 1);
    }
    int64_t tl;
    int c = classify_leaf(A, i, &tl);
    uint32_t lid = A.leaf_base + (uint32_t)i;
    A.need[lid] = c == 1 ? 1u : (uint32_t)tl;
    A.cls[lid] = (uint8_t)c;
    cntA += c == 1 ? 1 : (unsigned long long)tl;
    if (i >= 1) {
      pos_t span = A.node_e[i] - A.node_s[i];
      if (!A.runtime_merges) {
        mcost += span;
        if (!A.classic) comps += span;  // runcore.py:299-301
      }
      int64_t tn, tk;
      int cn = classify_node(A, i, &tn, &tk);
      A.cls[i] = (uint8_t)cn;
      if (cn == 1) { A.need[i] = 1; cntA += 1; }
      else if (cn == 2) {
        A.need[i] = (uint32_t)tn;
        mbig += span;
        int d = A.depth[i];
        atomicAdd(&s_cd[d], (uint32_t)tk);
        maxd = d > (int)maxd ? d : maxd;
      } else A.need[i] = 0;
    }
    }
    __syncthreads();
    for (int d = threadIdx.x; d < kMaxDepth; d += blockDim.x) {
      uint32_t v = s_cd[d];
      if (v) {
        atomicAdd(&chunk_depth[(i0 / ochunk) * kMaxDepth + d], v);
        dtl += v;
      }
    }
  }
  if (threadIdx.x < kMaxDepth && dtl) atomicAdd(&A.met->depth_tiles[threadIdx.x], dtl);
  unsigned long long s = block_sum(comps, sred);
  if (threadIdx.x == 0 && s) atomicAdd(&A.met->comparisons, s);
  s = block_sum(mcost, sred);
  if (threadIdx.x == 0 && s) atomicAdd(&A.met->merge_cost, s);
  s = block_sum(cntA, sred);
  if (threadIdx.x == 0 && s) atomicAdd(&A.met->phaseA, s);
  s = block_sum(mbig, sred);
  if (threadIdx.x == 0 && s) atomicAdd(&A.met->merge_cost_exec, s);
  maxd = warp_max(maxd);
  if ((threadIdx.x & 31) == 0 && maxd) atomicMax(&A.met->max_depth, (unsigned long long)maxd);
}

// Run by one whole block: per-depth slot bases (deepest first, after the
// phase-A tasks), then per depth the exclusive scan of the chunk task counts.
// Loads are issued in parallel / in batches (a load-store loop over global
// memory would serialize one round trip per iteration).
__device__ void d_task_offsets(DevMetrics* met) {
  __shared__ unsigned long long s_dt[kMaxDepth];
  __shared__ unsigned long long s_pa;
  __shared__ int s_md;
  for (int d = threadIdx.x; d < kMaxDepth; d += blockDim.x) s_dt[d] = met->depth_tiles[d];
  if (threadIdx.x == 0) {
    s_pa = met->phaseA;
    s_md = (int)met->max_depth;
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    unsigned long long base = s_pa;
    for (int d = s_md; d >= 0; --d) {
      unsigned long long v = s_dt[d];
      s_dt[d] = base;
      base += v;
    }
    met->n_tasks = base;
    met->cursorA = 0;
    met->task_ctr = s_pa;
    met->task_ctr_A = 0;
  }
  __syncthreads();
  for (int d = threadIdx.x; d <= s_md; d += blockDim.x) {
    met->depth_base[d] = s_dt[d];
    met->depth_cursor[d] = s_dt[d];
  }
}

// Per depth: exclusive scan of the chunk task counts, offset by depth_base.
__device__ void d_order_scan(const DevMetrics* __restrict__ met, uint32_t* __restrict__ chunk_depth) {
  int d = threadIdx.x;
  if (d >= kMaxDepth) return;
  int64_t r = (int64_t)met->n_leaves;
  int64_t oc = ord_chunk(r);
  int64_t nch = (r + oc - 1) / oc;
  uint32_t run = (uint32_t)met->depth_base[d];
  for (int64_t c = 0; c < nch; ++c) {
    uint32_t v = chunk_depth[c * kMaxDepth + d];
    chunk_depth[c * kMaxDepth + d] = run;
    run += v;
  }
}

__device__ void d_task_fill(ClassifyArgs A, const uint32_t* __restrict__ chunk_depth) {
  __shared__ uint32_t run[kMaxDepth];
  __shared__ uint32_t s_wsum[kMaxDepth * 8];  // [depth][warp]: warp totals, then warp offsets
  // staging lives in the kernel's dynamic shared memory (dead by this phase)
  extern __shared__ __align__(16) unsigned char smem_fill[];
  uint32_t* s_slot = reinterpret_cast<uint32_t*>(smem_fill);
  uint32_t* s_tk = s_slot + kOrdChunkMax;
  uint8_t* s_dep = smem_fill + kOrdChunkMax * 8;
  int64_t r = (int64_t)A.met->n_leaves;
  // phase-A tasks (any order): element-parallel, slots from one atomic per block
  __shared__ uint32_t s_sc[40];
  __shared__ unsigned long long s_base;
  for (int64_t i0 = blockIdx.x * (int64_t)blockDim.x; i0 < r; i0 += (int64_t)gridDim.x * blockDim.x) {
    const int64_t i = i0 + threadIdx.x;
    int c = 0, cn = 0;
    uint32_t tl = 0, lid = 0;
    if (i < r) {
      lid = A.leaf_base + (uint32_t)i;
      c = A.cls[lid];
      if (c == 2) tl = A.need[lid];
      if (i >= 1) cn = A.cls[i];
    }
    uint32_t cnt = (c == 1 ? 1u : (c == 2 ? tl : 0u)) + (cn == 1 ? 1u : 0u);
    uint32_t tot;
    uint32_t pre = block_excl_scan_u32(cnt, s_sc, &tot);
    if (threadIdx.x == 0) s_base = tot ? atomicAdd(&A.met->cursorA, (unsigned long long)tot) : 0ull;
    __syncthreads();
    unsigned long long slot = s_base + pre;
    if (c == 1) A.tasks[slot++] = make_task(kTaskFuse, 0, lid);
    else if (c == 2)
      for (uint32_t k = 0; k < tl; ++k) A.tasks[slot++] = make_task(kTaskLeaf, k, lid);
    if (cn == 1) A.tasks[slot++] = make_task(kTaskFuse, 0, (uint32_t)i);
    __syncthreads();
  }
  RS_DBG(A.met, 20);
  // merge tasks: slots by (depth, position); chunk boundaries staged in smem,
  // warp 0 assigns ordered slots, all threads write.
  const int64_t oc = ord_chunk(r);
  int64_t nch = (r + oc - 1) / oc;
  int lane = threadIdx.x & 31;
  // Few chunks (config 2: 13 for 3,230 leaves) would leave the record writes of
  // the tree's top -- thousands of tiles in one chunk -- to a handful of
  // blocks: every chunk is taken by `slices` blocks, which all rank its nodes
  // (cheap, redundant) and each write one slice of its task records.
  const int64_t slices = nch > 0 && (int64_t)gridDim.x / nch > 1 ? (int64_t)gridDim.x / nch : 1;
  for (int64_t vb = blockIdx.x; vb < nch * slices; vb += gridDim.x) {
    const int64_t ch = vb / slices;
    const uint32_t sl = (uint32_t)(vb % slices);
    __syncthreads();
    for (int d = threadIdx.x; d < kMaxDepth; d += blockDim.x) run[d] = chunk_depth[ch * kMaxDepth + d];
    int64_t i0 = ch * oc, i1 = (ch + 1) * oc < r ? (ch + 1) * oc : r;
    int64_t cnt_i = i1 - i0;
    for (int64_t x = threadIdx.x; x < cnt_i; x += blockDim.x) {
      int64_t i = i0 + x;
      uint32_t dv = 0xffu, tv = 0;
      if (i >= 1) {
        int c = A.cls[i];  // independent loads: one round trip
        uint32_t dd = A.depth[i], nd = A.need[i];
        if (c == 2) {
          dv = dd;
          tv = (nd + A.msuper - 1) / (uint32_t)A.msuper;
        }
      }
      s_dep[x] = (uint8_t)dv;
      s_slot[x] = tv;
      s_tk[x] = tv;
    }
    __syncthreads();
    RS_DBG(A.met, 21);
    // ordered slots, 256 nodes per round: every warp ranks its 32 nodes among
    // same-depth peers (shuffle prefix), per-depth warp totals are scanned
    // across warps, and `run` carries each depth's cursor to the next round
    for (int64_t g = 0; g < cnt_i; g += blockDim.x) {
      int64_t x = g + threadIdx.x;
      int d = x < cnt_i ? s_dep[x] : 255;
      uint32_t tk = x < cnt_i ? s_tk[x] : 0;
      uint32_t pre = 0;
#pragma unroll
      for (int k = 1; k < 32; ++k) {
        int dk = __shfl_up_sync(0xffffffffu, d, k);
        uint32_t tkk = __shfl_up_sync(0xffffffffu, tk, k);
        if (lane >= k && dk == d) pre += tkk;
      }
      uint32_t mask = __match_any_sync(0xffffffffu, d);
      const int wid = threadIdx.x >> 5;
      for (int q = threadIdx.x; q < kMaxDepth * 8; q += blockDim.x) s_wsum[q] = 0;
      __syncthreads();
      if (d != 255 && lane == 31 - __clz(mask)) s_wsum[d * 8 + wid] = pre + tk;  // warp total per depth
      __syncthreads();
      if (threadIdx.x < kMaxDepth) {  // depth d: exclusive scan over the 8 warps, advance the cursor
        uint32_t acc = run[threadIdx.x];
        for (int w = 0; w < (int)(blockDim.x >> 5); ++w) {
          uint32_t v = s_wsum[threadIdx.x * 8 + w];
          s_wsum[threadIdx.x * 8 + w] = acc;
          acc += v;
        }
        run[threadIdx.x] = acc;
      }
      __syncthreads();
      if (d != 255) s_slot[x] = s_wsum[d * 8 + wid] + pre;
      __syncthreads();
    }
    // rounds of blockDim nodes: every thread loads one node's merge descriptor
    // into shared memory (parallel round trips), then all threads write the
    // round's task records and per-task descriptors
    RS_DBG(A.met, 22);
    MDesc* s_md = reinterpret_cast<MDesc*>(smem_fill + kFillMdOff);
    const uint32_t mbase = (uint32_t)A.met->phaseA;  // first merge-task slot (final after classification)
    __shared__ uint32_t s_pre[256];  // blockDim == 256
    for (int64_t g = 0; g < cnt_i; g += blockDim.x) {
      int64_t x = g + threadIdx.x;
      const bool big = x < cnt_i && s_dep[x] != 255;
      if (big) s_md[threadIdx.x] = load_mdesc(A, (uint32_t)(i0 + x));
      // flatten the round's tasks over all threads: a node with hundreds of
      // tiles (the top of the tree) is not written by one warp
      uint32_t tot;
      uint32_t pre = block_excl_scan_u32(big ? s_tk[x] : 0u, s_sc, &tot);  // syncs: s_md visible
      s_pre[threadIdx.x] = pre;
      __syncthreads();
      RS_DBG(A.met, 23);
      const int ny = cnt_i - g < (int64_t)blockDim.x ? (int)(cnt_i - g) : (int)blockDim.x;
      for (uint32_t q = sl * blockDim.x + threadIdx.x; q < tot; q += (uint32_t)slices * blockDim.x) {
        int lo = 0, hi = ny - 1;  // last node y with s_pre[y] <= q
        while (lo < hi) {
          int md = (lo + hi + 1) >> 1;
          if (s_pre[md] <= q) lo = md; else hi = md - 1;
        }
        uint32_t k = q - s_pre[lo];
        store_merge_task(A, s_slot[g + lo] + k, mbase, s_md[lo], k);
      }
      __syncthreads();
      RS_DBG(A.met, 24);
    }
  }
}

// ---------------------------------------------------------------- searches
// Number of A elements among the first `diag` outputs of the stable merge of
// sorted A and B (ties: A first).  Whole warp participates; result in all lanes.
template <typename K>
__device__ int64_t warp_merge_path(const K* A, int64_t na, const K* B, int64_t nb, int64_t diag) {
  int lane = threadIdx.x & 31;
  int64_t lo = diag - nb > 0 ? diag - nb : 0;
  int64_t hi = diag < na ? diag : na;
  while (hi - lo > 32) {
    int64_t span = hi - lo;
    int64_t idx = lo + (span * (lane + 1)) / 33;
    bool pred = ldcg(A + idx) <= ldcg(B + (diag - 1 - idx));
    uint32_t bal = __ballot_sync(0xffffffffu, pred);
    int c = __popc(bal);
    int64_t nlo = c > 0 ? __shfl_sync(0xffffffffu, idx, c - 1) + 1 : lo;
    int64_t nhi = c < 32 ? __shfl_sync(0xffffffffu, idx, c < 32 ? c : 31) : hi;
    lo = nlo;
    hi = nhi;
  }
  int64_t idx = lo + lane;
  bool pred = idx < hi && ldcg(A + idx) <= ldcg(B + (diag - 1 - idx));
  return lo + __popc(__ballot_sync(0xffffffffu, pred));
}

// First index in [0, len) where `A[idx] < v` (strict=true) / `A[idx] <= v` fails.
template <typename K>
__device__ int64_t warp_count_below(const K* A, int64_t len, K v, bool or_equal) {
  int lane = threadIdx.x & 31;
  int64_t lo = 0, hi = len;
  while (hi - lo > 32) {
    int64_t span = hi - lo;
    int64_t idx = lo + (span * (lane + 1)) / 33;
    K x = ldcg(A + idx);
    bool pred = or_equal ? (x <= v) : (x < v);
    uint32_t bal = __ballot_sync(0xffffffffu, pred);
    int c = __popc(bal);
    int64_t nlo = c > 0 ? __shfl_sync(0xffffffffu, idx, c - 1) + 1 : lo;
    int64_t nhi = c < 32 ? __shfl_sync(0xffffffffu, idx, c < 32 ? c : 31) : hi;
    lo = nlo;
    hi = nhi;
  }
  int64_t idx = lo + lane;
  bool pred = false;
  if (idx < hi) {
    K x = ldcg(A + idx);
    pred = or_equal ? (x <= v) : (x < v);
  }
  return lo + __popc(__ballot_sync(0xffffffffu, pred));
}

// Thread-level merge path inside shared memory.
template <typename K>
__device__ __forceinline__ int smem_merge_path(const K* A, int na, const K* B, int nb, int diag) {
  int lo = diag - nb > 0 ? diag - nb : 0;
  int hi = diag < na ? diag : na;
  while (lo < hi) {
    int mid = (lo + hi) >> 1;
    if (A[mid] <= B[diag - 1 - mid]) lo = mid + 1; else hi = mid;
  }
  return lo;
}
template <typename K>
__device__ __forceinline__ int smem_count(const K* A, int len, K v, bool or_equal) {
  int lo = 0, hi = len;
  while (lo < hi) {
    int mid = (lo + hi) >> 1;
    bool p = or_equal ? (A[mid] <= v) : (A[mid] < v);
    if (p) lo = mid + 1; else hi = mid;
  }
  return lo;
}

// ------------------------------------------------------------- the executor
template <typename K, int TB>
struct Exec {
  using C = ExecCfg<K, TB>;
  using T = typename TagT<TB>::type;
  static constexpr bool HAS_TAGS = TB != 0;

  static constexpr size_t smem_merge() { return (size_t)C::TILE * (C::kb + TB) + 64; }
  // leaves of a fused subtree are >= max(w, 2) long except the array's last one
  static constexpr int maxb_for(int w) { return C::FCAP / (w > 2 ? w : 2) + 2; }
  // two symmetric span buffers (keys, tags), each with 32 B of bulk-copy alignment slack
  __host__ __device__ static constexpr size_t kbuf_bytes() { return (size_t)C::FCAP * C::kb + 32; }
  __host__ __device__ static constexpr size_t tbuf_bytes() { return HAS_TAGS ? (size_t)C::FCAP * TB + 32 : 0; }
  static constexpr size_t smem_fuse(int maxb) {
    return 2 * (kbuf_bytes() + tbuf_bytes()) + (size_t)(maxb + 1) * (3 * 2 + 1 + 2 + 2 + 2 + 4 + 1) + 256;
  }
  static constexpr size_t smem_bytes(int w) { return smem_fuse(maxb_for(w)); }

  // --- big-leaf tile: in-place reversal, or copy / reversed copy to buf[2] ---
  __device__ static void leaf_task(const ExecArgs& E, uint32_t i, uint32_t k) {
    pos_t s0 = E.leaf_start[i], len = E.leaf_start[i + 1] - s0;
    bool desc = (E.leaf_info[i] >> 31) != 0;
    int mode = leaf_mode(desc, E.leaf_depth[i]);
    K* k0 = reinterpret_cast<K*>(E.key[0]);
    K* k1 = reinterpret_cast<K*>(E.key[2]);  // copies go to the depth-1 buffer
    T* t0 = HAS_TAGS ? reinterpret_cast<T*>(E.tag[0]) : nullptr;
    T* t1 = HAS_TAGS ? reinterpret_cast<T*>(E.tag[2]) : nullptr;
    constexpr int U = 8;
    if (mode == kLeafSwap) {
      int64_t half = C::TILE / 2;
      int64_t x0 = (int64_t)k * half, x1 = x0 + half < len / 2 ? x0 + half : len / 2;
      for (int64_t xb = x0 + threadIdx.x; xb < x1; xb += (int64_t)blockDim.x * U) {
        K a[U], b[U];
        T ta[U], tb[U];
#pragma unroll
        for (int u = 0; u < U; ++u) {
          int64_t x = xb + (int64_t)u * blockDim.x;
          if (x < x1) {
            a[u] = ldcg(k0 + s0 + x);
            b[u] = ldcg(k0 + s0 + len - 1 - x);
            if (HAS_TAGS) { ta[u] = ldcg(t0 + s0 + x); tb[u] = ldcg(t0 + s0 + len - 1 - x); }
          }
        }
#pragma unroll
        for (int u = 0; u < U; ++u) {
          int64_t x = xb + (int64_t)u * blockDim.x;
          if (x < x1) {
            k0[s0 + x] = b[u];
            k0[s0 + len - 1 - x] = a[u];
            if (HAS_TAGS) { t0[s0 + x] = tb[u]; t0[s0 + len - 1 - x] = ta[u]; }
          }
        }
      }
    } else {
      int64_t x0 = (int64_t)k * C::TILE, x1 = x0 + C::TILE < len ? x0 + C::TILE : len;
      bool rev = mode == kLeafRevCopy;
      for (int64_t xb = x0 + threadIdx.x; xb < x1; xb += (int64_t)blockDim.x * U) {
        K a[U];
        T ta[U];
#pragma unroll
        for (int u = 0; u < U; ++u) {
          int64_t x = xb + (int64_t)u * blockDim.x;
          if (x < x1) {
            a[u] = ldcg(k0 + s0 + x);
            if (HAS_TAGS) ta[u] = ldcg(t0 + s0 + x);
          }
        }
#pragma unroll
        for (int u = 0; u < U; ++u) {
          int64_t x = xb + (int64_t)u * blockDim.x;
          if (x < x1) {
            pos_t to = rev ? s0 + len - 1 - x : s0 + x;
            k1[to] = a[u];
            if (HAS_TAGS) t1[to] = ta[u];
          }
        }
      }
    }
  }

  // --- fused subtree: form its leaves and run all of its merges in SMEM ---
  struct Span {
    pos_t s, e;
    int64_t la, lb;
    int droot;
  };
  __device__ static Span span_of(const ExecArgs& E, uint32_t u) {
    Span f;
    if (u >= E.leaf_base) {
      f.la = f.lb = u - E.leaf_base;
      f.s = E.leaf_start[f.la];
      f.e = E.leaf_start[f.la + 1];
      f.droot = E.leaf_depth[f.la];
    } else {
      f.la = E.node_a[u];
      f.lb = E.node_b[u];
      f.s = E.node_s[u];
      f.e = E.node_e[u];
      f.droot = E.depth[u];
    }
    return f;
  }
  __device__ static unsigned char* kbuf(unsigned char* smem, int b) { return smem + (size_t)b * kbuf_bytes(); }
  __device__ static unsigned char* tbuf(unsigned char* smem, int b) {
    return smem + 2 * kbuf_bytes() + (size_t)b * tbuf_bytes();
  }
  // Thread 0: bulk-copy the span's 16B-aligned cover into buffer b; element
  // offsets of the span inside it go to off[0] (keys) / off[1] (tags).
  __device__ static void span_issue(const ExecArgs& E, const Span& f, unsigned char* smem, int b, uint64_t* bar,
                                    int32_t* off) {
    fence_proxy_async_smem();  // earlier generic accesses of the buffer come first
    auto cover = [](const void* base, pos_t e0, pos_t e1, int es) {
      uintptr_t a0 = reinterpret_cast<uintptr_t>(base) + (uintptr_t)e0 * es;
      uintptr_t a1 = reinterpret_cast<uintptr_t>(base) + (uintptr_t)e1 * es;
      return (uint32_t)(((a1 + 15) & ~(uintptr_t)15) - (a0 & ~(uintptr_t)15));
    };
    uint32_t tx = cover(E.key[0], f.s, f.e, C::kb) + (HAS_TAGS ? cover(E.tag[0], f.s, f.e, TB) : 0u);
    mbar_arrive_tx(bar, tx);
    int32_t ok, ot = 0;
    tma_window(kbuf(smem, b), E.key[0], f.s, f.e, C::kb, bar, &ok);
    if (HAS_TAGS) tma_window(tbuf(smem, b), E.tag[0], f.s, f.e, TB, bar, &ot);
    off[0] = ok;
    off[1] = ot;
  }

  // Runs fused task u whose span was issued into buffer ib (offsets in off[]).
  // `hook()` runs in every thread once the span buffers are no longer read
  // except for the write-back of the result (buffer returned by the call); the
  // other buffer is then free.
  template <typename Step, typename Hook>
  __device__ static int fuse_task(const ExecArgs& E, const Span& f, int ib, unsigned char* smem, uint64_t* bar,
                                  uint32_t& fphase, int32_t* off, Step&& step, Hook&& hook,
                                  unsigned long long& comps) {
    __shared__ uint32_t s_scan[40];
    __shared__ int s_dmax;
    K* X[2];
    T* Y[2];
    unsigned char* p = smem + 2 * (kbuf_bytes() + tbuf_bytes());
    const int MB = E.maxb;
    uint16_t* ns = reinterpret_cast<uint16_t*>(p);
    uint16_t* nm = ns + MB;
    uint16_t* ne = nm + MB;
    uint16_t* lst = ne + MB;     // level node list
    uint16_t* loff = lst + MB;   // level output offsets
    uint16_t* lsv = loff + MB;   // leaf starts (MB + 1)
    uint32_t* linf = reinterpret_cast<uint32_t*>(lsv + MB + 2);  // leaf info (MB + 1), 4B-aligned
    uint8_t* ldpv = reinterpret_cast<uint8_t*>(linf + MB + 1);   // leaf depth parity
    uint8_t* dep = ldpv + MB + 1;

    const int64_t la = f.la, lb = f.lb;
    const pos_t s = f.s, e = f.e;
    const int droot = f.droot;
#ifdef RS_INSTR
    long long ti0 = clock64(), ti1 = 0, ti2 = 0, ti3 = 0;
#endif
    int len = int(e - s);
    RS_CHECK(0 < len && len <= C::FCAP && lb >= la && lb - la <= E.maxb - 2, "fuse task s %lld e %lld la %lld lb %lld",
             (long long)s, (long long)e, (long long)la, (long long)lb);
    // the subtree's node table while the span is in flight
    int nbd = int(lb - la);
    int dmax_local = droot;
    if (threadIdx.x == 0) s_dmax = droot;
    for (int x = threadIdx.x; x < nbd; x += blockDim.x) {
      int64_t jj = la + 1 + x;
      ns[x] = (uint16_t)(E.node_s[jj] - s);
      nm[x] = (uint16_t)(E.leaf_start[jj] - s);
      ne[x] = (uint16_t)(E.node_e[jj] - s);
      int dd = E.depth[jj];
      dep[x] = (uint8_t)dd;
      dmax_local = dd > dmax_local ? dd : dmax_local;
    }
    const int nlf = nbd + 1;
    __shared__ int s_nat;  // some leaf is a natural run needing a copy / reversal
    if (threadIdx.x == 0) s_nat = 0;
    __syncthreads();
    bool nat = false;
    for (int x = threadIdx.x; x < nlf; x += blockDim.x) {
      int64_t li = la + x;
      pos_t ls = E.leaf_start[li], le = E.leaf_start[li + 1];
      uint32_t info = E.leaf_info[li];
      uint8_t dp = (uint8_t)(E.leaf_depth[li] & 1);
      lsv[x] = (uint16_t)(ls - s);
      linf[x] = info;
      ldpv[x] = dp;
      uint32_t nl = info & 0x7fffffffu;
      bool natural = nl >= (uint32_t)E.w || (pos_t)nl >= le - ls;
      nat |= natural && ((info >> 31) != 0 || dp == 1);
    }
    if (nat) s_nat = 1;
    if (threadIdx.x == 0) {
      lsv[nlf] = (uint16_t)len;  // len <= FCAP < 65536
      step();
    }
    __syncthreads();
    if (nbd > 0) atomicMax(&s_dmax, dmax_local);
    mbar_wait(bar, fphase);
    fphase ^= 1u;
    X[0] = reinterpret_cast<K*>(kbuf(smem, ib)) + off[0];
    X[1] = reinterpret_cast<K*>(kbuf(smem, ib ^ 1));
    Y[0] = HAS_TAGS ? reinterpret_cast<T*>(tbuf(smem, ib)) + off[1] : nullptr;
    Y[1] = HAS_TAGS ? reinterpret_cast<T*>(tbuf(smem, ib ^ 1)) : nullptr;
#ifdef RS_INSTR
    ti1 = clock64();
#endif
    __builtin_assume(__isShared(X[0]));
    __builtin_assume(__isShared(X[1]));
    if (HAS_TAGS) {
      __builtin_assume(__isShared(Y[0]));
      __builtin_assume(__isShared(Y[1]));
    }
    __syncthreads();
    // leaves.  Natural runs (copy / reversal into the depth-parity buffer):
    // element-parallel over the whole span.  Runs extended by insertion sort
    // (runcore.py:215-248): warp per leaf.
    auto leaf_L = [&](int k, int ll) {
      uint32_t nl = linf[k] & 0x7fffffffu;
      return (nl >= (uint32_t)E.w) ? ll : (int)nl;
    };
    for (int x = s_nat ? (int)threadIdx.x : len; x < len; x += blockDim.x) {
      int lo = 0, hi = nlf - 1;  // last leaf with start <= x
      while (lo < hi) {
        int md = (lo + hi + 1) >> 1;
        if (lsv[md] <= x) lo = md; else hi = md - 1;
      }
      int ls = lsv[lo], le = lsv[lo + 1], ll = le - ls;
      if (leaf_L(lo, ll) < ll) continue;  // insertion-sort leaf: below
      bool desc = (linf[lo] >> 31) != 0;
      int dp = ldpv[lo];
      int r = x - ls;
      if (desc) {
        if (dp == 0) {
          if (r < ll / 2) {
            int y = le - 1 - r;
            K a = X[0][x], b = X[0][y];
            X[0][x] = b;
            X[0][y] = a;
            if (HAS_TAGS) { T ta = Y[0][x]; Y[0][x] = Y[0][y]; Y[0][y] = ta; }
          }
        } else {
          X[1][x] = X[0][le - 1 - r];
          if (HAS_TAGS) Y[1][x] = Y[0][le - 1 - r];
        }
      } else if (dp == 1) {
        X[1][x] = X[0][x];
        if (HAS_TAGS) Y[1][x] = Y[0][x];
      }
    }
    int wid = threadIdx.x >> 5, lane = threadIdx.x & 31, nwarp = blockDim.x >> 5;
    for (int k = wid; k < nlf; k += nwarp) {
      int ls = lsv[k], le = lsv[k + 1], ll = le - ls;
      int L = leaf_L(k, ll);
      if (L >= ll) continue;
      bool desc = (linf[k] >> 31) != 0;
      int dp = ldpv[k];
      {
        // insertionsort_presorted on the post-reversal chunk (runcore.py:215-248)
        int npre = L > 1 ? L : 1;
        auto vidx = [&](int t) { return (desc && t < L) ? ls + L - 1 - t : ls + t; };
        if (ll <= 32) {
          K xv = K(0);
          T tv = T(0);
          if (lane < ll) {
            xv = X[0][vidx(lane)];
            if (HAS_TAGS) tv = Y[0][vidx(lane)];
          }
          int g = 0, rank = 0;
          for (int q = 0; q < ll; ++q) {
            K y = __shfl_sync(0xffffffffu, xv, q);
            if (q < lane) { g += (y > xv); rank += (y <= xv); }
            else if (q > lane) rank += (y < xv);
          }
          unsigned long long c = 0;
          if (lane < ll && lane >= npre) c = (unsigned long long)(g + (g < lane ? 1 : 0));
          comps += c;
          __syncwarp();
          if (lane < ll) {
            X[dp][ls + rank] = xv;
            if (HAS_TAGS) Y[dp][ls + rank] = tv;
          }
        } else {
          K* dstk = X[1];
          T* dstt = Y[1];
          for (int t = lane; t < ll; t += 32) {
            K xv = X[0][vidx(t)];
            int g = 0, rank = 0;
            for (int q = 0; q < ll; ++q) {
              K y = X[0][vidx(q)];
              if (q < t) { g += (y > xv); rank += (y <= xv); }
              else if (q > t) rank += (y < xv);
            }
            if (t >= npre) comps += (unsigned long long)(g + (g < t ? 1 : 0));
            dstk[ls + rank] = xv;
            if (HAS_TAGS) dstt[ls + rank] = Y[0][vidx(t)];
          }
          __syncwarp();
          if (dp == 0) {
            for (int x = lane; x < ll; x += 32) {
              X[0][ls + x] = X[1][ls + x];
              if (HAS_TAGS) Y[0][ls + x] = Y[1][ls + x];
            }
          }
        }
      }
      __syncwarp();
    }
    if (threadIdx.x == 0) step();
    __syncthreads();
#ifdef RS_INSTR
    ti2 = clock64();
#endif
    if (nbd > 0) {
      int dmax = s_dmax;
      const int per = (nbd + blockDim.x - 1) / blockDim.x;
      for (int dd = dmax; dd >= droot; --dd) {
        // this level's nodes in position order with their output offsets
        // (packed nodes << 16 | elements; a level's elements <= FCAP < 2^16)
        uint32_t mine = 0;
        int x0 = threadIdx.x * per;
        for (int q = 0; q < per; ++q) {
          int x = x0 + q;
          if (x < nbd && dep[x] == dd) mine += (1u << 16) + (uint32_t)(ne[x] - ns[x]);
        }
        uint32_t total;
        uint32_t pre = block_excl_scan_u32(mine, s_scan, &total);
        uint32_t nidx = pre >> 16, eoff = pre & 0xffffu;
        for (int q = 0; q < per; ++q) {
          int x = x0 + q;
          if (x < nbd && dep[x] == dd) {
            lst[nidx] = (uint16_t)x;
            loff[nidx] = (uint16_t)eoff;
            ++nidx;
            eoff += ne[x] - ns[x];
          }
        }
        __syncthreads();
        const int nlev = int(total >> 16), tot = int(total & 0xffffu);
        const K* Xs = X[(dd + 1) & 1];
        K* Xd = X[dd & 1];
        const T* Ys = Y[(dd + 1) & 1];
        T* Yd = Y[dd & 1];
        __builtin_assume(__isShared(Xs));  // keep LDS/STS (not generic) in the merge loop
        __builtin_assume(__isShared(Xd));
        if (HAS_TAGS) {
          __builtin_assume(__isShared(Ys));
          __builtin_assume(__isShared(Yd));
        }
        // every thread merges one equal share of the level's concatenated output
        // odd shares: thread t starts at output t * cs, so the merge's reads and
        // writes of neighbouring threads fall in different banks (an even share,
        // 16 for a 4096-element span, made them 16-way conflicted)
        const int cs = ((tot + (int)blockDim.x - 1) / (int)blockDim.x) | 1;
        int o0 = threadIdx.x * cs;
        const int o1 = o0 + cs < tot ? o0 + cs : tot;
        if (o0 < o1) {
          int lo = 0, hi = nlev - 1;  // node: last level entry with loff <= o0
          while (lo < hi) {
            int md = (lo + hi + 1) >> 1;
            if (loff[md] <= o0) lo = md; else hi = md - 1;
          }
          for (int k = lo; o0 < o1; ++k) {
            int x = lst[k];
            int a0 = ns[x], mm = nm[x], e0 = ne[x];
            int na = mm - a0, nb = e0 - mm, size = e0 - a0;
            int o = o0 - loff[k];
            int cnt = size - o < o1 - o0 ? size - o : o1 - o0;
            int ai = smem_merge_path(Xs + a0, na, Xs + mm, nb, o);
            int bi = o - ai;
            for (int q = 0; q < cnt; ++q) {
              bool takeA = (bi >= nb) || (ai < na && Xs[a0 + ai] <= Xs[mm + bi]);
              int si = takeA ? a0 + ai : mm + bi;
              Xd[a0 + o + q] = Xs[si];
              if (HAS_TAGS) Yd[a0 + o + q] = Ys[si];
              ai += takeA;
              bi += !takeA;
            }
            if (E.classic && o == 0) {
              K maxL = Xs[mm - 1], maxR = Xs[e0 - 1];
              int rl = smem_count(Xs + mm, nb, maxL, false);
              int lr = smem_count(Xs + a0, na, maxR, true);
              int pl = na - 1 + rl, pr = nb - 1 + lr;
              comps += (unsigned long long)((pl < pr ? pl : pr) + 1);
            }
            o0 += cnt;
          }
        }
        __syncthreads();
      }
    }
#ifdef RS_INSTR
    ti3 = clock64();
    if (threadIdx.x == 0) {  // sub-phases of the slowest fused task: tables+span, leaves, levels (cycles)
      unsigned long long tot = (unsigned long long)(ti3 - ti0);
      if (tot > E.met->peek[0]) {
        E.met->peek[0] = tot;
        E.met->peek[1] = (unsigned long long)(ti1 - ti0);
        E.met->peek[2] = (unsigned long long)(ti2 - ti1);
        E.met->peek[3] = (unsigned long long)(ti3 - ti2);
        E.met->peek[4] = (unsigned long long)(s_dmax - droot + 1);
      }
    }
#endif
    hook();  // result in X[droot & 1]; the other buffer is free
    K* gd = reinterpret_cast<K*>(E.key[item_buf(droot)]);  // in place unless depth 1
    T* hd = HAS_TAGS ? reinterpret_cast<T*>(E.tag[item_buf(droot)]) : nullptr;
    const K* Xr = X[droot & 1];
    const T* Yr = Y[droot & 1];
    for (int x = threadIdx.x; x < len; x += blockDim.x) {
      gd[s + x] = Xr[x];
      if (HAS_TAGS) hd[s + x] = Yr[x];
    }
    return ib ^ (droot & 1);
  }
};

// Phase A: fused subtrees and big-leaf tiles (no dependencies among them).
// Thread 0 claims the next task and fetches its record and span while the
// current one runs; a fused next task's span is bulk-copied into the span
// buffer the current task has finished with, overlapping its write-back.
template <typename K, int TB>
__global__ void __launch_bounds__(kExecThreads, 3) k_phaseA(ExecArgs E) {
  using X = Exec<K, TB>;
  using Span = typename X::Span;
  extern __shared__ __align__(16) unsigned char smem[];
  __shared__ unsigned long long sred[32];
  __shared__ __align__(8) uint64_t s_bar;
  __shared__ uint64_t s_rec;       // record of the task to run next (kind 3: none)
  __shared__ int32_t s_off[2];     // its span's offsets in buffer s_ib, if issued
  __shared__ int s_ib, s_issued;
  pdl_wait();  // the prep's outputs are complete and visible
  const unsigned long long ntasks = E.met->phaseA;
  constexpr uint64_t kNone = ~0ull;
  // thread 0's view of the next task
  uint64_t nrec = kNone;
  unsigned long long nt = 0;
  Span nf{};
  // the claim is a chain of dependent round trips; stage() advances it one
  // step so thread 0 never waits on it in the middle of a task
  int nst = 0;
  auto stage = [&]() {
    if (nst == 0) nt = atomicAdd(&E.met->task_ctr_A, 1ull);
    else if (nst == 1) nrec = nt < ntasks ? E.tasks[nt] : kNone;
    else if (nst == 2 && nrec != kNone && task_kind(nrec) == kTaskFuse) nf = X::span_of(E, task_id(nrec));
    if (nst < 3) ++nst;
  };
  auto claim = [&]() {
    nst = 0;
    while (nst < 3) stage();
  };
  if (threadIdx.x == 0) {
    mbar_init(&s_bar, 1);
    mbar_fence_init();
    claim();
    s_rec = nrec;
    s_ib = 0;
    s_issued = 0;
    if (nrec != kNone && task_kind(nrec) == kTaskFuse) {
      X::span_issue(E, nf, smem, 0, &s_bar, s_off);
      s_issued = 1;
    }
  }
  __syncthreads();
  uint32_t fphase = 0;
  unsigned long long comps = 0;
  for (;;) {
    uint64_t rec = s_rec;
    int ib = s_ib;
    int issued = s_issued;
    if (rec == kNone) {
      pdl_trigger();  // no more tasks for this CTA: k_merge_exec may start launching
      break;
    }
    uint32_t kind = task_kind(rec), id = task_id(rec), tile = task_tile(rec);
#ifdef RS_INSTR
    const long long t_task0 = clock64();
#endif
    __syncthreads();  // everyone has read the shared slots
    if (threadIdx.x == 0) {
      nst = 0;
      stage();  // claim issued; record and span follow during the task
    }
    // thread 0 publishes the next task; a fused one is issued into buffer `fb`
    auto publish = [&](int fb) {
      if (threadIdx.x == 0) {
        while (nst < 3) stage();
        s_rec = nrec;
        s_ib = fb;
        s_issued = 0;
        if (nrec != kNone && task_kind(nrec) == kTaskFuse) {
          X::span_issue(E, nf, smem, fb, &s_bar, s_off);
          s_issued = 1;
        }
      }
    };
    if (kind == kTaskLeaf) {
      X::leaf_task(E, id - E.leaf_base, tile);
      publish(ib);  // no buffer in use
    } else {
      Span f = X::span_of(E, id);
      if (!issued) {  // (never: a fused task is always issued when published)
        if (threadIdx.x == 0) X::span_issue(E, f, smem, ib, &s_bar, s_off);
        __syncthreads();
      }
      X::fuse_task(E, f, ib, smem, &s_bar, fphase, s_off, stage,
                   [&]() { publish(ib ^ (f.droot & 1) ^ 1); }, comps);
    }
    __syncthreads();
    if (threadIdx.x == 0) release_add_u32(E.done + id, 1u);
#ifdef RS_INSTR
    if (threadIdx.x == 0) {  // phase-A task durations: max, sum, count, and the max task's size
      unsigned long long dur = (unsigned long long)(clock64() - t_task0);
      atomicMax(&E.met->prep_dbg[25], dur);
      atomicAdd(&E.met->prep_dbg[26], dur);
      atomicAdd(&E.met->prep_dbg[27], 1ull);
      if (kind != kTaskLeaf) {
        Span f = X::span_of(E, id);
        atomicMax(&E.met->prep_dbg[28], (dur << 24) | (unsigned long long)(f.e - f.s));
        atomicMax(&E.met->prep_dbg[29], (dur << 24) | (unsigned long long)(f.lb - f.la));
      }
      atomicMax(&E.met->prep_dbg[30], (dur << 24) | (unsigned long long)kind);
      atomicMax(&E.met->prep_dbg[31], (unsigned long long)clock64());  // latest end (SM clock, rough)
    }
#endif
  }
  unsigned long long sum = block_sum(comps, sred);
  if (threadIdx.x == 0 && sum) atomicAdd(&E.met->comparisons, sum);
}

}  // namespace rs
