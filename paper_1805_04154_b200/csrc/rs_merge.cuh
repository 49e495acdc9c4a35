// rs_merge.cuh -- warp-specialized TMA merge executor for the large tree nodes.
//
// Reference: runcore.py:251-279 (_stable_merge: stable two-run merge, ties go
// to the left run), runcore.py:282-326 (merge_cost / comparison accounting),
// sorters.py:478-516 (every internal node of the power tree is one merge).
//
// Each CTA = 1 producer warp + 8 consumer warps, with an S-stage shared-memory
// ring guarded by mbarriers:
//   producer  claims a "super task" (up to kSuper consecutive output tiles of
//             one node), waits until both children are complete (per-node
//             counters, acquire loads), finds the merge-path split of every
//             tile boundary with lane-group parallel searches in HBM, then for
//             each tile issues 1D TMA bulk copies (cp.async.bulk) of its A and
//             B input windows into a free stage, completing on the stage's
//             full barrier.
//   consumers merge the stage (per-thread merge path in SMEM, IPT outputs per
//             thread held in registers), write the result back into the stage
//             and stream it to HBM with coalesced stores, publish the tile on
//             the node's counter, and release the stage.
// Task order is deepest-first, so every wait is on an earlier task and the
// persistent grid (all CTAs resident) cannot deadlock.
#pragma once
#include "rs_common.cuh"
#include "rs_exec.cuh"

namespace rs {

#ifndef RS_MDESC
#define RS_MDESC 1
#endif
constexpr int kSuperMax = 15;          // tiles per merge task: runtime, <= 15 (lane groups of >= 2)
#ifndef RS_STAGES
#define RS_STAGES 2
#endif
#ifndef RS_IPT8
#define RS_IPT8 15
#endif
#ifndef RS_IPT4
#define RS_IPT4 31
#endif
#ifndef RS_MERGE_CTAS
#define RS_MERGE_CTAS 3
#endif
constexpr int kStages = RS_STAGES;     // smem ring depth
#ifndef RS_CONSUMER_WARPS
#define RS_CONSUMER_WARPS 8
#endif
constexpr int kConsumerThreads = 32 * RS_CONSUMER_WARPS;  // consumer warps
#ifndef RS_PRODUCERS
#define RS_PRODUCERS 1
#endif
constexpr int kProducers = RS_PRODUCERS;  // 1: one producer feeds both stages; 2: one stage each
// RS_FETCHER: a fetcher warp claims the next task, loads its descriptor and
// acquires its children's counters while the producer searches and issues
// the current one (a one-slot shared-memory ticket queue between them).
#ifndef RS_FETCHER
#define RS_FETCHER 0
#endif
constexpr int kFetchers = RS_FETCHER ? 1 : 0;
constexpr int kRoleWarps = kProducers + 1 + kFetchers;  // producers, signaller, fetcher
constexpr int kMergeThreads = kConsumerThreads + 32 * kRoleWarps;

template <typename K, int TB>
struct MergeCfg {
  static constexpr int kb = sizeof(K);
  static constexpr int eb = kb + TB;
  static constexpr int IPT = eb == 4 ? RS_IPT4 : (eb <= 8 ? RS_IPT8 : (eb <= 12 ? 11 : 7));  // odd: conflict-free write-back
  static constexpr int TILE = kConsumerThreads * IPT;
  static constexpr int KBYTES = TILE * kb + 128;
  static constexpr int TBYTES = TB ? TILE * TB + 128 : 0;
  static constexpr int STAGE = KBYTES + TBYTES;
  static constexpr size_t SMEM = (size_t)kStages * STAGE + 1024;
};

struct StageHdr {
  pos_t dst;     // first output element index
  int32_t len;   // outputs in this tile
  int32_t la;    // A elements
  int32_t offA;  // element offsets inside the stage's key region
  int32_t offB;
  int32_t toffA; // element offsets inside the stage's tag region
  int32_t toffB;
  uint32_t node;
  int32_t parity;  // destination buffer
  int32_t end;
  int32_t pad;
#ifdef RS_DEBUG_CHECKS
  const void* dbg_srcB;  // global address of the B window's first element
  uint32_t dbg_cB;       // right child id
  uint32_t dbg_dnB;      // its counter when the producer found it ready
#endif
};

__device__ __forceinline__ void consumer_sync() { asm volatile("bar.sync 1, %0;" ::"r"(kConsumerThreads) : "memory"); }

struct MergeArgs {
  void* key[3];
  void* tag[3];
  int classic;
  int msuper;  // merge tiles per task (ClassifyArgs::msuper)
  const pos_t* leaf_start;
  const uint8_t* depth;
  const pos_t* node_s;
  const pos_t* node_e;
  const uint32_t* child;
  const uint32_t* need;
  uint32_t* done;
  const uint64_t* tasks;
  const MDesc* mdesc;  // per merge task (RS_MDESC), index = task - first merge task
  long long mdesc_cap;
  DevMetrics* met;
  const uint8_t* cls;  // unified id -> class (2 = merge node for internal ids)
  uint32_t leaf_base;
  int skipchk;  // top-down / bottom-up: one comparison per node, in-order merges skipped (sorters.py:545-550,575-578)
};

// Lane-group merge-path search: lanes [g*G, g*G+G) cooperate on diagonal `diag`
// of group g.  Returns the split (number of A elements) in every lane.  `side`
// runs once per round trip, between issuing the step's loads and consuming
// them, so another dependent load chain can overlap the search's latency.
template <typename K>
__device__ __forceinline__ K ld_volatile_k(const K* p) { return *reinterpret_cast<const volatile K*>(p); }
struct NoSide {
  __device__ __forceinline__ void operator()() const {}
};
template <typename K, typename Side = NoSide>
__device__ __forceinline__ int64_t group_merge_path(const K* A, int64_t na, const K* B, int64_t nb, int64_t diag,
                                                    bool active, int G, Side&& side = Side()) {
  // Each lane probes kProbe positions per round trip: a group of G lanes cuts
  // the interval (G * kProbe + 1) ways.  The predicate A[i] <= B[diag-1-i] is
  // monotone in i, so the number of true probes locates the split.
#ifndef RS_PROBE
#define RS_PROBE 2
#endif
  constexpr int kProbe = RS_PROBE;
  int lane = threadIdx.x & 31;
  int g = lane / G, gl = lane % G;
  const int GP = G * kProbe;
  const uint32_t gmask = (G == 32 ? 0xffffffffu : ((1u << G) - 1u)) << (g * G);
  int64_t lo = 0, hi = 0;
  if (active) {
    lo = diag - nb > 0 ? diag - nb : 0;
    hi = diag < na ? diag : na;
  }
  for (;;) {
    bool need = active && (hi - lo > GP);
    if (!__any_sync(0xffffffffu, need)) break;
    // probes at lo + k*step, k = 1..GP (step >= 1 since span > GP): one division
    int64_t step = (hi - lo) / (GP + 1);
    K xa[kProbe], xb[kProbe];
#pragma unroll
    for (int q = 0; q < kProbe; ++q) {
      xa[q] = K(0);
      xb[q] = K(0);
      if (need) {
        int64_t idx = lo + step * (gl * kProbe + q + 1);
        xa[q] = ldcg(A + idx);
        xb[q] = ldcg(B + (diag - 1 - idx));
      }
    }
    side();
    int c = 0;
#pragma unroll
    for (int q = 0; q < kProbe; ++q) c += __popc(__ballot_sync(0xffffffffu, need && xa[q] <= xb[q]) & gmask);
    if (need) {
      int64_t nlo = c > 0 ? lo + step * c + 1 : lo;
      int64_t nhi = c < GP ? lo + step * (c + 1) : hi;
      lo = nlo;
      hi = nhi;
    }
  }
  K xa[kProbe], xb[kProbe];
  bool fin[kProbe];
#pragma unroll
  for (int q = 0; q < kProbe; ++q) {
    int64_t idx = lo + gl * kProbe + q;
    fin[q] = active && idx < hi;
    xa[q] = K(0);
    xb[q] = K(0);
    if (fin[q]) {
      xa[q] = ldcg(A + idx);
      xb[q] = ldcg(B + (diag - 1 - idx));
    }
  }
  side();
  int c = 0;
#pragma unroll
  for (int q = 0; q < kProbe; ++q) c += __popc(__ballot_sync(0xffffffffu, fin[q] && xa[q] <= xb[q]) & gmask);
  return lo + c;
}

// The producer's view of one claimed merge task, fetched in dependent stages
// (claim -> record -> node + children -> children's tile counts) so the chain
// can be advanced one round trip at a time while other work is in flight.
struct PTask {
  unsigned long long t;
  uint32_t j, sk, c0, c1, nd0, nd1, dn0, dn1;
  uint8_t cl0, cl1;  // class of internal children (2 = merge node), 0 for leaves
  pos_t s, e, m;
  int d;
  int st;  // stages done: 1 claimed, 2 record, 3 node, 4 need, 5 counters (speculative)
  unsigned long long tbase;  // first merge task: descriptor index = t - tbase
  bool valid;
  __device__ __forceinline__ void claim(DevMetrics* met) {
    t = 0;
    if ((threadIdx.x & 31) == 0) t = atomicAdd(&met->task_ctr, 1ull);
    st = 1;
  }
  // static round robin: this producer's next task index (no atomic, so the
  // whole fetch chain can run ahead of time)
  __device__ __forceinline__ void claim_static(unsigned long long& snext, unsigned long long stride) {
    t = snext;
    snext += stride;
    st = 1;
  }
  template <typename Args>
  __device__ __forceinline__ void advance(const Args& E, unsigned long long ntasks) {
    if (st == 1) {
      t = __shfl_sync(0xffffffffu, t, 0);
      valid = t < ntasks;
#if RS_MDESC
      // one 48-byte descriptor instead of the record -> node -> children chain
      // (tasks beyond the descriptor array's bound take the chain below)
      if (valid && (long long)(t - tbase) >= E.mdesc_cap) {
        uint64_t rec = E.tasks[t];
        j = task_id(rec);
        sk = task_tile(rec);
        st = 2;
        return;
      }
      if (valid) {
        const MDesc md = E.mdesc[t - tbase];
        j = md.j;
        sk = md.sk;
        s = md.s_d & kMdescPosMask;
        d = (int)(md.s_d >> 56);
        m = md.m_cl & kMdescPosMask;
        e = md.e;
        c0 = md.c0;
        c1 = md.c1;
        nd0 = md.nd0;
        nd1 = md.nd1;
        cl0 = ((md.m_cl >> 56) & 1) ? 2 : 0;
        cl1 = ((md.m_cl >> 57) & 1) ? 2 : 0;
      }
      st = 3;  // next: the children's counters
#else
      uint64_t rec = valid ? E.tasks[t] : 0ull;
      j = task_id(rec);
      sk = task_tile(rec);
#endif
    } else if (st == 2) {
      if (valid) {
        c0 = E.child[2 * j];
        c1 = E.child[2 * j + 1];
        s = E.node_s[j];
        e = E.node_e[j];
        m = E.leaf_start[j];
        d = E.depth[j];
      }
    } else if (st == 3) {
      if (valid) {
        nd0 = E.need[c0];
        nd1 = E.need[c1];
        cl0 = c0 < E.leaf_base ? E.cls[c0] : 0;
        cl1 = c1 < E.leaf_base ? E.cls[c1] : 0;
      }
    } else if (st == 4) {
      // early acquire of the children's counters (overlapping the search's
      // loads): if they already read complete, ready() costs nothing
      dn0 = valid && nd0 ? ld_acquire_u32(E.done + c0) : 0u;
      dn1 = valid && nd1 ? ld_acquire_u32(E.done + c1) : 0u;
    }
    if (st < 5) ++st;
  }
  template <typename Args>
  __device__ __forceinline__ void finish(const Args& E, unsigned long long ntasks) {
    while (st < 5) advance(E, ntasks);
  }
  // Children complete (with acquire semantics)?
  __device__ __forceinline__ bool ready(const uint32_t* done) {
    if (dn0 >= nd0 && dn1 >= nd1) return true;
    dn0 = nd0 ? ld_acquire_u32(done + c0) : 0u;
    dn1 = nd1 ? ld_acquire_u32(done + c1) : 0u;
    return dn0 >= nd0 && dn1 >= nd1;
  }
};

template <typename K>
__device__ int64_t warp_count(const K* A, int64_t len, K v, bool or_equal) {
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

// AHEAD: claim the next task during the current one's search (chosen at launch:
// multi-tile tasks only, see the producer).
template <typename K, int TB, bool AHEAD>
__global__ void __launch_bounds__(kMergeThreads, RS_MERGE_CTAS) k_merge_exec(MergeArgs E) {
  using C = MergeCfg<K, TB>;
  using T = typename TagT<TB>::type;
  constexpr bool HT = TB != 0;
  extern __shared__ __align__(128) unsigned char smem_m[];
  unsigned char* smem = smem_m;
  __shared__ __align__(8) uint64_t full_bar[kStages];
  __shared__ __align__(8) uint64_t empty_bar[kStages];
  __shared__ __align__(8) uint64_t stored_bar[kStages];
  __shared__ StageHdr hdr[kStages];
  __shared__ __align__(8) uint64_t tk_full, tk_empty;  // fetcher -> producer ticket slot
  __shared__ PTask tk_box;

  int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (threadIdx.x == 0) {
    for (int s = 0; s < kStages; ++s) {
      mbar_init(&full_bar[s], 1);
      mbar_init(&empty_bar[s], 1);
      mbar_init(&stored_bar[s], kConsumerThreads / 32);
    }
    mbar_init(&tk_full, 1);
    mbar_init(&tk_empty, 1);
    mbar_fence_init();
  }
  __syncthreads();
  pdl_wait();  // phase A (and the prep before it) complete and visible
  unsigned long long ntasks = E.met->n_tasks;
  // first merge task (after the phase-A tasks); not task_ctr, which other CTAs may already have advanced
  const unsigned long long t_first = E.met->phaseA;

  if (kFetchers && warp == kProducers + 1) {
    // -------------------------------------------------------------- fetcher
    // Claims tasks in order and hands each, descriptor loaded and children's
    // counters acquired, to the producer through the one-slot ticket: the
    // claim -> descriptor -> counters chain of task t+1 runs while the
    // producer searches and issues task t.  Tasks still wait only on tasks
    // claimed before them, and the CTA finishes its tasks in claim order, so
    // the resident grid cannot deadlock.
    uint32_t ph = 0;
    for (;;) {
      PTask p;
      p.tbase = t_first;
      p.claim(E.met);
      p.finish(E, ntasks);
      if (lane == 0) {
        mbar_wait(&tk_empty, ph ^ 1);
        tk_box = p;
        mbar_arrive(&tk_full);
      }
      ph ^= 1;
      __syncwarp();
      if (!p.valid) break;
    }
    return;
  }

  if (warp < kProducers) {
    // ------------------------------------------------------------- producer
    unsigned long long comps = 0, mcost = 0;
    int stage = kProducers == 1 ? 0 : warp;
    uint32_t phase = 0;  // flips when stage wraps (kProducers 2: every tile of its stage)
    const int kSuper = E.msuper;
    const int G = 32 / (kSuper + 1);
    // The next task may be claimed and its descriptor fetched while the
    // current task's merge-path search runs (each is a chain of dependent global
    // round trips; interleaving hides one behind the other).  Claiming one task
    // ahead cannot deadlock: the current task is ready, so it completes, and
    // every task waits only on tasks claimed before it.
    // Multi-tile tasks (long searches) claim the next task ahead and hide its
    // fetch chain in the search; single-tile tasks claim just in time -- a task
    // held ahead adds to the waits at level transitions (measured: cfg1-3 6-13%
    // faster just in time, cfg4 (7 tiles/task) 2% faster ahead).  A compile-time
    // choice: a runtime flag costs the just-in-time path its gain.
#ifndef RS_STATIC
#define RS_STATIC 0
#endif
    // RS_STATIC: task t goes to producer t mod (grid producers); every wait is
    // still on a smaller task index, so the resident grid cannot deadlock, and
    // with no claim atomic the next task's fetch chain runs during the search.
    constexpr bool kStatic = RS_STATIC != 0;
    constexpr bool ahead = AHEAD || kStatic;
    const unsigned long long sstride = (unsigned long long)gridDim.x * kProducers;
    unsigned long long snext = t_first + (unsigned long long)blockIdx.x * kProducers + (unsigned long long)warp;
    PTask cur, nxt;
    cur.tbase = nxt.tbase = t_first;
    uint32_t tph = 0;
    auto pop = [&](PTask& x) {  // the fetcher's next ticket
      if (lane == 0) mbar_wait(&tk_full, tph);
      __syncwarp();
      x = tk_box;
      __syncwarp();
      if (lane == 0) mbar_arrive(&tk_empty);
      tph ^= 1;
      // the fetcher's acquire of the children's counters, made this warp's
      // (the ticket's mbarrier hand-off orders it; the fence extends it GPU-wide)
      fence_acquire_gpu();
    };
    if (kFetchers) pop(cur);
    else {
      if (kStatic) cur.claim_static(snext, sstride);
      else cur.claim(E.met);
      cur.finish(E, ntasks);
    }
    while (cur.valid) {
      RS_T0(tw);
      if (!cur.ready(E.done)) {
        unsigned ns = 32;
        do {
          __nanosleep(ns);
          if (ns < 256) ns <<= 1;
        } while (!cur.ready(E.done));
      }
      if (lane == 0) RS_ACC(E.met, 5, tw);
      if (ahead && !kFetchers) {
        if (kStatic) nxt.claim_static(snext, sstride);
        else nxt.claim(E.met);
      }
      const uint32_t j = cur.j, sk = cur.sk;
      const pos_t s = cur.s, e = cur.e, m = cur.m;
      const int d = cur.d;
      if (lane == 0) {
        RS_T0(tf);
        fence_proxy_async_global();  // acquired generic-proxy data -> TMA reads
        RS_ACC(E.met, 6, tf);
#ifdef RS_INSTR
        atomicAdd(&E.met->depth_wait[d], (unsigned long long)(clock64() - tw));
#endif
        RS_ACC(E.met, 0, tw);
      }
      __syncwarp();
      RS_T0(tsrch);
      // children: merge nodes in buf[node_buf(d + 1)], phase-A items in buf[item_buf(d + 1)]
      const int ba = cur.cl0 == 2 ? node_buf(d + 1) : item_buf(d + 1);
      const int bb = cur.cl1 == 2 ? node_buf(d + 1) : item_buf(d + 1);
      const K* srcA = reinterpret_cast<const K*>(E.key[ba]);
      const K* srcB = reinterpret_cast<const K*>(E.key[bb]);
      const T* tsrcA = HT ? reinterpret_cast<const T*>(E.tag[ba]) : nullptr;
      const T* tsrcB = HT ? reinterpret_cast<const T*>(E.tag[bb]) : nullptr;
      int64_t tot = e - s, na = m - s, nb = e - m;
      int64_t ntile = (tot + C::TILE - 1) / C::TILE;
      int64_t kbeg = (int64_t)sk * kSuper;
      int64_t kend = kbeg + kSuper < ntile ? kbeg + kSuper : ntile;
      int g = lane / G;
      int64_t diag = (kbeg + g) * (int64_t)C::TILE;
      if (diag > tot) diag = tot;
      bool in_range = g <= (kend - kbeg) && g < kSuper + 1 && lane < G * (kSuper + 1);
      bool trivial = diag == 0 || diag == tot;
      int64_t split = group_merge_path(srcA + s, na, srcB + m, nb, diag, in_range && !trivial, G,
                                       [&]() {
                                         if (ahead && !kFetchers) nxt.advance(E, ntasks);
                                       });
      if (ahead && !kFetchers) nxt.finish(E, ntasks);
      if (diag == 0) split = 0;
      else if (diag == tot) split = na;
      if (lane == 0) RS_ACC(E.met, 1, tsrch);
      RS_T0(tiss);
#ifndef RS_CLAIM_EARLY
#define RS_CLAIM_EARLY 0  // 1: measured 1-2 us slower (a task claimed during the issue is held)
#endif
      // just in time, but the claim's atomic round trip overlaps this task's issue
      if (!ahead && !kFetchers && RS_CLAIM_EARLY) nxt.claim(E.met);
      bool merged = true;  // the reference performs this merge (Metrics)
      if (E.skipchk && kbeg == 0) {
        // sorters.py:545-550 / 575-578: one comparison; an in-order pair is not
        // merged (the stable merge below then equals the concatenation)
        K lastL = ldcg(srcA + m - 1), firstR = ldcg(srcB + m);
        merged = !(lastL <= firstR);
        if (lane == 0) {
          comps += 1;
          if (merged) {
            mcost += (unsigned long long)tot;
            if (!E.classic) comps += (unsigned long long)tot;  // runcore.py:299-301
          }
        }
      }
      if (E.classic && kbeg == 0 && merged) {
        // runcore.py:321-324
        K maxL = ldcg(srcA + m - 1), maxR = ldcg(srcB + e - 1);
        int64_t rl = warp_count(srcB + m, nb, maxL, false);
        int64_t lr = warp_count(srcA + s, na, maxR, true);
        int64_t pl = na - 1 + rl, pr = nb - 1 + lr;
        if (lane == 0) comps += (unsigned long long)((pl < pr ? pl : pr) + 1);
      }
      for (int64_t k = kbeg; k < kend; ++k) {
        int gi = int(k - kbeg);
        int64_t i0 = __shfl_sync(0xffffffffu, split, gi * G);
        int64_t i1 = __shfl_sync(0xffffffffu, split, (gi + 1) * G);
        if (lane == 0) {
          RS_T0(te);
          mbar_wait(&empty_bar[stage], phase ^ 1);
          RS_ACC(E.met, 2, te);
          int64_t o0 = k * (int64_t)C::TILE;
          int64_t o1 = o0 + C::TILE < tot ? o0 + C::TILE : tot;
          int64_t j0 = o0 - i0, j1 = o1 - i1;
          RS_CHECK(0 <= i0 && i0 <= i1 && i1 <= na && 0 <= j0 && j0 <= j1 && j1 <= nb && o1 - o0 <= C::TILE,
                   "node %u k %lld s %lld m %lld e %lld i0 %lld i1 %lld j0 %lld j1 %lld", j, (long long)k,
                   (long long)s, (long long)m, (long long)e, (long long)i0, (long long)i1, (long long)j0,
                   (long long)j1);
          RS_CHECK(j < E.leaf_base && s < m && m < e, "bad node %u s %lld m %lld e %lld", j, (long long)s,
                   (long long)m, (long long)e);
          unsigned char* sk_base = smem + (size_t)stage * C::STAGE;
          StageHdr& h = hdr[stage];
          h.dst = s + o0;
          h.len = int32_t(o1 - o0);
          h.la = int32_t(i1 - i0);
          h.node = j;
          h.parity = node_buf(d);  // destination buffer index
#ifdef RS_DEBUG_CHECKS
          h.dbg_srcB = srcB + m + j0;
          h.dbg_cB = cur.c1;
          h.dbg_dnB = cur.dn1;
#endif
          h.end = 0;
          // expected bytes first (tx count may complete before arrive otherwise)
          uintptr_t ka0 = reinterpret_cast<uintptr_t>(srcA + s + i0), ka1 = reinterpret_cast<uintptr_t>(srcA + s + i1);
          uintptr_t kb0 = reinterpret_cast<uintptr_t>(srcB + m + j0), kb1 = reinterpret_cast<uintptr_t>(srcB + m + j1);
          uint32_t bA = i1 > i0 ? (uint32_t)(((ka1 + 15) & ~(uintptr_t)15) - (ka0 & ~(uintptr_t)15)) : 0u;
          uint32_t bB = j1 > j0 ? (uint32_t)(((kb1 + 15) & ~(uintptr_t)15) - (kb0 & ~(uintptr_t)15)) : 0u;
          uint32_t tx = bA + bB;
          uint32_t tA = 0, tBb = 0;
          if (HT) {
            uintptr_t ta0 = reinterpret_cast<uintptr_t>(tsrcA + s + i0), ta1 = reinterpret_cast<uintptr_t>(tsrcA + s + i1);
            uintptr_t tb0 = reinterpret_cast<uintptr_t>(tsrcB + m + j0), tb1 = reinterpret_cast<uintptr_t>(tsrcB + m + j1);
            tA = i1 > i0 ? (uint32_t)(((ta1 + 15) & ~(uintptr_t)15) - (ta0 & ~(uintptr_t)15)) : 0u;
            tBb = j1 > j0 ? (uint32_t)(((tb1 + 15) & ~(uintptr_t)15) - (tb0 & ~(uintptr_t)15)) : 0u;
            tx += tA + tBb;
          }
#ifdef RS_DEBUG_CHECKS
          // poison the head of the stage so a copy that never landed is recognizable
          {
            K* pk = reinterpret_cast<K*>(sk_base);
            for (int q = 0; q < 96; ++q) pk[q] = (K)0x7eadbeef;
            fence_proxy_async_smem();
          }
#endif
          // the whole header (window offsets included) is written BEFORE the
          // arrival: the phase can complete as soon as the bytes land, and the
          // arrival's release is what makes these writes visible to consumers
          h.offA = i1 > i0 ? int32_t((ka0 & 15) / sizeof(K)) : 0;
          h.offB = (j1 > j0 ? int32_t((kb0 & 15) / sizeof(K)) : 0) + int32_t(bA / sizeof(K));
          if (HT) {
            uintptr_t ta0 = reinterpret_cast<uintptr_t>(tsrcA + s + i0);
            uintptr_t tb0 = reinterpret_cast<uintptr_t>(tsrcB + m + j0);
            h.toffA = i1 > i0 ? int32_t((ta0 & 15) / (TB ? TB : 1)) : 0;
            h.toffB = (j1 > j0 ? int32_t((tb0 & 15) / (TB ? TB : 1)) : 0) + int32_t(tA / (TB ? TB : 1));
          }
          mbar_arrive_tx(&full_bar[stage], tx);
          int32_t o_;
          tma_window(sk_base, srcA, s + i0, s + i1, sizeof(K), &full_bar[stage], &o_);
          tma_window(sk_base + bA, srcB, m + j0, m + j1, sizeof(K), &full_bar[stage], &o_);
          if (HT) {
            unsigned char* tg = sk_base + C::KBYTES;
            tma_window(tg, tsrcA, s + i0, s + i1, TB, &full_bar[stage], &o_);
            tma_window(tg + tA, tsrcB, m + j0, m + j1, TB, &full_bar[stage], &o_);
          }
        }
        __syncwarp();
        if (kProducers == 1) {
          if (++stage == kStages) { stage = 0; phase ^= 1; }
        } else {
          phase ^= 1;
        }
      }
      if (lane == 0) RS_ACC(E.met, 7, tiss);
      if (kFetchers) pop(nxt);
      else if (!ahead) {  // just in time: no task held ahead
        if (!RS_CLAIM_EARLY) nxt.claim(E.met);
        nxt.finish(E, ntasks);
      }
      cur = nxt;
    }
    if (lane == 0) {
      mbar_wait(&empty_bar[stage], phase ^ 1);
      hdr[stage].end = 1;
      mbar_arrive(&full_bar[stage]);
      if (comps) atomicAdd(&E.met->comparisons, comps);
      if (mcost) atomicAdd(&E.met->merge_cost, mcost);
    }
    return;
  }

  if (warp == kProducers) {
    // ------------------------------------------------------------ signaller
    // Streams each merged tile from its stage to HBM (bulk store of the 16B-
    // aligned middle, lanes store the unaligned head / tail), hands the stage
    // back once the copy engine has read it, and publishes the tile (counter
    // add) after the writes are complete and fenced -- the consumers never
    // wait on global stores.
    constexpr int VK = 16 / sizeof(K);
    constexpr int VT = HT ? 16 / (HT ? TB : 1) : 1;
    int stage = 0;
    uint32_t phase = 0;
    uint32_t sph[kStages];
    bool alive[kStages];
#pragma unroll
    for (int q = 0; q < kStages; ++q) { sph[q] = 0; alive[q] = true; }
    int nalive = kStages;
    for (;;) {
      if (kProducers == 1) {
        mbar_wait(&stored_bar[stage], phase);
      } else {  // the stage the consumers finished (any order)
        if (nalive == 0) break;
        stage = -1;
        while (stage < 0) {
#pragma unroll
          for (int q = 0; q < kStages; ++q)
            if (stage < 0 && alive[q] && mbar_test_wait(&stored_bar[q], sph[q])) stage = q;
        }
        sph[stage] ^= 1;
      }
      const StageHdr h = hdr[stage];
      if (h.end) {
        if (kProducers == 1) break;
        alive[stage] = false;
        --nalive;
        continue;
      }
      unsigned char* base = smem + (size_t)stage * C::STAGE;
      K* sk = reinterpret_cast<K*>(base);
      T* st = reinterpret_cast<T*>(base + C::KBYTES);
      const int len = h.len;
      K* gdst = reinterpret_cast<K*>(E.key[h.parity]) + h.dst;
      const int pad = int((reinterpret_cast<uintptr_t>(gdst) & 15) / sizeof(K));
      int h0 = (VK - pad) % VK;
      if (h0 > len) h0 = len;
      const int nvec = (len - h0) / VK;
      const int tail0 = h0 + nvec * VK;
      if (lane < h0) gdst[lane] = sk[pad + lane];
      if (lane < len - tail0) gdst[tail0 + lane] = sk[pad + tail0 + lane];
      T* tdst = nullptr;
      int th0 = 0, tnvec = 0, ttail0 = 0, tpad = 0;
      if (HT) {
        tdst = reinterpret_cast<T*>(E.tag[h.parity]) + h.dst;
        tpad = int((reinterpret_cast<uintptr_t>(tdst) & 15) / (HT ? TB : 1));
        th0 = (VT - tpad) % VT;
        if (th0 > len) th0 = len;
        tnvec = (len - th0) / VT;
        ttail0 = th0 + tnvec * VT;
        if (lane < th0) tdst[lane] = st[tpad + lane];
        if (lane < len - ttail0) tdst[ttail0 + lane] = st[tpad + ttail0 + lane];
      }
      __syncwarp();
      if (lane == 0) {
        if (nvec > 0) tma_store_1d(gdst + h0, sk + pad + h0, (uint32_t)nvec * 16u);
        if (HT && tnvec > 0) tma_store_1d(tdst + th0, st + tpad + th0, (uint32_t)tnvec * 16u);
        bulk_commit();
        bulk_wait_read0();
        mbar_arrive(&empty_bar[stage]);  // the stage may be refilled
        bulk_wait0();                    // the tile's bulk writes are performed
#ifdef RS_DEBUG_CHECKS
        for (int i = 0; i + 1 < len; ++i) {
          K x0 = ld_volatile_k(gdst + i), x1 = ld_volatile_k(gdst + i + 1);
          if (!(x0 <= x1)) {
            printf("tile unsorted in global after store: node %u dst %lld i %d len %d h0 %d nvec %d pad %d smem %lld %lld glob %lld %lld\n",
                   h.node, (long long)h.dst, i, len, h0, nvec, pad, (long long)sk[pad + i], (long long)sk[pad + i + 1],
                   (long long)x0, (long long)x1);
            __trap();
          }
        }
#endif
        fence_proxy_async_global();      // async-proxy writes -> generic / other proxies
      }
      __syncwarp();
      __threadfence();  // this warp's head / tail stores and the bulk writes, GPU-wide
      if (lane == 0) asm volatile("red.relaxed.gpu.global.add.u32 [%0], 1;" ::"l"(E.done + h.node) : "memory");
      __syncwarp();
      if (kProducers == 1 && ++stage == kStages) { stage = 0; phase ^= 1; }
    }
    return;
  }

  // --------------------------------------------------------------- consumers
  int ct = threadIdx.x - 32 * kRoleWarps;
  int cl = ct & 31;
  int stage = 0;
  uint32_t phase = 0;
  __shared__ int s_pick;
  uint32_t cph[kStages];
  bool alive[kStages];
#pragma unroll
  for (int q = 0; q < kStages; ++q) { cph[q] = 0; alive[q] = true; }
  int nalive = kStages;
  for (;;) {
    RS_T0(tf);
    if (kProducers == 1) {
      mbar_wait(&full_bar[stage], phase);
    } else {
      // the first stage to fill (independent producers: a fixed order could wait
      // on a task whose dependency sits in the other stage)
      if (nalive == 0) break;
      if (ct == 0) {
        int q0 = -1;
        while (q0 < 0) {
#pragma unroll
          for (int q = 0; q < kStages; ++q)
            if (q0 < 0 && alive[q] && mbar_test_wait(&full_bar[q], cph[q])) q0 = q;
        }
        s_pick = q0;
      }
      consumer_sync();
      stage = s_pick;
      mbar_wait(&full_bar[stage], cph[stage]);  // completed: orders the bulk data for this thread
      cph[stage] ^= 1;
    }
    if (ct == 0) RS_ACC(E.met, 3, tf);
    RS_T0(tk);
    const StageHdr h = hdr[stage];
    if (h.end) {
      if (cl == 0) mbar_arrive(&stored_bar[stage]);
      if (kProducers == 1) break;
      alive[stage] = false;
      --nalive;
      consumer_sync();  // s_pick read by all before it is rewritten
      continue;
    }
    unsigned char* base = smem + (size_t)stage * C::STAGE;
    K* sk = reinterpret_cast<K*>(base);
    T* st = reinterpret_cast<T*>(base + C::KBYTES);
    const K* A = sk + h.offA;
    const K* B = sk + h.offB;
    const T* TA = HT ? st + h.toffA : nullptr;
    const T* TBp = HT ? st + h.toffB : nullptr;
    int len = h.len, la = h.la, lb = len - la;
#ifdef RS_DEBUG_CHECKS
    for (int i = ct; i + 1 < la; i += kConsumerThreads)
      RS_CHECK(A[i] <= A[i + 1], "A window unsorted: node %u dst %lld i %d la %d", h.node, (long long)h.dst, i, la);
    for (int i = ct; i + 1 < lb; i += kConsumerThreads) {
      if (!(B[i] <= B[i + 1])) {
        const K* gB = reinterpret_cast<const K*>(h.dbg_srcB);
        K g0 = ld_volatile_k(gB + i), g1 = ld_volatile_k(gB + i + 1);
        printf("B window unsorted: node %u dst %lld i %d lb %d smem %lld %lld global-now %lld %lld child %u dn@ready %u "
               "done-now %u need %u\n",
               h.node, (long long)h.dst, i, lb, (long long)B[i], (long long)B[i + 1], (long long)g0, (long long)g1,
               h.dbg_cB, h.dbg_dnB, ld_acquire_u32(E.done + h.dbg_cB), E.need[h.dbg_cB]);
        __trap();
      }
    }
#endif
    int d0 = ct * C::IPT;
    int cnt = len - d0;
    cnt = cnt < 0 ? 0 : (cnt > C::IPT ? C::IPT : cnt);
    K rk[C::IPT];
    T rt[HT ? C::IPT : 1];
    if (cnt > 0) {
      // lean merge-path search: lo = #A outputs before diagonal d0
      int lo = d0 - lb > 0 ? d0 - lb : 0;
      int len_s = (d0 < la ? d0 : la) - lo;
      while (len_s > 0) {
        int half = len_s >> 1;
        int mid = lo + half;
        bool c = A[mid] <= B[d0 - 1 - mid];
        lo = c ? mid + 1 : lo;
        len_s = c ? len_s - half - 1 : half;
      }
      const K* pa = A + lo;
      const K* pb = B + (d0 - lo);
      const K* ea = A + la;
      const K* eb = B + lb;
      K va = *pa, vb = *pb;
      if (cnt == C::IPT) {
#pragma unroll
        for (int q = 0; q < C::IPT; ++q) {
          bool p = (pa < ea) && (pb >= eb || va <= vb);
          rk[q] = p ? va : vb;
          if (HT) rt[q] = p ? TA[pa - A] : TBp[pb - B];
          pa += p;
          pb += !p;
          K nv = *(p ? pa : pb);
          va = p ? nv : va;
          vb = p ? vb : nv;
        }
      } else {
#pragma unroll
        for (int q = 0; q < C::IPT; ++q) {
          if (q < cnt) {
            bool p = (pa < ea) && (pb >= eb || va <= vb);
            rk[q] = p ? va : vb;
            if (HT) rt[q] = p ? TA[pa - A] : TBp[pb - B];
            pa += p;
            pb += !p;
            K nv = *(p ? pa : pb);
            va = p ? nv : va;
            vb = p ? vb : nv;
          }
        }
      }
    }
    // stage the merged tile in SMEM with the destination's 16B phase; the
    // signaller streams it out with bulk stores and publishes it
    const int pad = int((reinterpret_cast<uintptr_t>(reinterpret_cast<K*>(E.key[h.parity]) + h.dst) & 15) /
                        sizeof(K));
    const int tpad = HT ? int((reinterpret_cast<uintptr_t>(reinterpret_cast<T*>(E.tag[h.parity]) + h.dst) & 15) /
                              (HT ? TB : 1))
                        : 0;
    consumer_sync();  // every thread's merge has read the stage's inputs
#pragma unroll
    for (int q = 0; q < C::IPT; ++q) {
      if (q < cnt) {
        sk[pad + d0 + q] = rk[q];
        if (HT) st[tpad + d0 + q] = rt[q];
      }
    }
#ifdef RS_DEBUG_CHECKS
    consumer_sync();
    for (int i = ct; i + 1 < len; i += kConsumerThreads)
      RS_CHECK(sk[pad + i] <= sk[pad + i + 1], "merged tile unsorted in smem: node %u dst %lld i %d len %d la %d",
               h.node, (long long)h.dst, i, len, la);
    consumer_sync();
#endif
    // generic SMEM writes -> visible to the bulk copy engine, then one arrival per warp
    fence_proxy_async_smem();
    __syncwarp();
    if (cl == 0) mbar_arrive(&stored_bar[stage]);
    if (ct == 0) RS_ACC(E.met, 4, tk);
    if (kProducers == 1 && ++stage == kStages) { stage = 0; phase ^= 1; }
  }
}

}  // namespace rs
