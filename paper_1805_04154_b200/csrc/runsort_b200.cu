// runsort_b200.cu -- C ABI (include/runsort_b200.h) and launch orchestration.
//
// Pipeline for powersort (reference sorters.py:430-519), all on one stream,
// no host synchronisation until the caller asks for the Metrics:
//   1. k_scan_tables   pair-type bits + per-tile min-run candidate tables
//   2. k_group_compose / k_group_entries / k_tile_entries / k_emit_leaves
//                      -> leaf starts and natural-run info (sorters.py:462-470)
//   3. k_keys_powers   midpoint keys, node powers (sorters.py:414-423)
//   4. k_scan_*        left/right ancestor counts -> depths, max stack height
//   5. k_tree          trie ranges, parents, children, spans
//   6. k_classify / k_task_offsets / k_task_fill   executor task list
//   7. k_execute       persistent dataflow executor (leaves + merges)
#include <algorithm>
#include <chrono>
#include <functional>
#include <map>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <mutex>
#include <string>
#include <vector>

#include "../../include/runsort_b200.h"
#include "rs_baseline.cuh"
#include "rs_chain.cuh"
#include "rs_common.cuh"
#include "rs_exec.cuh"
#include "rs_host.h"
#include "rs_kway.cuh"
#include "rs_merge.cuh"
#include "rs_prep.cuh"
#include "rs_peek.cuh"
#include "rs_tree.cuh"

using namespace rs;

namespace {

thread_local std::string g_err;

constexpr int kPhases = 3;  // prep, phase A, merge
struct Prof {
  bool on = false;
  bool created = false;
  bool recorded = false;
  cudaEvent_t ev[kPhases + 1];
  const DevMetrics* met = nullptr;  // of the last profiled call
};
thread_local Prof g_prof;

void prof_mark(int i, cudaStream_t st) {
  if (!g_prof.on) return;
  if (!g_prof.created) {
    for (auto& e : g_prof.ev) cudaEventCreate(&e);
    g_prof.created = true;
  }
  cudaEventRecord(g_prof.ev[i], st);
  if (i == kPhases) g_prof.recorded = true;
}
void prof_set_met(const DevMetrics* m) {
  if (g_prof.on) g_prof.met = m;
}

int fail(int code, const std::string& msg) {
  g_err = msg;
  return code;
}

#define RS_CUDA(call)                                                                    \
  do {                                                                                   \
    cudaError_t e_ = (call);                                                             \
    if (e_ != cudaSuccess)                                                               \
      return fail(RS_ECUDA, std::string(#call " failed: ") + cudaGetErrorString(e_));   \
  } while (0)

size_t align_up(size_t x, size_t a) { return (x + a - 1) / a * a; }

// Tuning overrides (environment), read once per process: the product path
// never calls getenv per sort (thread-safe static initialisation).
struct Tunables {
  int chain_tile = 0;    // RS_CHAIN_TILE: force 1024 / 2048 / 2560-position chain tiles
  int fcap = 0;          // RS_FCAP: cap the fused-subtree size
  int merge_super = 0;   // RS_MERGE_SUPER: tiles per merge task
  int fuse_avg = 256;    // RS_FUSE_AVG: fuse subtrees when n < fuse_avg * r
  int merge_ahead = -1;  // RS_MERGE_AHEAD: claim-ahead merge producer (-1 = from msuper)
  bool no_pdl = false;   // RS_NO_PDL: plain launches instead of programmatic dependent launch
  bool prep_twice = false;  // RS_PREP_TWICE (RS_INSTR builds): a second, warm-code prep
  int debug_algo = -1;   // RS_DEBUG_ALGO: rs_debug_counters reads another algorithm's layout
  bool host_trace = false;  // RS_HOST_TRACE: rs_sort_host phase timings on stderr
  int small_fuse = 1;          // RS_SMALL_FUSE: small-tree path fuses >= 3-leaf subtrees of long leaves
  int est_c0 = 0, est_c1 = 0;  // RS_EST_C0 / RS_EST_C1: small-tree merge-job order model (ns; 0 = defaults)
};
const Tunables& tun() {
  static const Tunables t = [] {
    Tunables v;
    auto geti = [](const char* k, int d) {
      const char* e = getenv(k);
      return e ? atoi(e) : d;
    };
    v.chain_tile = geti("RS_CHAIN_TILE", 0);
    v.fcap = geti("RS_FCAP", 0);
    v.merge_super = geti("RS_MERGE_SUPER", 0);
    v.fuse_avg = geti("RS_FUSE_AVG", 256);
    v.merge_ahead = geti("RS_MERGE_AHEAD", -1);
    v.no_pdl = getenv("RS_NO_PDL") != nullptr;
    v.prep_twice = getenv("RS_PREP_TWICE") != nullptr;
    v.debug_algo = geti("RS_DEBUG_ALGO", -1);
    v.host_trace = getenv("RS_HOST_TRACE") != nullptr;
    v.small_fuse = geti("RS_SMALL_FUSE", 1);
    v.est_c0 = geti("RS_EST_C0", 0);
    v.est_c1 = geti("RS_EST_C1", 0);
    return v;
  }();
  return t;
}

constexpr size_t kMaxSmemPerBlock = 227 * 1024;

// Dynamic shared memory of k_prep for (w, key bytes, chain tile).
size_t prep_smem_bytes(int w, int kb, int ct) {
  int W1 = w + 1;
  int maxw = kMaxWinWords(w, ct);
  int batch = (int)((40 * 1024 - (size_t)W1 * 8) / ((size_t)W1 * 8));
  if (batch < 1) batch = 1;
  if (batch > kTableBatch) batch = kTableBatch;
  int gbatch = (int)(40 * 1024 / ((size_t)W1 * 8));
  if (gbatch < 1) gbatch = 1;
  int tbatch = gbatch < kChainGroup ? gbatch : kChainGroup;
  size_t sm = 8 * (size_t)chain_warp_bytes(w, kb, ct);
  sm = std::max(sm, (size_t)kFillSmem + 64);
  sm = std::max(sm, (size_t)batch * W1 * 8 + (size_t)W1 * 8 + 64);
  sm = std::max(sm, (size_t)gbatch * W1 * 8);
  sm = std::max(sm, (size_t)tbatch * W1 * 8);
  sm = std::max(sm, (size_t)8 * (maxw * 2 + (maxw + 1) / 2 + 1) * 4);
  sm = std::max(sm, small_smem_bytes());
  return sm;
}

// Positions per chain tile (k_prep is instantiated for 512, 1024, 2048 and 2560):
// up to 2^22 keys 512 (short leaves make the per-tile walks and the leaf emission serial chains of
// tile / min_run_len steps; measured on random permutations and config-2-shaped inputs);
// below ~7M keys 2048-position tiles leave most prep warps without a tile and
// 1024 is faster (cfg1, n = 2^20: -9%); above that 2560 (fewer tiles for
// the group/emit phases; 2048 remains the shared-memory fallback).  A function of n only, so every layout agrees.
// Large min_run_len values step the tile down until the prep's per-warp
// windows fit in shared memory (a function of (n, w, key bytes) only).
inline int chain_tile_for(int64_t n, int w, int kb) {
  int ct;
  if (int v = tun().chain_tile) ct = v >= 2560 ? 2560 : (v >= 2048 ? 2048 : (v >= 1024 ? 1024 : 512));  // tuning override
  else if (n <= ((int64_t)1 << 22) && w <= 64) ct = 512;  // round 2: cfg1 (2^20) -17 us vs 1024, random 4M -13 us, cfg2-shaped 2M equal
  else if (n < (int64_t)2048 * 3552) ct = 1024;
  else ct = 2560;  // round 2: cfg2 (1e7) -2.8 us vs 2048 (3 repeats), cfg3 -4 us, cfg4 -30 us
  while (ct > 1024 && prep_smem_bytes(w, kb, ct) > kMaxSmemPerBlock) ct = ct == 2560 ? 2048 : 1024;
  return ct;
}

struct Layout {
  // inputs
  int64_t n;
  int w, kb, tb;
  int chain_t;  // positions per chain tile
  int tile, fcap;
  // derived sizes
  int64_t words, ntiles, ngroups, r_max, nchunks, max_tasks;
  uint32_t leaf_base;
  // offsets
  size_t o_key1, o_tag1, o_key2, o_tag2, o_ascw, o_tables, o_gtab, o_gentry, o_goff, o_tentry, o_toff;
  size_t o_leaf_start, o_leaf_info, o_leaf_depth, o_K, o_P, o_la, o_ra, o_depth;
  size_t o_node_a, o_node_b, o_node_s, o_node_e, o_parent, o_child, o_need, o_done;
  size_t o_agg, o_tasks, o_mdesc, o_chunkdep, o_cls, o_jobs, o_met, total;
  int64_t mdesc_cap;  // merge-task descriptors (indexed from the first merge task)
  // peeksort replay
  int algo;
  int full_ws;  // RS_ALGO_FULL_WS: replay capacity n + 1 instead of the compact one
  int64_t front_cap, rec_cap, sum_words, wchunks;
  size_t o_front0, o_front1, o_pnodes, o_pleaves, o_prevs, o_lbits, o_wpre, o_wchunk, o_nozero, o_noone;
};

int exec_tile(int kb, int tb) {
  if (kb == 4) return tb == 0 ? ExecCfg<int32_t, 0>::TILE : (tb == 4 ? ExecCfg<int32_t, 4>::TILE : ExecCfg<int32_t, 8>::TILE);
  return tb == 0 ? ExecCfg<int64_t, 0>::TILE : (tb == 4 ? ExecCfg<int64_t, 4>::TILE : ExecCfg<int64_t, 8>::TILE);
}
int exec_fcap(int kb, int tb) {
  if (kb == 4) return tb == 0 ? ExecCfg<int32_t, 0>::FCAP : (tb == 4 ? ExecCfg<int32_t, 4>::FCAP : ExecCfg<int32_t, 8>::FCAP);
  return tb == 0 ? ExecCfg<int64_t, 0>::FCAP : (tb == 4 ? ExecCfg<int64_t, 4>::FCAP : ExecCfg<int64_t, 8>::FCAP);
}

// Peeksort's replay capacity (recursive calls per level, leaves, merge nodes,
// reversals; also its leaf bound r_max).  Leaves can be single elements, so
// only n + 1 is safe for every input (RS_ALGO_FULL_WS: ~290 bytes per
// element).  The compact default holds n / 12 + 4096 of each -- min_run_len =
// 24 on a random permutation gives ~n / 17 leaves -- with the frontier
// ping-pong laid over the two scratch key/tag buffers, which nothing uses
// before the executors run; a replay that would overflow restores the input
// and reports RS_ECAPACITY (rs_peek.cuh), and the caller sorts again with
// RS_ALGO_FULL_WS.
int64_t peek_capacity(int64_t n, bool full) {
  int64_t c = n / 12 + 4096;
  return full || c > n + 1 ? n + 1 : c;
}

// `algo` may carry RS_ALGO_FULL_WS.
Layout make_layout(int64_t n, int w, int kb, int tb, int algo) {
  Layout L{};
  L.full_ws = (algo & RS_ALGO_FULL_WS) != 0;
  algo &= ~RS_ALGO_FULL_WS;
  L.algo = algo;
  L.n = n;
  L.w = w;
  L.kb = kb;
  L.tb = tb;
  L.tile = exec_tile(kb, tb);
  L.fcap = exec_fcap(kb, tb);
  if (int v = tun().fcap) L.fcap = std::max(2, std::min(L.fcap, v));  // tuning override
  L.words = (n + 31) / 32 + 2;
  L.chain_t = chain_tile_for(n, w, kb);
  L.ntiles = (n + L.chain_t - 1) / L.chain_t;
  L.ngroups = (L.ntiles + kChainGroup - 1) / kChainGroup;
  int64_t minleaf = w > 2 ? w : 2;
  if (algo == RS_ALGO_TOP_DOWN) minleaf = (w + 1) / 2;  // halves of ranges > w
  if (algo == RS_ALGO_BOTTOM_UP) minleaf = w;            // chunks of w
  L.r_max = n / minleaf + 2;
  if (L.r_max > n + 1) L.r_max = n + 1;
  if (algo == RS_ALGO_PEEKSORT) {  // leaves can be single elements
    if (peek_capacity(n, false) == n + 1) L.full_ws = 1;  // small n: the compact capacity is the full one
    L.r_max = peek_capacity(n, L.full_ws);
  }
  L.leaf_base = (uint32_t)(L.r_max + 1);
  L.nchunks = (L.r_max + kScanThreads - 1) / kScanThreads + 1;
  int levels = 2;
  for (int64_t x = n; x; x >>= 1) ++levels;
  L.max_tasks = (int64_t)levels * (n / L.tile + n / L.fcap + 2) + 3 * L.r_max + 2 * (n / L.tile) + 16;
  size_t off = 0;
  auto take = [&](size_t bytes) {
    size_t o = off;
    off = align_up(off + bytes, 256);
    return o;
  };
  L.o_key1 = take((size_t)n * kb + 64);
  L.o_tag1 = take((size_t)n * tb + 64);
  L.o_key2 = take((size_t)n * kb + 64);
  L.o_tag2 = take((size_t)n * tb + 64);
  L.o_ascw = take((size_t)L.words * 4);
  bool pk = algo == RS_ALGO_PEEKSORT;
  L.o_tables = take(pk ? 0 : (size_t)L.ntiles * (w + 1) * 8);
  L.o_gtab = take(pk ? 0 : (size_t)L.ngroups * (w + 1) * 8);
  L.o_gentry = take((size_t)L.ngroups * 4);
  L.o_goff = take((size_t)L.ngroups * 8);
  L.o_tentry = take((size_t)L.ntiles * 4);
  L.o_toff = take((size_t)L.ntiles * 8);
  L.o_leaf_start = take((size_t)(L.r_max + 1) * 8);
  L.o_leaf_info = take((size_t)L.r_max * 4);
  L.o_leaf_depth = take((size_t)L.r_max);
  L.o_K = take((size_t)L.r_max * 8);
  L.o_P = take((size_t)L.r_max);
  L.o_la = take((size_t)L.r_max);
  L.o_ra = take((size_t)L.r_max);
  L.o_depth = take((size_t)L.r_max);
  L.o_node_a = take((size_t)L.r_max * 4);
  L.o_node_b = take((size_t)L.r_max * 4);
  L.o_node_s = take((size_t)L.r_max * 8);
  L.o_node_e = take((size_t)L.r_max * 8);
  L.o_parent = take((size_t)(2 * L.r_max + 2) * 4);
  L.o_child = take((size_t)(2 * L.r_max + 2) * 4);
  L.o_need = take((size_t)(2 * L.r_max + 2) * 4);
  L.o_done = take((size_t)(2 * L.r_max + 2) * 4);
  L.o_agg = take((size_t)2 * L.nchunks * sizeof(MC));
  L.o_tasks = take((size_t)L.max_tasks * 8);
  // merge tasks <= sum over merge nodes of (span / tile + 1): merge_cost <= n * levels elements
  // in tiles of >= 1792 (16-byte elements), plus one per merge node (<= r_max; peeksort:
  // fused subtrees or >= 8-element average leaves).  Overflow is caught on the device.
  L.mdesc_cap = (int64_t)levels * (n / 1792 + 1) + (algo == RS_ALGO_PEEKSORT ? std::min<int64_t>(n / 8, L.r_max) : L.r_max) + 64;
  if (L.mdesc_cap > L.max_tasks) L.mdesc_cap = L.max_tasks;
  L.o_mdesc = take((size_t)L.mdesc_cap * sizeof(MDesc));
  L.o_chunkdep = take((size_t)((L.r_max + kOrdChunkMin - 1) / kOrdChunkMin + 1) * kMaxDepth * 4);
  L.o_cls = take((size_t)(2 * L.r_max + 2));
  L.o_jobs = take(small_jobs_bytes());
  if (pk) {
    L.rec_cap = L.r_max;
    L.sum_words = skip_tree_words(L.words);
    L.wchunks = (L.words + kWordChunk - 1) / kWordChunk + 1;
    if (L.full_ws) {
      L.front_cap = L.rec_cap;
      L.o_front0 = take((size_t)L.front_cap * sizeof(PeekItem));
      L.o_front1 = take((size_t)L.front_cap * sizeof(PeekItem));
    } else {
      // the frontier ping-pong over the scratch buffers (key1 + tag1, key2 + tag2)
      L.o_front0 = L.o_key1;
      L.o_front1 = L.o_key2;
      int64_t fit = (int64_t)(std::min(L.o_key2 - L.o_key1, L.o_ascw - L.o_key2) / sizeof(PeekItem));
      L.front_cap = std::min(L.rec_cap, fit);
    }
    L.o_pnodes = take((size_t)L.rec_cap * 32);
    L.o_pleaves = take((size_t)L.rec_cap * 32);
    L.o_prevs = take((size_t)L.rec_cap * 16);
    L.o_lbits = take((size_t)L.words * 4);
    L.o_wpre = take((size_t)L.words * 4);
    L.o_wchunk = take((size_t)L.wchunks * 4);
    L.o_nozero = take((size_t)L.sum_words * 4);
    L.o_noone = take((size_t)L.sum_words * 4);
  }
  L.o_met = take(sizeof(DevMetrics));
  L.total = off + 256;
  return L;
}

struct DevInfo {
  int sms = 0;
  bool init = false;
};
std::mutex g_mu;
DevInfo g_dev[64];

int device_sms(int* sms) {
  int dev;
  RS_CUDA(cudaGetDevice(&dev));
  std::lock_guard<std::mutex> lk(g_mu);
  if (!g_dev[dev].init) {
    RS_CUDA(cudaDeviceGetAttribute(&g_dev[dev].sms, cudaDevAttrMultiProcessorCount, dev));
    g_dev[dev].init = true;
  }
  *sms = g_dev[dev].sms;
  return RS_OK;
}

// Per-device launch geometry, computed once under g_mu.  The shared-memory
// attribute of a kernel only ever grows (concurrent sorts with different
// min_run_len on other threads never see it shrink under their launch), and
// occupancies are cached per (device, shared-memory size).
struct OccKey {
  const void* fn;
  int dev;
  size_t smem;
  bool operator<(const OccKey& o) const {
    return fn != o.fn ? fn < o.fn : (dev != o.dev ? dev < o.dev : smem < o.smem);
  }
};
std::map<OccKey, int> g_occ;                         // guarded by g_mu
std::map<std::pair<const void*, int>, size_t> g_attr;  // guarded by g_mu

int occupancy(const void* fn, int threads, size_t smem, size_t attr_smem, int* occ, const char* what) {
  int dev;
  RS_CUDA(cudaGetDevice(&dev));
  std::lock_guard<std::mutex> lk(g_mu);
  size_t& cur = g_attr[{fn, dev}];
  size_t want = std::max(smem, attr_smem);
  if (want > cur) {
    RS_CUDA(cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)want));
    cur = want;
  }
  auto it = g_occ.find(OccKey{fn, dev, smem});
  if (it == g_occ.end()) {
    int o = 0;
    RS_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&o, fn, threads, smem));
    if (o < 1) return fail(RS_ECUDA, std::string(what) + " does not fit on an SM");
    it = g_occ.emplace(OccKey{fn, dev, smem}, o).first;
  }
  *occ = it->second;
  return RS_OK;
}

template <typename K, int TB>
int exec_grid(int sms, int w, int* grid_a, size_t* smem_a, int* grid_m, size_t* smem_m) {
  *smem_a = Exec<K, TB>::smem_bytes(w);
  *smem_m = MergeCfg<K, TB>::SMEM;
  int oa, om, om2;
  if (int e = occupancy((const void*)k_phaseA<K, TB>, kExecThreads, *smem_a, Exec<K, TB>::smem_bytes(1), &oa,
                        "phase-A kernel"))
    return e;
  if (int e = occupancy((const void*)k_merge_exec<K, TB, false>, kMergeThreads, *smem_m, *smem_m, &om,
                        "merge executor"))
    return e;
  if (int e = occupancy((const void*)k_merge_exec<K, TB, true>, kMergeThreads, *smem_m, *smem_m, &om2,
                        "merge executor"))
    return e;
  *grid_a = sms * oa;
  *grid_m = sms * std::min(om, om2);
  return RS_OK;
}

// Launch with programmatic stream serialization: the kernel may start while
// the previous kernel on the stream finishes (it calls pdl_wait() before
// touching that kernel's outputs).  RS_NO_PDL=1 launches normally.
template <typename Kern, typename Arg>
cudaError_t pdl_launch(Kern kern, int grid, int block, size_t smem, cudaStream_t st, const Arg& arg) {
  const bool off = tun().no_pdl;
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(grid);
  cfg.blockDim = dim3(block);
  cfg.dynamicSmemBytes = smem;
  cfg.stream = st;
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  at[0].val.programmaticStreamSerializationAllowed = off ? 0 : 1;
  cfg.attrs = at;
  cfg.numAttrs = 1;
  return cudaLaunchKernelEx(&cfg, kern, arg);
}

template <typename K, int CT>
int prep_grid(int sms, size_t smem, int* grid) {
  int o;
  if (int e = occupancy((const void*)k_prep<K, CT>, 256, smem, smem, &o, "prep kernel")) return e;
  *grid = sms * o;
  return RS_OK;
}

// Tiles per merge task: enough tasks per tree level to keep every executor
// CTA busy (>= ~8 per CTA), as many tiles as that allows so the producer's
// split searches (one HBM round trip per step) are shared by more tiles.
template <typename K, int TB>
int merge_super(int64_t n, int sms) {
  int64_t ctas = (int64_t)sms * 3;
  int64_t per_level_tiles = n / MergeCfg<K, TB>::TILE;
  int64_t s = per_level_tiles / (8 * ctas);
  if (int v = tun().merge_super) s = v;  // tuning override
  if (s < 1) s = 1;
  if (s > 7) s = 7;
  return (int)s;
}

struct WsView {
  DevMetrics* met;
  uint32_t *ascw, *gentry, *tentry, *need, *done, *child, *chunkdep;
  uint2 *tables, *gtab;
  uint64_t *goff, *toff, *Kk, *tasks;
  MDesc* mdesc;
  pos_t *leaf_start, *node_s, *node_e;
  uint32_t* leaf_info;
  uint8_t *leaf_depth, *P, *la, *ra, *depth, *cls;
  int32_t *node_a, *node_b, *parent;
  MC* agg;
  void* key1;
  void* tag1;
  void* key2;
  void* tag2;
  unsigned char* jobs;
};

WsView view(unsigned char* ws, const Layout& L) {
  auto at = [&](size_t o) { return ws + o; };
  WsView V;
  V.met = reinterpret_cast<DevMetrics*>(at(L.o_met));
  V.ascw = reinterpret_cast<uint32_t*>(at(L.o_ascw));
  V.tables = reinterpret_cast<uint2*>(at(L.o_tables));
  V.gtab = reinterpret_cast<uint2*>(at(L.o_gtab));
  V.gentry = reinterpret_cast<uint32_t*>(at(L.o_gentry));
  V.goff = reinterpret_cast<uint64_t*>(at(L.o_goff));
  V.tentry = reinterpret_cast<uint32_t*>(at(L.o_tentry));
  V.toff = reinterpret_cast<uint64_t*>(at(L.o_toff));
  V.leaf_start = reinterpret_cast<pos_t*>(at(L.o_leaf_start));
  V.leaf_info = reinterpret_cast<uint32_t*>(at(L.o_leaf_info));
  V.leaf_depth = at(L.o_leaf_depth);
  V.Kk = reinterpret_cast<uint64_t*>(at(L.o_K));
  V.P = at(L.o_P);
  V.la = at(L.o_la);
  V.ra = at(L.o_ra);
  V.depth = at(L.o_depth);
  V.node_a = reinterpret_cast<int32_t*>(at(L.o_node_a));
  V.node_b = reinterpret_cast<int32_t*>(at(L.o_node_b));
  V.node_s = reinterpret_cast<pos_t*>(at(L.o_node_s));
  V.node_e = reinterpret_cast<pos_t*>(at(L.o_node_e));
  V.parent = reinterpret_cast<int32_t*>(at(L.o_parent));
  V.child = reinterpret_cast<uint32_t*>(at(L.o_child));
  V.need = reinterpret_cast<uint32_t*>(at(L.o_need));
  V.done = reinterpret_cast<uint32_t*>(at(L.o_done));
  V.agg = reinterpret_cast<MC*>(at(L.o_agg));
  V.tasks = reinterpret_cast<uint64_t*>(at(L.o_tasks));
  V.mdesc = reinterpret_cast<MDesc*>(at(L.o_mdesc));
  V.chunkdep = reinterpret_cast<uint32_t*>(at(L.o_chunkdep));
  V.cls = reinterpret_cast<uint8_t*>(at(L.o_cls));
  V.jobs = at(L.o_jobs);
  V.key1 = at(L.o_key1);
  V.tag1 = at(L.o_tag1);
  V.key2 = at(L.o_key2);
  V.tag2 = at(L.o_tag2);
  return V;
}

TreeArrays tree_arrays(const WsView& V, const Layout& L) {
  return TreeArrays{V.leaf_start, V.leaf_info, V.Kk, V.P, V.la, V.ra, V.depth, V.leaf_depth, V.node_a,
                    V.node_b, V.parent, V.child, V.node_s, V.node_e, L.leaf_base};
}

// Fused phase-A subtrees only for short leaves on average (measured on B200:
// cfg1's 24-element leaves gain 2x from fusing, cfg2/cfg4's ~1-3K-element runs
// merge faster in the executor).
int fuse_avg() { return tun().fuse_avg; }

template <typename K, int TB>
ClassifyArgs classify_args(const WsView& V, const Layout& L, int64_t n, int w, int classic, int msuper, int peek,
                           int runtime_merges = 0, int fcap = -1) {
  return ClassifyArgs{n, w, classic, fcap >= 0 ? fcap : L.fcap, L.tile, MergeCfg<K, TB>::TILE, msuper, peek,
                      runtime_merges, L.leaf_base,
                      V.leaf_start, V.leaf_info, V.leaf_depth, V.depth, V.node_s, V.node_e, V.parent, V.need,
                      V.cls, V.tasks, V.met, V.node_a, V.node_b, Exec<K, TB>::maxb_for(w), fuse_avg(), V.child,
                      V.mdesc, L.mdesc_cap};
}

// Phase A (fused subtrees, large leaves) + the merge executor.
template <typename K, int TB>
int launch_exec(K* keys, void* tags, int64_t n, int w, int classic, int msuper, const WsView& V, const Layout& L,
                int sms, cudaStream_t st, int skipchk = 0) {
  int grid_a, grid_m;
  size_t smem_a, smem_m;
  if (int e = exec_grid<K, TB>(sms, w, &grid_a, &smem_a, &grid_m, &smem_m)) return e;
  ExecArgs E;
  E.key[0] = keys;
  E.key[1] = V.key1;
  E.key[2] = V.key2;
  E.tag[2] = V.tag2;
  E.tag[0] = tags;
  E.tag[1] = V.tag1;
  E.n = n;
  E.w = w;
  E.classic = classic;
  E.leaf_base = L.leaf_base;
  E.leaf_start = V.leaf_start;
  E.leaf_info = V.leaf_info;
  E.leaf_depth = V.leaf_depth;
  E.depth = V.depth;
  E.node_a = V.node_a;
  E.node_b = V.node_b;
  E.node_s = V.node_s;
  E.node_e = V.node_e;
  E.child = V.child;
  E.need = V.need;
  E.done = V.done;
  E.tasks = V.tasks;
  E.met = V.met;
  E.maxb = Exec<K, TB>::maxb_for(w);
  if (cudaError_t e_ = pdl_launch(k_phaseA<K, TB>, grid_a, kExecThreads, smem_a, st, E))
    return fail(RS_ECUDA, std::string("k_phaseA launch failed: ") + cudaGetErrorString(e_));
  if (cudaError_t e_ = cudaGetLastError())
    return fail(RS_ECUDA, std::string("k_phaseA launch/exec failed: ") + cudaGetErrorString(e_));
  prof_mark(2, st);
  MergeArgs M;
  M.key[0] = E.key[0];
  M.key[1] = E.key[1];
  M.tag[0] = E.tag[0];
  M.tag[1] = E.tag[1];
  M.key[2] = E.key[2];
  M.tag[2] = E.tag[2];
  M.cls = V.cls;
  M.leaf_base = L.leaf_base;
  M.classic = classic;
  M.msuper = msuper;
  M.skipchk = skipchk;
  M.leaf_start = V.leaf_start;
  M.depth = V.depth;
  M.node_s = V.node_s;
  M.node_e = V.node_e;
  M.child = V.child;
  M.need = V.need;
  M.done = V.done;
  M.tasks = V.tasks;
  M.mdesc = V.mdesc;
  M.mdesc_cap = L.mdesc_cap;
  M.met = V.met;
  bool ahead = msuper > 1;
  if (tun().merge_ahead >= 0) ahead = tun().merge_ahead != 0;  // tuning override
  cudaError_t le = ahead ? pdl_launch(k_merge_exec<K, TB, true>, grid_m, kMergeThreads, smem_m, st, M)
                         : pdl_launch(k_merge_exec<K, TB, false>, grid_m, kMergeThreads, smem_m, st, M);
  if (le != cudaSuccess) return fail(RS_ECUDA, std::string("k_merge_exec launch failed: ") + cudaGetErrorString(le));
  if (cudaError_t e_ = cudaGetLastError())
    return fail(RS_ECUDA, std::string("k_merge_exec launch/exec failed: ") + cudaGetErrorString(e_));
  prof_mark(3, st);
  return RS_OK;
}

template <typename K, int TB>
int run_powersort(K* keys, void* tags, int64_t n, int w, int classic, unsigned char* ws, const Layout& L,
                  cudaStream_t st, int leaves_only = 0) {
  int sms;
  if (int e = device_sms(&sms)) return e;
  WsView V = view(ws, L);
  prof_mark(0, st);
  prof_set_met(V.met);
  // everything before the executors in one cooperative kernel
  const int ct = L.chain_t;
  int W1 = w + 1;
  int batch = (int)((40 * 1024 - (size_t)W1 * 8) / ((size_t)W1 * 8));
  if (batch < 1) batch = 1;
  if (batch > kTableBatch) batch = kTableBatch;
  int gbatch = (int)(40 * 1024 / ((size_t)W1 * 8));
  if (gbatch < 1) gbatch = 1;
  int tbatch = gbatch < kChainGroup ? gbatch : kChainGroup;
  size_t sm = prep_smem_bytes(w, (int)sizeof(K), ct);
  if (sm > kMaxSmemPerBlock) return fail(RS_EUNSUPPORTED, "min_run_len too large for the prep kernel's shared memory");
  int F = n <= ((int64_t)1 << 31) ? 32 : 63;
  int64_t nch_max = (L.r_max + kOrdChunkMin - 1) / kOrdChunkMin;
  PrepArgs PA;
  PA.keys = keys;
  PA.n = n;
  PA.w = w;
  PA.F = F;
  PA.batch = batch;
  PA.gbatch = gbatch;
  PA.tbatch = tbatch;
  PA.ntiles = L.ntiles;
  PA.ngroups = L.ngroups;
  PA.r_max = L.r_max;
  PA.nchunks = L.nchunks;
  PA.ascw = V.ascw;
  PA.tables = V.tables;
  PA.gtab = V.gtab;
  PA.gentry = V.gentry;
  PA.goff = V.goff;
  PA.tentry = V.tentry;
  PA.toff = V.toff;
  PA.agg = V.agg;
  PA.chunkdep = V.chunkdep;
  PA.chunkdep_words = (nch_max + 1) * kMaxDepth;
  PA.done = V.done;
  PA.done_words = 2 * L.r_max + 2;
  PA.T = tree_arrays(V, L);
  PA.leaves_only = leaves_only;
  int msuper = merge_super<K, TB>(n, sms);
  PA.CA = classify_args<K, TB>(V, L, n, w, classic, msuper, 0);
  PA.CA.la = V.la;  // the grid path's classification derives the depths
  PA.CA.ra = V.ra;
  PA.CA.small_fuse = tun().small_fuse;
  if (tun().est_c0 > 0) PA.CA.est_c0 = tun().est_c0;
  if (tun().est_c1 > 0) PA.CA.est_c1 = tun().est_c1;
  PA.jobs = SmallJobs::at(V.jobs);
  int grid_p;
  void* kprep = ct == 512    ? (void*)k_prep<K, 512>
                : ct == 1024 ? (void*)k_prep<K, 1024>
                : ct == 2560 ? (void*)k_prep<K, 2560>
                             : (void*)k_prep<K, 2048>;
  if (int e = (ct == 512    ? prep_grid<K, 512>(sms, sm, &grid_p)
               : ct == 1024 ? prep_grid<K, 1024>(sms, sm, &grid_p)
               : ct == 2560 ? prep_grid<K, 2560>(sms, sm, &grid_p)
                            : prep_grid<K, 2048>(sms, sm, &grid_p)))
    return e;
  void* kargs[] = {&PA};
  RS_CUDA(cudaLaunchCooperativeKernel(kprep, dim3(grid_p), dim3(256), kargs, sm, st));
#ifdef RS_INSTR
  if (tun().prep_twice)  // experiment: a second, warm-code prep (idempotent)
    RS_CUDA(cudaLaunchCooperativeKernel(kprep, dim3(grid_p), dim3(256), kargs, sm, st));
#endif
  if (leaves_only) return RS_OK;
  prof_mark(1, st);
  return launch_exec<K, TB>(keys, tags, n, w, classic, msuper, V, L, sms, st);
}

// ------------------------------------------------ baseline sorters' trees
// Host-built merge trees in the workspace's tree format: leaves i = 0..r-1
// (unified id leaf_base + i), internal node j = the boundary between leaf j-1
// and leaf j (the first leaf of its right subtree), depth = distance from the
// root.  Nodes are appended in creation order, children before parents.
struct HostTree {
  int64_t r = 0;
  uint32_t leaf_base = 0;
  std::vector<int64_t> start;    // r + 1 leaf starts
  std::vector<int32_t> first, last;  // per unified id: first / last leaf (nodes: index j)
  std::vector<int32_t> na, nb;   // [j] leaf range
  std::vector<uint32_t> child;   // [2j + side]
  std::vector<uint32_t> order;   // internal nodes in creation order
  uint64_t max_stack = 0;
  void init(int64_t r_, uint32_t lb) {
    r = r_;
    leaf_base = lb;
    na.assign(r, 0);
    nb.assign(r, 0);
    child.assign(2 * (size_t)r, 0);
    order.clear();
  }
  int32_t lfirst(uint32_t id) const { return id >= leaf_base ? (int32_t)(id - leaf_base) : na[id]; }
  int32_t llast(uint32_t id) const { return id >= leaf_base ? (int32_t)(id - leaf_base) : nb[id]; }
  uint32_t join(uint32_t lid, uint32_t rid) {  // merge two adjacent subtrees
    uint32_t j = (uint32_t)lfirst(rid);
    na[j] = lfirst(lid);
    nb[j] = llast(rid);
    child[2 * (size_t)j] = lid;
    child[2 * (size_t)j + 1] = rid;
    order.push_back(j);
    return j;
  }
};

// sorters.py:524-552: ranges of <= w elements are leaves, others split at the midpoint
void build_top_down(HostTree& H, int64_t n, int w) {
  H.start.clear();
  std::vector<std::pair<int64_t, int64_t>> leaves;
  // leaves in order (iterative DFS, left first)
  std::vector<std::pair<int64_t, int64_t>> stk{{0, n - 1}};
  while (!stk.empty()) {
    auto [l, r] = stk.back();
    stk.pop_back();
    if (r - l + 1 <= w) { leaves.push_back({l, r}); continue; }
    int64_t m = l + (r - l) / 2;
    stk.push_back({m + 1, r});
    stk.push_back({l, m});
  }
  H.init((int64_t)leaves.size(), H.leaf_base);
  for (auto& lr : leaves) H.start.push_back(lr.first);
  H.start.push_back(n);
  // joins bottom-up: recurse again over positions, mapping ranges to leaf ids
  std::function<uint32_t(int64_t, int64_t, int64_t&)> rec = [&](int64_t l, int64_t r, int64_t& next) -> uint32_t {
    if (r - l + 1 <= w) return H.leaf_base + (uint32_t)(next++);
    int64_t m = l + (r - l) / 2;
    uint32_t a = rec(l, m, next);
    uint32_t b = rec(m + 1, r, next);
    return H.join(a, b);
  };
  int64_t next = 0;
  rec(0, n - 1, next);
}

// sorters.py:555-581: chunks of w, then passes merging block pairs of width w, 2w, ...
void build_bottom_up(HostTree& H, int64_t n, int w) {
  int64_t r = (n + w - 1) / w;
  H.init(r, H.leaf_base);
  H.start.resize(r + 1);
  for (int64_t k = 0; k < r; ++k) H.start[k] = k * w;
  H.start[r] = n;
  std::vector<uint32_t> cur(r);
  for (int64_t k = 0; k < r; ++k) cur[k] = H.leaf_base + (uint32_t)k;
  for (int64_t width = w; width < n; width *= 2) {
    int64_t nb = (int64_t)cur.size();
    std::vector<uint32_t> nxt;
    for (int64_t k = 0; k < nb; k += 2) {
      if (k + 1 < nb) nxt.push_back(H.join(cur[k], cur[k + 1]));
      else nxt.push_back(cur[k]);
    }
    cur.swap(nxt);
  }
}

// sorters.py:587-635 over the leaf lengths (runs already detected and extended)
void build_alpha(HostTree& H, const std::vector<int64_t>& starts, double alpha, bool pre_push) {
  int64_t r = (int64_t)starts.size() - 1;
  H.init(r, H.leaf_base);
  H.start = starts;
  struct E { uint32_t id; int64_t len; };
  std::vector<E> st;
  uint64_t hmax = 0;
  for (int64_t i = 0; i < r; ++i) {
    int64_t len = starts[i + 1] - starts[i];
    auto merge_top_two = [&]() {
      E b = st.back(); st.pop_back();
      E a = st.back(); st.pop_back();
      st.push_back({H.join(a.id, b.id), a.len + b.len});
    };
    if (pre_push)
      while (st.size() >= 2 && st.back().len < len) merge_top_two();
    st.push_back({H.leaf_base + (uint32_t)i, len});
    while (st.size() >= 2 && (double)st[st.size() - 2].len < alpha * (double)st.back().len) merge_top_two();
    if (st.size() > hmax) hmax = st.size();
  }
  // cleanup: merge the stack bottom-up, left to right
  while (st.size() >= 2) {
    E a = st[0], b = st[1];
    st.erase(st.begin(), st.begin() + 2);
    st.insert(st.begin(), E{H.join(a.id, b.id), a.len + b.len});
  }
  H.max_stack = hmax;
}

// Depths (root = 0) and the workspace arrays; uploads on `st`.  A forest is
// allowed: every parentless node or leaf is a root at depth 0 (writes buf[0]).
// Boundaries that are not nodes of this tree get an empty span and an
// unfusable leaf range, which classification turns into a class-2 node with
// zero tiles: no task, no merge cost, no comparisons.  `leaf_info` (r entries)
// replaces the leaf table when given (write_leaves).
int upload_tree(const HostTree& H, const WsView& V, const Layout& L, cudaStream_t st, bool write_leaves,
                const std::vector<uint32_t>* leaf_info = nullptr) {
  int64_t r = H.r;
  std::vector<uint8_t> depth(r > 0 ? r : 1, 0), ldepth(r, 0);
  std::vector<int32_t> parent(L.leaf_base + r, -1);
  std::vector<pos_t> ns(r, 0), ne(r, 0);
  std::vector<int32_t> na(H.na), nb(H.nb);
  std::vector<uint8_t> is_node(r > 0 ? r : 1, 0);
  for (int64_t k = (int64_t)H.order.size() - 1; k >= 0; --k) {  // parents before children
    uint32_t j = H.order[k];
    int d = parent[j] < 0 ? 0 : depth[parent[j]] + 1;
    if (d > 63) return fail(RS_EUNSUPPORTED, "merge tree deeper than 63 levels");
    depth[j] = (uint8_t)d;
    is_node[j] = 1;
    ns[j] = H.start[H.na[j]];
    ne[j] = H.start[H.nb[j] + 1];
    for (int side = 0; side < 2; ++side) {
      uint32_t c = H.child[2 * (size_t)j + side];
      parent[c] = (int32_t)j;
      if (c >= H.leaf_base) ldepth[c - H.leaf_base] = (uint8_t)(d + 1);
    }
  }
  for (int64_t j = 1; j < r; ++j)
    if (!is_node[j]) {
      na[j] = 0;
      nb[j] = 0x3fffffff;  // more internal nodes than any fused subtree holds
    }
  if (write_leaves) {
    std::vector<uint32_t> info1(leaf_info ? 0 : r, 1u);  // natural run of length 1: insertion sort from one presorted element
    const std::vector<uint32_t>& info = leaf_info ? *leaf_info : info1;
    RS_CUDA(cudaMemcpyAsync(V.leaf_start, H.start.data(), (r + 1) * sizeof(pos_t), cudaMemcpyHostToDevice, st));
    RS_CUDA(cudaMemcpyAsync(V.leaf_info, info.data(), r * sizeof(uint32_t), cudaMemcpyHostToDevice, st));
  }
  RS_CUDA(cudaMemcpyAsync(V.leaf_depth, ldepth.data(), r, cudaMemcpyHostToDevice, st));
  RS_CUDA(cudaMemcpyAsync(V.depth, depth.data(), r, cudaMemcpyHostToDevice, st));
  RS_CUDA(cudaMemcpyAsync(V.node_a, na.data(), r * sizeof(int32_t), cudaMemcpyHostToDevice, st));
  RS_CUDA(cudaMemcpyAsync(V.node_b, nb.data(), r * sizeof(int32_t), cudaMemcpyHostToDevice, st));
  RS_CUDA(cudaMemcpyAsync(V.node_s, ns.data(), r * sizeof(pos_t), cudaMemcpyHostToDevice, st));
  RS_CUDA(cudaMemcpyAsync(V.node_e, ne.data(), r * sizeof(pos_t), cudaMemcpyHostToDevice, st));
  RS_CUDA(cudaMemcpyAsync(V.parent, parent.data(), parent.size() * sizeof(int32_t), cudaMemcpyHostToDevice, st));
  RS_CUDA(cudaMemcpyAsync(V.child, H.child.data(), H.child.size() * sizeof(uint32_t), cudaMemcpyHostToDevice, st));
  RS_CUDA(cudaStreamSynchronize(st));  // the host vectors go out of scope
  return RS_OK;
}

// Classification + ordered task list for the tree in the workspace, then the executor.
template <typename K, int TB>
int exec_tree(K* keys, void* tags, int64_t n, int w, int classic, int no_detect, int fixed, const WsView& V,
              const Layout& L, int sms, cudaStream_t st) {
  int msuper = merge_super<K, TB>(n, sms);
  // top-down / bottom-up: no run detection term, merges counted at run time, no
  // fused subtrees (their merges may be skipped); alpha sorts: powersort's accounting
  ClassifyArgs CA = classify_args<K, TB>(V, L, n, w, classic, msuper, no_detect, fixed, fixed ? 0 : -1);
  size_t sm = (size_t)kFillSmem + 64;
  int occ;
  if (int e = occupancy((const void*)k_tree_tasks, 256, sm, sm, &occ, "task-list kernel")) return e;
  uint32_t* cd = V.chunkdep;
  void* kargs[] = {&CA, &cd};
  RS_CUDA(cudaLaunchCooperativeKernel((void*)k_tree_tasks, dim3(sms * occ), dim3(256), kargs, sm, st));
  prof_mark(1, st);
  return launch_exec<K, TB>(keys, tags, n, w, classic, msuper, V, L, sms, st, fixed);
}

// Alpha-stack / alpha-merge trees can be arbitrarily deep (increasing run
// lengths chain every run into one left spine: depth = runs - 1), while the
// executor orders its tasks in kMaxDepth depth buckets.  Such trees run in
// passes over height bands: pass p merges the nodes of height in
// (62(p-1), 62p], every maximal subtree of height <= 62p being a root of the
// pass's forest, with the previous pass's subtrees -- sorted, in place in
// buf[0] -- as its leaves (natural runs, no detection term).  Every node is
// merged once with the same children as in one pass, so the output, the merge
// cost and the comparisons are the single-pass ones.
template <typename K, int TB>
int run_deep_tree(const HostTree& H, K* keys, void* tags, int64_t n, int w, int classic, const WsView& V,
                  const Layout& L, int sms, cudaStream_t st) {
  const int64_t r = H.r;
  const uint32_t lb = H.leaf_base;
  std::vector<int32_t> h(r, 0), par(r, -1), lpar(r, -1);
  auto height = [&](uint32_t id) { return id >= lb ? 0 : h[id]; };
  for (uint32_t j : H.order) {
    uint32_t c0 = H.child[2 * (size_t)j], c1 = H.child[2 * (size_t)j + 1];
    h[j] = 1 + std::max(height(c0), height(c1));
    for (uint32_t c : {c0, c1}) (c >= lb ? lpar[c - lb] : par[c]) = (int32_t)j;
  }
  const int32_t band = 62;
  const int32_t hroot = H.order.empty() ? 0 : h[H.order.back()];
  for (int32_t p = 1; (int64_t)band * (p - 1) < hroot; ++p) {
    const int32_t W0 = band * (p - 1), W1 = band * p;
    // units (this pass's leaves): maximal subtrees of height <= W0, by first leaf
    std::vector<int32_t> first;
    for (int64_t i = 0; i < r; ++i)
      if (p == 1 || lpar[i] < 0 || h[lpar[i]] > W0) first.push_back((int32_t)i);
    if (p > 1)
      for (uint32_t j : H.order)
        if (h[j] <= W0 && (par[j] < 0 || h[par[j]] > W0)) first.push_back(H.na[j]);
    std::sort(first.begin(), first.end());
    const int64_t R = (int64_t)first.size();
    std::vector<int32_t> unit(r);
    for (int64_t k = 0, i = 0; i < r; ++i) {
      while (k + 1 < R && first[k + 1] <= i) ++k;
      unit[i] = (int32_t)k;
    }
    HostTree P;
    P.leaf_base = lb;
    P.init(R, lb);
    P.start.resize(R + 1);
    std::vector<uint32_t> info(R);
    for (int64_t k = 0; k < R; ++k) {
      P.start[k] = H.start[first[k]];
      int64_t len = (k + 1 < R ? H.start[first[k + 1]] : n) - P.start[k];
      info[k] = (uint32_t)std::min<int64_t>(len, w);  // a natural run: no insertion sort
    }
    P.start[R] = n;
    auto pid = [&](uint32_t id) -> uint32_t {
      if (id >= lb) return lb + (uint32_t)unit[id - lb];
      if (h[id] <= W0) return lb + (uint32_t)unit[H.na[id]];
      return (uint32_t)unit[id];  // a node of this pass: the boundary at its right child's first leaf
    };
    for (uint32_t j : H.order)
      if (h[j] > W0 && h[j] <= W1) {
        uint32_t got = P.join(pid(H.child[2 * (size_t)j]), pid(H.child[2 * (size_t)j + 1]));
        if (got != (uint32_t)unit[j]) return fail(RS_EINVARIANT, "deep-tree pass: node boundary mismatch");
      }
    if (p > 1) {  // keep the counters, reset the scheduling state
      DevMetrics hm;
      RS_CUDA(cudaMemcpyAsync(&hm, V.met, sizeof(DevMetrics), cudaMemcpyDeviceToHost, st));
      RS_CUDA(cudaStreamSynchronize(st));
      if (hm.error) return fail(RS_EINVARIANT, "device invariant failure");
      DevMetrics z;
      memset(&z, 0, sizeof z);
      z.merge_cost = hm.merge_cost;
      z.comparisons = hm.comparisons;
      z.runs_detected = hm.runs_detected;
      z.max_stack_height = hm.max_stack_height;
      z.n_leaves = (unsigned long long)R;
      RS_CUDA(cudaMemcpyAsync(V.met, &z, sizeof z, cudaMemcpyHostToDevice, st));
      RS_CUDA(cudaMemsetAsync(V.done, 0, (2 * L.r_max + 2) * sizeof(uint32_t), st));
      int64_t nch_max = (L.r_max + kOrdChunkMin - 1) / kOrdChunkMin;
      RS_CUDA(cudaMemsetAsync(V.chunkdep, 0, (nch_max + 1) * kMaxDepth * sizeof(uint32_t), st));
    }
    if (int e = upload_tree(P, V, L, st, p > 1, &info)) return e;
    if (int e = exec_tree<K, TB>(keys, tags, n, w, classic, p > 1 ? 1 : 0, 0, V, L, sms, st)) return e;
  }
  return RS_OK;
}

template <typename K, int TB>
int run_baseline(int algo, K* keys, void* tags, int64_t n, int w, int classic, double alpha, unsigned char* ws,
                 const Layout& L, cudaStream_t st) {
  int sms;
  if (int e = device_sms(&sms)) return e;
  WsView V = view(ws, L);
  HostTree H;
  H.leaf_base = L.leaf_base;
  const bool fixed = algo == RS_ALGO_TOP_DOWN || algo == RS_ALGO_BOTTOM_UP;
  if (fixed) {
    prof_mark(0, st);
    prof_set_met(V.met);
    RS_CUDA(cudaMemsetAsync(V.met, 0, sizeof(DevMetrics), st));
    RS_CUDA(cudaMemsetAsync(V.done, 0, (2 * L.r_max + 2) * sizeof(uint32_t), st));
    int64_t nch_max = (L.r_max + kOrdChunkMin - 1) / kOrdChunkMin;
    RS_CUDA(cudaMemsetAsync(V.chunkdep, 0, (nch_max + 1) * kMaxDepth * sizeof(uint32_t), st));
    if (algo == RS_ALGO_TOP_DOWN) build_top_down(H, n, w);
    else build_bottom_up(H, n, w);
    if (H.r > L.r_max) return fail(RS_EINVARIANT, "baseline tree exceeds the leaf bound");
    uint64_t r64 = (uint64_t)H.r;
    RS_CUDA(cudaMemcpyAsync(&V.met->n_leaves, &r64, 8, cudaMemcpyHostToDevice, st));
    if (int e = upload_tree(H, V, L, st, true)) return e;
  } else {
    // runs detected and extended exactly like powersort (sorters.py:595-604)
    if (int e = run_powersort<K, TB>(keys, tags, n, w, classic, ws, L, st, 1)) return e;
    DevMetrics hm;
    RS_CUDA(cudaMemcpyAsync(&hm, V.met, sizeof(DevMetrics), cudaMemcpyDeviceToHost, st));
    RS_CUDA(cudaStreamSynchronize(st));
    if (hm.error) return fail(RS_EINVARIANT, "device invariant failure (leaf count exceeded bound)");
    std::vector<int64_t> starts(hm.n_leaves + 1);
    RS_CUDA(cudaMemcpyAsync(starts.data(), V.leaf_start, starts.size() * sizeof(int64_t), cudaMemcpyDeviceToHost, st));
    RS_CUDA(cudaStreamSynchronize(st));
    build_alpha(H, starts, alpha, algo == RS_ALGO_ALPHA_MERGE);
    RS_CUDA(cudaMemcpyAsync(&V.met->max_stack_height, &H.max_stack, 8, cudaMemcpyHostToDevice, st));
    int deepest = 0;
    {
      std::vector<int32_t> hh(H.r > 0 ? H.r : 1, 0);
      for (uint32_t j : H.order) {
        uint32_t c0 = H.child[2 * (size_t)j], c1 = H.child[2 * (size_t)j + 1];
        hh[j] = 1 + std::max(c0 >= H.leaf_base ? 0 : hh[c0], c1 >= H.leaf_base ? 0 : hh[c1]);
      }
      if (!H.order.empty()) deepest = hh[H.order.back()] - 1;  // depth of the deepest node
    }
    if (deepest > 63) return run_deep_tree<K, TB>(H, keys, tags, n, w, classic, V, L, sms, st);
    if (int e = upload_tree(H, V, L, st, false)) return e;
  }
  return exec_tree<K, TB>(keys, tags, n, w, classic, fixed ? 1 : 0, fixed ? 1 : 0, V, L, sms, st);
}

template <typename K, int TB>
int run_peeksort(K* keys, void* tags, int64_t n, int w, int classic, unsigned char* ws, const Layout& L,
                 cudaStream_t st) {
  int sms;
  if (int e = device_sms(&sms)) return e;
  WsView V = view(ws, L);
  prof_mark(0, st);
  prof_set_met(V.met);
  auto at = [&](size_t o) { return ws + o; };
  PeekArgs PK;
  PK.keys = keys;
  PK.tags = tags;
  PK.tag_bytes = TB;
  PK.n = n;
  PK.w = w;
  PK.ascw = V.ascw;
  PK.no_zero = reinterpret_cast<uint32_t*>(at(L.o_nozero));
  PK.no_one = reinterpret_cast<uint32_t*>(at(L.o_noone));
  PK.front[0] = reinterpret_cast<PeekItem*>(at(L.o_front0));
  PK.front[1] = reinterpret_cast<PeekItem*>(at(L.o_front1));
  PK.front_cap = L.front_cap;
  PK.nodes = reinterpret_cast<pos_t*>(at(L.o_pnodes));
  PK.leaves = reinterpret_cast<pos_t*>(at(L.o_pleaves));
  PK.revs = reinterpret_cast<pos_t*>(at(L.o_prevs));
  PK.rec_cap = L.rec_cap;
  PK.lbits = reinterpret_cast<uint32_t*>(at(L.o_lbits));
  PK.wpre = reinterpret_cast<uint32_t*>(at(L.o_wpre));
  PK.chunk = reinterpret_cast<uint32_t*>(at(L.o_wchunk));
  PK.words = L.words;
  PK.T = tree_arrays(V, L);
  int msuper = merge_super<K, TB>(n, sms);
  PK.CA = classify_args<K, TB>(V, L, n, w, classic, msuper, 1);
  int64_t nch_max = (L.r_max + kOrdChunkMin - 1) / kOrdChunkMin;
  PK.chunkdep = V.chunkdep;
  PK.chunkdep_words = (nch_max + 1) * kMaxDepth;
  PK.done = V.done;
  PK.done_words = 2 * L.r_max + 2;
  size_t sm = (size_t)kFillSmem + 64;
  int occ;
  if (int e = occupancy((const void*)k_peek<K, TB>, 256, sm, sm, &occ, "peeksort kernel")) return e;
  void* kargs[] = {&PK};
  RS_CUDA(cudaLaunchCooperativeKernel((void*)k_peek<K, TB>, dim3(sms * occ), dim3(256), kargs, sm, st));
  prof_mark(1, st);
  return launch_exec<K, TB>(keys, tags, n, w, classic, msuper, V, L, sms, st);
}

int validate(int algo, int key_dtype, int tag_bytes, int64_t n, int32_t w, int32_t merge_kind, int* kb) {
  if (algo < RS_ALGO_POWERSORT || algo > RS_ALGO_ALPHA_MERGE) return fail(RS_EINVAL, "unknown algorithm");
  if (key_dtype == RS_KEY_I32) *kb = 4;
  else if (key_dtype == RS_KEY_I64) *kb = 8;
  else return fail(RS_EUNSUPPORTED, "keys must be int32 or int64");
  if (tag_bytes != 0 && tag_bytes != 4 && tag_bytes != 8) return fail(RS_EUNSUPPORTED, "tags must be 4 or 8 bytes wide");
  if (n < 0) return fail(RS_EINVAL, "n must be >= 0");
  if (w < 1) return fail(RS_EINVAL, "min_run_len must be >= 1");
  if (merge_kind != RS_MERGE_BITONIC && merge_kind != RS_MERGE_CLASSIC)
    return fail(RS_EINVAL, "merge_kind must be one of ('bitonic', 'classic')");
  if (w > exec_fcap(*kb, tag_bytes))
    return fail(RS_EUNSUPPORTED, "min_run_len exceeds the device path's fused-subtree capacity");
  if (n >= ((int64_t)1 << 40)) return fail(RS_EUNSUPPORTED, "n >= 2^40 is not supported");
  if (algo != RS_ALGO_PEEKSORT && algo != RS_ALGO_TOP_DOWN && algo != RS_ALGO_BOTTOM_UP && n > 1 &&
      prep_smem_bytes(w, *kb, chain_tile_for(n, w, *kb)) > kMaxSmemPerBlock)
    return fail(RS_EUNSUPPORTED, "min_run_len exceeds the run-detection kernel's shared-memory capacity");
  return RS_OK;
}

int read_metrics(const Layout& L, unsigned char* ws, cudaStream_t st, rs_metrics* out) {
  DevMetrics hm;
  RS_CUDA(cudaMemcpyAsync(&hm, ws + L.o_met, sizeof(DevMetrics), cudaMemcpyDeviceToHost, st));
  RS_CUDA(cudaStreamSynchronize(st));
  if (hm.error == kErrPeekCapacity)
    return fail(RS_ECAPACITY, "peeksort replay exceeded the compact workspace (input unchanged): sort again with "
                              "RS_ALGO_PEEKSORT | RS_ALGO_FULL_WS");
  if (hm.error) return fail(RS_EINVARIANT, "device invariant failure (leaf count exceeded bound)");
  if (out) {
    out->merge_cost = hm.merge_cost;
    out->comparisons = hm.comparisons;
    out->runs_detected = hm.runs_detected;
    out->max_stack_height = hm.max_stack_height;
  }
  return RS_OK;
}

int export_tree(const Layout& L, unsigned char* ws, cudaStream_t st, rs_tree* tree) {
  DevMetrics hm;
  RS_CUDA(cudaMemcpyAsync(&hm, ws + L.o_met, sizeof(DevMetrics), cudaMemcpyDeviceToHost, st));
  RS_CUDA(cudaStreamSynchronize(st));
  int64_t r = (int64_t)hm.n_leaves;
  tree->n_leaves = r;
  if (r > tree->capacity) return fail(RS_EINVAL, "tree capacity too small");
  std::vector<int64_t> starts(r + 1);
  RS_CUDA(cudaMemcpyAsync(starts.data(), ws + L.o_leaf_start, (r + 1) * 8, cudaMemcpyDeviceToHost, st));
  std::vector<uint8_t> P(r), D(r);
  if (r > 1) {
    RS_CUDA(cudaMemcpyAsync(P.data(), ws + L.o_P, r, cudaMemcpyDeviceToHost, st));
    RS_CUDA(cudaMemcpyAsync(D.data(), ws + L.o_depth, r, cudaMemcpyDeviceToHost, st));
  }
  RS_CUDA(cudaStreamSynchronize(st));
  for (int64_t i = 0; i < r; ++i)
    if (tree->leaf_len) tree->leaf_len[i] = starts[i + 1] - starts[i];
  for (int64_t j = 1; j < r; ++j) {
    if (tree->node_power) tree->node_power[j - 1] = L.algo == RS_ALGO_POWERSORT ? P[j] : 0;
    if (tree->node_depth) tree->node_depth[j - 1] = D[j];
  }
  return RS_OK;
}

// ------------------------------------------------ sorted runs -> one run
// W sorted runs laid out back to back in one buffer merged in place by the
// executor along a balanced binary tree (log2 W passes of the tuned merge,
// ties to the earlier run).  The NCCL plane of the sharded sort merges its
// received runs this way (dist.py); the runs are natural leaves, so phase A
// has nothing to do except copying depth-1 leaves (W = 2).
int merge_runs_w(int64_t n, int nruns, int kb, int tb) {
  int64_t w = n / (2 * (int64_t)(nruns > 0 ? nruns : 1));
  int64_t cap = exec_fcap(kb, tb);
  if (w > cap) w = cap;
  if (w < 2) w = 2;
  return (int)w;
}

template <typename K, int TB>
int run_merge_runs(K* keys, void* tags, int64_t n, const std::vector<int64_t>& starts, unsigned char* ws,
                   const Layout& L, cudaStream_t st) {
  int sms;
  if (int e = device_sms(&sms)) return e;
  WsView V = view(ws, L);
  const int64_t R = (int64_t)starts.size() - 1;
  if (R > L.r_max) return fail(RS_EINVARIANT, "more runs than the layout holds");
  HostTree H;
  H.leaf_base = L.leaf_base;
  H.init(R, L.leaf_base);
  H.start = starts;
  std::vector<uint32_t> cur(R);
  for (int64_t k = 0; k < R; ++k) cur[k] = L.leaf_base + (uint32_t)k;
  while (cur.size() > 1) {
    std::vector<uint32_t> nxt;
    for (size_t k = 0; k + 1 < cur.size(); k += 2) nxt.push_back(H.join(cur[k], cur[k + 1]));
    if (cur.size() & 1) nxt.push_back(cur.back());
    cur.swap(nxt);
  }
  RS_CUDA(cudaMemsetAsync(V.met, 0, sizeof(DevMetrics), st));
  RS_CUDA(cudaMemsetAsync(V.done, 0, (2 * L.r_max + 2) * sizeof(uint32_t), st));
  int64_t nch_max = (L.r_max + kOrdChunkMin - 1) / kOrdChunkMin;
  RS_CUDA(cudaMemsetAsync(V.chunkdep, 0, (nch_max + 1) * kMaxDepth * sizeof(uint32_t), st));
  uint64_t r64 = (uint64_t)R;
  RS_CUDA(cudaMemcpyAsync(&V.met->n_leaves, &r64, 8, cudaMemcpyHostToDevice, st));
  std::vector<uint32_t> info(R);
  for (int64_t k = 0; k < R; ++k) info[k] = (uint32_t)std::min<int64_t>(starts[k + 1] - starts[k], L.w);  // natural
  if (int e = upload_tree(H, V, L, st, true, &info)) return e;
  return exec_tree<K, TB>(keys, tags, n, L.w, 0, 1, 0, V, L, sms, st);
}

template <typename K>
int dispatch_tags(int algo, K* keys, int tb, void* tags, int64_t n, int w, int classic, double alpha,
                  unsigned char* ws, const Layout& L, cudaStream_t st) {
  if (algo >= RS_ALGO_TOP_DOWN) {
    if (tb == 0) return run_baseline<K, 0>(algo, keys, nullptr, n, w, classic, alpha, ws, L, st);
    if (tb == 4) return run_baseline<K, 4>(algo, keys, tags, n, w, classic, alpha, ws, L, st);
    return run_baseline<K, 8>(algo, keys, tags, n, w, classic, alpha, ws, L, st);
  }
  if (algo == RS_ALGO_PEEKSORT) {
    if (tb == 0) return run_peeksort<K, 0>(keys, nullptr, n, w, classic, ws, L, st);
    if (tb == 4) return run_peeksort<K, 4>(keys, tags, n, w, classic, ws, L, st);
    return run_peeksort<K, 8>(keys, tags, n, w, classic, ws, L, st);
  }
  if (tb == 0) return run_powersort<K, 0>(keys, nullptr, n, w, classic, ws, L, st);
  if (tb == 4) return run_powersort<K, 4>(keys, tags, n, w, classic, ws, L, st);
  return run_powersort<K, 8>(keys, tags, n, w, classic, ws, L, st);
}

// ------------------------------------------------ rs_sort_host helpers
// The calling thread's stream for host-buffer sorts on `dev` (kept).
cudaStream_t host_stream(int dev) {
  thread_local std::vector<cudaStream_t> per_dev;
  if ((int)per_dev.size() <= dev) per_dev.resize(dev + 1, nullptr);
  if (!per_dev[dev] && cudaStreamCreateWithFlags(&per_dev[dev], cudaStreamNonBlocking) != cudaSuccess) {
    per_dev[dev] = nullptr;
  }
  return per_dev[dev];
}

// RS_HOST_TRACE=1: wall-clock phases of rs_sort_host on stderr.
struct HostTrace {
  bool on = tun().host_trace;
  std::chrono::steady_clock::time_point t0 = std::chrono::steady_clock::now(), last = t0;
  std::string line;
  void mark(const char* what) {
    if (!on) return;
    auto t = std::chrono::steady_clock::now();
    char b[96];
    snprintf(b, sizeof b, " %s %.3f", what, std::chrono::duration<double, std::milli>(t - last).count());
    line += b;
    last = t;
  }
  void print(int64_t n) {
    if (!on) return;
    fprintf(stderr, "[rs_sort_host n=%lld total %.3f ms]%s\n", (long long)n,
            std::chrono::duration<double, std::milli>(last - t0).count(), line.c_str());
  }
};

// ------------------------------------------------ cross-GPU merge (rs_kway.cuh)
int load_shards(const rs_shard* shards, int w, int tag_bytes, KwayShards* S) {
  if (w < 1 || w > kKwayMaxW) return fail(RS_EINVAL, "between 1 and 8 shards");
  if (!shards) return fail(RS_EINVAL, "null shard list");
  memset(S, 0, sizeof(*S));
  S->w = w;
  for (int i = 0; i < w; ++i) {
    if (shards[i].hi < shards[i].lo || shards[i].lo < 0) return fail(RS_EINVAL, "shard range must satisfy 0 <= lo <= hi");
    if (shards[i].hi > shards[i].lo && !shards[i].keys) return fail(RS_EINVAL, "null shard keys");
    if (tag_bytes && shards[i].hi > shards[i].lo && !shards[i].tags) return fail(RS_EINVAL, "null shard tags");
    S->keys[i] = shards[i].keys;
    S->tags[i] = shards[i].tags;
    S->lo[i] = shards[i].lo;
    S->hi[i] = shards[i].hi;
  }
  return RS_OK;
}

struct KwayLayout {
  int64_t spacing, npiv, npiv_cap;
  KwayPiv piv;
  size_t o_bounds, o_nitems, o_claim, o_items, o_nitems2, total;
  int64_t kmax;  // item-count bound
};

// out_len: the merged length (the ranges' total); with device-resident ranges
// only it is known on the host, which bounds the pivot count.
template <typename K, int TB>
KwayLayout kway_layout(const KwayShards& S, int64_t out_len, bool dev_ranges, int sms) {
  KwayLayout KL{};
  int64_t M = out_len;
  (void)sms;
  // pivots every `sp` elements of each shard: a work item (between consecutive
  // pivots in global order) holds at most sp elements of each shard, so at most
  // ITEM in all -- it fits the merge kernel's shared-memory buffers
  int64_t sp = KwayCfg<K, TB>::spacing(S.w);
  KL.spacing = sp;
  KL.piv.off[0] = 0;
  if (!dev_ranges) {
    for (int i = 0; i < S.w; ++i) KL.piv.off[i + 1] = KL.piv.off[i] + (S.hi[i] - S.lo[i] + sp - 1) / sp;
    KL.npiv = KL.piv.off[S.w];
    KL.npiv_cap = KL.npiv;
  } else {
    KL.npiv = 0;
    KL.npiv_cap = M / sp + S.w;
  }
  size_t off = 0;
  KL.o_bounds = off;
  off = align_up(off + (size_t)(KL.npiv_cap + 2) * S.w * 8, 256);
  KL.o_nitems = off;
  off = align_up(off + 8, 256);
  KL.o_claim = off;
  off = align_up(off + 8, 256);
  KL.kmax = M / KwayCfg<K, TB>::GROUP + 2;
  KL.o_items = off;
  off = align_up(off + (size_t)(KL.kmax + 1) * 8, 256);
  KL.o_nitems2 = off;
  off = align_up(off + 8, 256);
  KL.total = off + 256;
  return KL;
}

template <typename K, int TB>
int run_kway(const KwayShards& S, const int64_t* dsplit, int64_t out_len, void* out_keys, void* out_tags,
             unsigned char* ws, size_t ws_bytes, cudaStream_t st) {
  int sms;
  if (int e = device_sms(&sms)) return e;
  KwayLayout KL = kway_layout<K, TB>(S, out_len, dsplit != nullptr, sms);
  if (ws_bytes < KL.total) return fail(RS_ENOMEM, "k-way merge workspace too small");
  if (S.w == 1) {  // a copy, no pivots or items
    int g = (int)std::min<int64_t>((out_len + 255) / 256, (int64_t)sms * 8);
    k_kway_copy1<K, TB><<<g > 0 ? g : 1, 256, 0, st>>>(S, dsplit, out_keys, out_tags);
    RS_CUDA(cudaGetLastError());
    return RS_OK;
  }
  int64_t* bounds = reinterpret_cast<int64_t*>(ws + KL.o_bounds);
  int64_t* nitems = reinterpret_cast<int64_t*>(ws + KL.o_nitems);
  unsigned long long* claim = reinterpret_cast<unsigned long long*>(ws + KL.o_claim);
  RS_CUDA(cudaMemsetAsync(claim, 0, 8, st));
  int64_t pw = (KL.npiv_cap > 0 ? KL.npiv_cap : 1) * 32;
  int pgrid = (int)std::min<int64_t>((pw + 255) / 256, (int64_t)sms * 8);
  if (pgrid < 1) pgrid = 1;
  k_kway_pivots<K><<<pgrid, 256, 0, st>>>(S, KL.spacing, KL.piv, KL.npiv, bounds, dsplit, nitems);
  RS_CUDA(cudaGetLastError());
  int64_t* item_rows = reinterpret_cast<int64_t*>(ws + KL.o_items);
  int64_t* nitems2 = reinterpret_cast<int64_t*>(ws + KL.o_nitems2);
  int igrid = (int)std::min<int64_t>((KL.kmax + 255) / 256, (int64_t)sms * 8);
  if (igrid < 1) igrid = 1;
  k_kway_items<<<igrid, 256, 0, st>>>(bounds, S.w, nitems, KwayCfg<K, TB>::GROUP, KL.kmax, item_rows, nitems2);
  RS_CUDA(cudaGetLastError());
  size_t sm = KwayCfg<K, TB>::SMEM;
  int occ;
  if (int e = occupancy((const void*)k_kway_merge<K, TB>, KwayCfg<K, TB>::THREADS, sm, sm, &occ,
                        "k-way merge kernel"))
    return e;
  KwayMergeArgs A;
  A.S = S;
  A.bounds = bounds;
  A.nitems = nitems2;
  A.item_rows = item_rows;
  A.out_keys = out_keys;
  A.out_tags = out_tags;
  A.claim = claim;
  int grid = (int)std::min<int64_t>((int64_t)sms * occ, KL.kmax);
  k_kway_merge<K, TB><<<grid, KwayCfg<K, TB>::THREADS, sm, st>>>(A);
  RS_CUDA(cudaGetLastError());
  return RS_OK;
}

template <int TB>
int kway_dispatch_tb(int key_dtype, const KwayShards& S, const int64_t* dsplit, int64_t M, void* ok, void* ot,
                     unsigned char* ws, size_t wsb, cudaStream_t st) {
  if (key_dtype == RS_KEY_I64) return run_kway<int64_t, TB>(S, dsplit, M, ok, ot, ws, wsb, st);
  return run_kway<int32_t, TB>(S, dsplit, M, ok, ot, ws, wsb, st);
}

int kway_dispatch(int key_dtype, int tag_bytes, const KwayShards& S, const int64_t* dsplit, int64_t M, void* ok,
                  void* ot, unsigned char* ws, size_t wsb, cudaStream_t st) {
  if (tag_bytes == 0) return kway_dispatch_tb<0>(key_dtype, S, dsplit, M, ok, ot, ws, wsb, st);
  if (tag_bytes == 4) return kway_dispatch_tb<4>(key_dtype, S, dsplit, M, ok, ot, ws, wsb, st);
  return kway_dispatch_tb<8>(key_dtype, S, dsplit, M, ok, ot, ws, wsb, st);
}

size_t kway_ws(int key_dtype, int tag_bytes, const KwayShards& S, int64_t M, bool dev_ranges) {
  int sms;
  if (device_sms(&sms)) sms = 148;
  if (key_dtype == RS_KEY_I64) {
    return tag_bytes == 0 ? kway_layout<int64_t, 0>(S, M, dev_ranges, sms).total
                          : (tag_bytes == 4 ? kway_layout<int64_t, 4>(S, M, dev_ranges, sms).total
                                            : kway_layout<int64_t, 8>(S, M, dev_ranges, sms).total);
  }
  return tag_bytes == 0 ? kway_layout<int32_t, 0>(S, M, dev_ranges, sms).total
                        : (tag_bytes == 4 ? kway_layout<int32_t, 4>(S, M, dev_ranges, sms).total
                                          : kway_layout<int32_t, 8>(S, M, dev_ranges, sms).total);
}

}  // namespace

extern "C" {

int rs_corank(int key_dtype, const rs_shard* shards, int w, const int64_t* targets, int ntargets, int64_t* out,
              void* workspace, size_t ws_bytes, void* stream) {
  KwayShards S;
  if (int e = load_shards(shards, w, 0, &S)) return e;
  if (ntargets < 0 || (ntargets > 0 && (!targets || !out))) return fail(RS_EINVAL, "null targets / out");
  if (ntargets == 0) return RS_OK;
  size_t need = (size_t)ntargets * 8 * (1 + w) + 512;
  if (!workspace || ws_bytes < need) return fail(RS_ENOMEM, "co-rank workspace too small");
  int64_t total = 0;
  for (int i = 0; i < w; ++i) total += S.hi[i] - S.lo[i];
  for (int b = 0; b < ntargets; ++b)
    if (targets[b] < 0 || targets[b] > total) return fail(RS_EINVAL, "co-rank target outside [0, total]");
  cudaStream_t st = reinterpret_cast<cudaStream_t>(stream);
  int64_t* dt = reinterpret_cast<int64_t*>(workspace);
  int64_t* dout = reinterpret_cast<int64_t*>(reinterpret_cast<unsigned char*>(workspace) +
                                             align_up((size_t)ntargets * 8, 256));
  RS_CUDA(cudaMemcpyAsync(dt, targets, (size_t)ntargets * 8, cudaMemcpyHostToDevice, st));
  if (key_dtype == RS_KEY_I64) k_corank<int64_t><<<ntargets, kCorankThreads, 0, st>>>(S, dt, dout, nullptr, 0);
  else k_corank<int32_t><<<ntargets, kCorankThreads, 0, st>>>(S, dt, dout, nullptr, 0);
  RS_CUDA(cudaGetLastError());
  RS_CUDA(cudaMemcpyAsync(out, dout, (size_t)ntargets * w * 8, cudaMemcpyDeviceToHost, st));
  RS_CUDA(cudaStreamSynchronize(st));
  return RS_OK;
}

size_t rs_kway_workspace_bytes(int key_dtype, int tag_bytes, const rs_shard* shards, int w) {
  KwayShards S;
  if (load_shards(shards, w, 0, &S)) return 0;
  int64_t M = 0;
  for (int i = 0; i < w; ++i) M += S.hi[i] - S.lo[i];
  return kway_ws(key_dtype, tag_bytes, S, M, false);
}

int rs_kway_merge(int key_dtype, int tag_bytes, const rs_shard* shards, int w, void* out_keys, void* out_tags,
                  void* workspace, size_t ws_bytes, void* stream) {
  KwayShards S;
  if (key_dtype != RS_KEY_I32 && key_dtype != RS_KEY_I64) return fail(RS_EUNSUPPORTED, "keys must be int32 or int64");
  if (tag_bytes != 0 && tag_bytes != 4 && tag_bytes != 8) return fail(RS_EUNSUPPORTED, "tags must be 4 or 8 bytes wide");
  if (int e = load_shards(shards, w, tag_bytes, &S)) return e;
  int64_t M = 0;
  for (int i = 0; i < w; ++i) M += S.hi[i] - S.lo[i];
  if (M == 0) return RS_OK;
  if (!out_keys || (tag_bytes && !out_tags) || !workspace) return fail(RS_EINVAL, "null output or workspace");
  return kway_dispatch(key_dtype, tag_bytes, S, nullptr, M, out_keys, out_tags,
                       reinterpret_cast<unsigned char*>(workspace), ws_bytes, reinterpret_cast<cudaStream_t>(stream));
}

int rs_corank_rank(int key_dtype, const rs_shard* shards, int w, const int64_t* dlens, int rank, int64_t* dsplit,
                   void* stream) {
  KwayShards S;
  if (key_dtype != RS_KEY_I32 && key_dtype != RS_KEY_I64) return fail(RS_EUNSUPPORTED, "keys must be int32 or int64");
  if (w < 1 || w > kKwayMaxW || !shards) return fail(RS_EINVAL, "between 1 and 8 shards");
  if (rank < 0 || rank >= w || !dlens || !dsplit) return fail(RS_EINVAL, "bad rank / null device arrays");
  memset(&S, 0, sizeof(S));
  S.w = w;
  for (int i = 0; i < w; ++i) {
    S.keys[i] = shards[i].keys;
    S.tags[i] = shards[i].tags;
  }
  cudaStream_t st = reinterpret_cast<cudaStream_t>(stream);
  if (key_dtype == RS_KEY_I64) k_corank<int64_t><<<2, kCorankThreads, 0, st>>>(S, nullptr, dsplit, dlens, rank);
  else k_corank<int32_t><<<2, kCorankThreads, 0, st>>>(S, nullptr, dsplit, dlens, rank);
  RS_CUDA(cudaGetLastError());
  return RS_OK;
}

size_t rs_kway_split_workspace_bytes(int key_dtype, int tag_bytes, int w, int64_t out_len) {
  if (w < 1 || w > kKwayMaxW || out_len < 0) return 0;
  KwayShards S;
  memset(&S, 0, sizeof(S));
  S.w = w;
  return kway_ws(key_dtype, tag_bytes, S, out_len, true);
}

int rs_kway_merge_split(int key_dtype, int tag_bytes, const rs_shard* shards, int w, const int64_t* dsplit,
                        int64_t out_len, void* out_keys, void* out_tags, void* workspace, size_t ws_bytes,
                        void* stream) {
  KwayShards S;
  if (key_dtype != RS_KEY_I32 && key_dtype != RS_KEY_I64) return fail(RS_EUNSUPPORTED, "keys must be int32 or int64");
  if (tag_bytes != 0 && tag_bytes != 4 && tag_bytes != 8) return fail(RS_EUNSUPPORTED, "tags must be 4 or 8 bytes wide");
  if (w < 1 || w > kKwayMaxW || !shards || !dsplit) return fail(RS_EINVAL, "between 1 and 8 shards, device split");
  if (out_len == 0) return RS_OK;
  if (!out_keys || (tag_bytes && !out_tags) || !workspace) return fail(RS_EINVAL, "null output or workspace");
  memset(&S, 0, sizeof(S));
  S.w = w;
  for (int i = 0; i < w; ++i) {
    S.keys[i] = shards[i].keys;
    S.tags[i] = shards[i].tags;
  }
  return kway_dispatch(key_dtype, tag_bytes, S, dsplit, out_len, out_keys, out_tags,
                       reinterpret_cast<unsigned char*>(workspace), ws_bytes, reinterpret_cast<cudaStream_t>(stream));
}

int rs_ipc_alloc(size_t bytes, void** ptr, void* handle) {
  if (!ptr || !handle) return fail(RS_EINVAL, "null ptr / handle");
  *ptr = nullptr;
  if (cudaMalloc(ptr, bytes ? bytes : 256) != cudaSuccess) {
    cudaGetLastError();
    return fail(RS_ENOMEM, "cudaMalloc of an IPC-shareable shard buffer failed");
  }
  cudaIpcMemHandle_t h;
  if (cudaError_t e = cudaIpcGetMemHandle(&h, *ptr)) {
    cudaFree(*ptr);
    *ptr = nullptr;
    return fail(RS_ECUDA, std::string("cudaIpcGetMemHandle failed: ") + cudaGetErrorString(e));
  }
  memcpy(handle, &h, sizeof(h));
  return RS_OK;
}

int rs_ipc_open(const void* handle, void** ptr) {
  if (!ptr || !handle) return fail(RS_EINVAL, "null ptr / handle");
  cudaIpcMemHandle_t h;
  memcpy(&h, handle, sizeof(h));
  RS_CUDA(cudaIpcOpenMemHandle(ptr, h, cudaIpcMemLazyEnablePeerAccess));
  return RS_OK;
}

int rs_ipc_close(void* ptr) {
  RS_CUDA(cudaIpcCloseMemHandle(ptr));
  return RS_OK;
}

int rs_ipc_free(void* ptr) {
  RS_CUDA(cudaFree(ptr));
  return RS_OK;
}

size_t rs_workspace_bytes(int algo, int key_dtype, int tag_bytes, int64_t n, int32_t min_run_len) {
  (void)algo;
  int kb = key_dtype == RS_KEY_I64 ? 8 : 4;
  if (n <= 1) return 256;
  if (min_run_len < 1) min_run_len = 1;
  return make_layout(n, min_run_len, kb, tag_bytes, algo).total;
}

int rs_sort(int algo, int key_dtype, void* keys, int tag_bytes, void* tags, int64_t n, int32_t min_run_len,
            int32_t merge_kind, void* workspace, size_t ws_bytes, void* stream, rs_metrics* out, rs_tree* tree) {
  return rs_sort_ex(algo, key_dtype, keys, tag_bytes, tags, n, min_run_len, merge_kind, 2.0, workspace, ws_bytes,
                    stream, out, tree);
}

int rs_sort_ex(int algo, int key_dtype, void* keys, int tag_bytes, void* tags, int64_t n, int32_t min_run_len,
               int32_t merge_kind, double alpha, void* workspace, size_t ws_bytes, void* stream, rs_metrics* out,
               rs_tree* tree) {
  int kb;
  const int algo_ws = algo;  // may carry RS_ALGO_FULL_WS (peeksort's replay capacity)
  algo &= ~RS_ALGO_FULL_WS;
  if (int e = validate(algo, key_dtype, tag_bytes, n, min_run_len, merge_kind, &kb)) return e;
  if (!(alpha > 1.0)) return fail(RS_EINVAL, "alpha must be > 1");
  if (tree && algo >= RS_ALGO_TOP_DOWN) return fail(RS_EUNSUPPORTED, "the baseline sorters record no merge tree");
  if (tags == nullptr) tag_bytes = 0;
  if (n <= 1) {  // sorters.py:445-450 (top-down / bottom-up leave the counters alone, :534/:565)
    if (out) {
      memset(out, 0, sizeof(*out));
      out->runs_detected = (algo == RS_ALGO_TOP_DOWN || algo == RS_ALGO_BOTTOM_UP) ? 0 : (uint64_t)n;
    }
    if (tree) {
      tree->n_leaves = n;
      if (n == 1 && tree->capacity >= 1 && tree->leaf_len) tree->leaf_len[0] = 1;
    }
    return RS_OK;
  }
  if (!keys || !workspace) return fail(RS_EINVAL, "null keys or workspace");
  Layout L = make_layout(n, min_run_len, kb, tag_bytes, algo_ws);
  if (ws_bytes < L.total) return fail(RS_ENOMEM, "workspace too small");
  cudaStream_t st = reinterpret_cast<cudaStream_t>(stream);
  unsigned char* ws = reinterpret_cast<unsigned char*>(workspace);
  int e;
  if (kb == 4) e = dispatch_tags<int32_t>(algo, reinterpret_cast<int32_t*>(keys), tag_bytes, tags, n, min_run_len,
                                        merge_kind, alpha, ws, L, st);
  else e = dispatch_tags<int64_t>(algo, reinterpret_cast<int64_t*>(keys), tag_bytes, tags, n, min_run_len,
                                  merge_kind, alpha, ws, L, st);
  if (e) return e;
  if (out || tree) {
    if ((e = read_metrics(L, ws, st, out))) return e;
    if (tree && (e = export_tree(L, ws, st, tree))) return e;
  }
  return RS_OK;
}

size_t rs_merge_runs_workspace_bytes(int key_dtype, int tag_bytes, int64_t n, int nruns) {
  int kb = key_dtype == RS_KEY_I64 ? 8 : 4;
  if (n <= 1 || nruns <= 1) return 256;
  return make_layout(n, merge_runs_w(n, nruns, kb, tag_bytes), kb, tag_bytes, RS_ALGO_BOTTOM_UP).total;
}

int rs_merge_runs(int key_dtype, void* keys, int tag_bytes, void* tags, int64_t n, const int64_t* run_starts,
                  int nruns, void* workspace, size_t ws_bytes, void* stream) {
  if (key_dtype != RS_KEY_I32 && key_dtype != RS_KEY_I64) return fail(RS_EUNSUPPORTED, "keys must be int32 or int64");
  if (tag_bytes != 0 && tag_bytes != 4 && tag_bytes != 8) return fail(RS_EUNSUPPORTED, "tags must be 4 or 8 bytes wide");
  if (tags == nullptr) tag_bytes = 0;
  if (nruns < 0 || (nruns > 0 && !run_starts)) return fail(RS_EINVAL, "null run starts");
  if (n < 0) return fail(RS_EINVAL, "n must be >= 0");
  std::vector<int64_t> starts;  // non-empty runs only
  for (int k = 0; k < nruns; ++k) {
    if (run_starts[k] < 0 || run_starts[k + 1] < run_starts[k] || run_starts[k + 1] > n)
      return fail(RS_EINVAL, "run starts must be non-decreasing within [0, n]");
    if (run_starts[k + 1] > run_starts[k]) starts.push_back(run_starts[k]);
  }
  if (nruns > 0 && (run_starts[0] != 0 || run_starts[nruns] != n)) return fail(RS_EINVAL, "the runs must cover [0, n)");
  if (starts.size() <= 1) return RS_OK;  // already one run
  starts.push_back(n);
  if (!keys || !workspace) return fail(RS_EINVAL, "null keys or workspace");
  const int kb = key_dtype == RS_KEY_I64 ? 8 : 4;
  // the layout as rs_merge_runs_workspace_bytes sized it (nruns, empty runs included)
  Layout L = make_layout(n, merge_runs_w(n, nruns, kb, tag_bytes), kb, tag_bytes, RS_ALGO_BOTTOM_UP);
  if (ws_bytes < L.total) return fail(RS_ENOMEM, "workspace too small");
  cudaStream_t st = reinterpret_cast<cudaStream_t>(stream);
  unsigned char* ws = reinterpret_cast<unsigned char*>(workspace);
  if (kb == 4) {
    int32_t* k = reinterpret_cast<int32_t*>(keys);
    if (tag_bytes == 0) return run_merge_runs<int32_t, 0>(k, nullptr, n, starts, ws, L, st);
    if (tag_bytes == 4) return run_merge_runs<int32_t, 4>(k, tags, n, starts, ws, L, st);
    return run_merge_runs<int32_t, 8>(k, tags, n, starts, ws, L, st);
  }
  int64_t* k = reinterpret_cast<int64_t*>(keys);
  if (tag_bytes == 0) return run_merge_runs<int64_t, 0>(k, nullptr, n, starts, ws, L, st);
  if (tag_bytes == 4) return run_merge_runs<int64_t, 4>(k, tags, n, starts, ws, L, st);
  return run_merge_runs<int64_t, 8>(k, tags, n, starts, ws, L, st);
}

int rs_fetch_metrics(int algo, int key_dtype, int tag_bytes, int64_t n, int32_t min_run_len, void* workspace,
                     void* stream, rs_metrics* out) {
  (void)algo;
  if (n <= 1) {
    if (out) { memset(out, 0, sizeof(*out)); out->runs_detected = (uint64_t)n; }
    return RS_OK;
  }
  int kb = key_dtype == RS_KEY_I64 ? 8 : 4;
  Layout L = make_layout(n, min_run_len, kb, tag_bytes, algo);
  return read_metrics(L, reinterpret_cast<unsigned char*>(workspace), reinterpret_cast<cudaStream_t>(stream), out);
}

int rs_export_tree(int algo, int key_dtype, int tag_bytes, int64_t n, int32_t min_run_len, void* workspace,
                   void* stream, rs_tree* tree) {
  if (!tree) return fail(RS_EINVAL, "null tree");
  if ((algo & ~RS_ALGO_FULL_WS) != RS_ALGO_POWERSORT && (algo & ~RS_ALGO_FULL_WS) != RS_ALGO_PEEKSORT)
    return fail(RS_EUNSUPPORTED, "the baseline sorters record no merge tree");
  if (n <= 1) {
    tree->n_leaves = n;
    if (n == 1 && tree->capacity >= 1 && tree->leaf_len) tree->leaf_len[0] = 1;
    return RS_OK;
  }
  int kb = key_dtype == RS_KEY_I64 ? 8 : 4;
  Layout L = make_layout(n, min_run_len, kb, tag_bytes, algo);
  unsigned char* ws = reinterpret_cast<unsigned char*>(workspace);
  cudaStream_t st = reinterpret_cast<cudaStream_t>(stream);
  if (tree->capacity == 0) {  // size query: n_leaves only
    DevMetrics hm;
    RS_CUDA(cudaMemcpyAsync(&hm, ws + L.o_met, sizeof(DevMetrics), cudaMemcpyDeviceToHost, st));
    RS_CUDA(cudaStreamSynchronize(st));
    tree->n_leaves = (int64_t)hm.n_leaves;
    return RS_OK;
  }
  return export_tree(L, ws, st, tree);
}

int rs_sort_host(int algo, int key_dtype, void* keys, int tag_bytes, void* tags, int64_t n, int32_t min_run_len,
                 int32_t merge_kind, rs_metrics* out, rs_tree* tree) {
  return rs_sort_host_ex(algo, key_dtype, keys, tag_bytes, tags, n, min_run_len, merge_kind, 2.0, out, tree);
}

int rs_sort_host_ex(int algo, int key_dtype, void* keys, int tag_bytes, void* tags, int64_t n, int32_t min_run_len,
                    int32_t merge_kind, double alpha, rs_metrics* out, rs_tree* tree) {
  int kb;
  int algo_ws = algo;  // may carry RS_ALGO_FULL_WS; set here when the compact peeksort replay overflows
  algo &= ~RS_ALGO_FULL_WS;
  if (int e = validate(algo, key_dtype, tag_bytes, n, min_run_len, merge_kind, &kb)) return e;
  if (!(alpha > 1.0)) return fail(RS_EINVAL, "alpha must be > 1");
  if (tags == nullptr) tag_bytes = 0;
  if (n <= 1) return rs_sort_ex(algo, key_dtype, keys, tag_bytes, tags, n, min_run_len, merge_kind, alpha, nullptr, 0,
                                nullptr, out, tree);
  if (!keys) return fail(RS_EINVAL, "null keys");
  int dev;
  RS_CUDA(cudaGetDevice(&dev));
  Layout L = make_layout(n, min_run_len, kb, tag_bytes, algo_ws);
  size_t ws = L.total;
  HostTrace tr;
  {
    // device scratch comes from the stream-ordered pool; keep freed blocks
    // cached in it instead of returning them to the driver at every sync
    static std::once_flag pool_once[64];
    std::call_once(pool_once[dev & 63], [dev] {
      cudaMemPool_t pool;
      if (cudaDeviceGetDefaultMemPool(&pool, dev) == cudaSuccess) {
        uint64_t thr = UINT64_MAX;
        cudaMemPoolSetAttribute(pool, cudaMemPoolAttrReleaseThreshold, &thr);
      }
    });
  }
  void *dk = nullptr, *dt = nullptr, *dws = nullptr;
  cudaStream_t st = host_stream(dev);
  if (!st) return fail(RS_ECUDA, "stream creation failed");
  int rc = RS_OK;
  host::Session& S = host::session_for(dev);
  std::vector<host::Span> spans;
  do {
    if (cudaMallocAsync(&dk, (size_t)n * kb + 64, st) != cudaSuccess ||
        (tag_bytes && cudaMallocAsync(&dt, (size_t)n * tag_bytes + 64, st) != cudaSuccess) ||
        cudaMallocAsync(&dws, ws, st) != cudaSuccess) {
      cudaGetLastError();
      rc = fail(RS_ENOMEM, "device allocation failed");
      break;
    }
    spans.push_back({reinterpret_cast<unsigned char*>(keys), reinterpret_cast<unsigned char*>(dk), (size_t)n * kb});
    if (tag_bytes)
      spans.push_back({reinterpret_cast<unsigned char*>(tags), reinterpret_cast<unsigned char*>(dt),
                       (size_t)n * tag_bytes});
    if (!S.init((size_t)n * (kb + tag_bytes))) {
      rc = fail(RS_ENOMEM, "pinned staging allocation failed");
      break;
    }
    tr.mark("alloc+init");
    if (!S.h2d(spans, st)) {
      rc = fail(RS_ECUDA, "host-to-device copy failed");
      break;
    }
    tr.mark("h2d queued");
    int d = 0;
    for (;;) {
      rc = rs_sort_ex(algo_ws, key_dtype, dk, tag_bytes, dt, n, min_run_len, merge_kind, alpha, dws, ws, st, nullptr,
                      nullptr);
      if (rc) break;
      tr.mark("sort queued");
      unsigned char* wsp = reinterpret_cast<unsigned char*>(dws);
      d = S.d2h(spans, st, [&]() -> int {
        int e = read_metrics(L, wsp, st, out);  // synchronizes: the sort is complete
        tr.mark("sort done");
        if (!e && tree) e = export_tree(L, wsp, st, tree);
        return e;
      });
      tr.mark("d2h done");
      if (d != RS_ECAPACITY || (algo_ws & RS_ALGO_FULL_WS)) break;
      // peeksort outgrew its compact replay arrays: the device restored the
      // keys and tags, nothing was written back -- sort again, worst-case capacity
      algo_ws |= RS_ALGO_FULL_WS;
      L = make_layout(n, min_run_len, kb, tag_bytes, algo_ws);
      ws = L.total;
      cudaFreeAsync(dws, st);
      dws = nullptr;
      if (cudaMallocAsync(&dws, ws, st) != cudaSuccess) {
        cudaGetLastError();
        rc = fail(RS_ENOMEM, "device allocation failed (peeksort worst-case workspace)");
        break;
      }
    }
    if (rc) break;
    if (d > 0) rc = d;  // the device's verdict (nothing was written back)
    else if (d < 0) rc = fail(RS_ECUDA, "device-to-host copy failed");
  } while (0);
  if (dk) cudaFreeAsync(dk, st);
  if (dt) cudaFreeAsync(dt, st);
  if (dws) cudaFreeAsync(dws, st);
  cudaStreamSynchronize(st);
  tr.mark("freed");
  tr.print(n);
  return rc;
}

int rs_debug_counters(int key_dtype, int tag_bytes, int64_t n, int32_t min_run_len, void* workspace, uint64_t* out,
                      int cap) {
  if (n <= 1 || !workspace || !out) return 0;
  int kb = key_dtype == RS_KEY_I64 ? 8 : 4;
  int da = tun().debug_algo;  // instrumentation: the layout of another algorithm's workspace
  Layout L = make_layout(n, min_run_len, kb, tag_bytes, da >= 0 ? da : RS_ALGO_POWERSORT);
  DevMetrics hm;
  RS_CUDA(cudaDeviceSynchronize());
  RS_CUDA(cudaMemcpy(&hm, reinterpret_cast<unsigned char*>(workspace) + L.o_met, sizeof(DevMetrics),
                     cudaMemcpyDeviceToHost));
  int k = 0;
  for (; k < cap && k < 8; ++k) out[k] = hm.instr[k];
  if (k < cap) out[k++] = hm.n_tasks;
  if (k < cap) out[k++] = hm.phaseA;
  for (int d = 0; d < kMaxDepth && k < cap; ++d) out[k++] = hm.depth_wait[d];
  for (int d = 0; d < kMaxDepth && k < cap; ++d) out[k++] = hm.depth_tiles[d];
  for (int d = 0; d < 16 && k < cap; ++d) out[k++] = hm.prep_ts[d];
  for (int d = 0; d < 16 && k < cap; ++d) out[k++] = hm.prep_arr[d];
  for (int d = 0; d < 32 && k < cap; ++d) out[k++] = hm.prep_dbg[d];
  for (int d = 0; d < 8 && k < cap; ++d) out[k++] = hm.peek[d];
  return k;
}

int32_t rs_max_min_run_len(int key_dtype, int tag_bytes) {
  int kb = key_dtype == RS_KEY_I64 ? 8 : 4;
  int w = exec_fcap(kb, tag_bytes);
  while (w > 1 && prep_smem_bytes(w, kb, 1024) > kMaxSmemPerBlock) --w;  // smallest chain tile
  return w;
}

int rs_profile(int enable) {
  g_prof.on = enable != 0;
  g_prof.recorded = false;
  return RS_OK;
}

int rs_profile_read(double* ms, int cap) {
  if (!g_prof.recorded) return 0;
  if (cudaEventSynchronize(g_prof.ev[kPhases]) != cudaSuccess) return 0;
  int k = 0;
  for (int i = 0; i < kPhases && i < cap; ++i) {
    float t = 0.f;
    cudaEventElapsedTime(&t, g_prof.ev[i], g_prof.ev[i + 1]);
    ms[k++] = t;
  }
  if (k < cap && g_prof.met) {
    unsigned long long v = 0;
    if (cudaMemcpy(&v, &g_prof.met->merge_cost_exec, 8, cudaMemcpyDeviceToHost) == cudaSuccess) ms[k++] = (double)v;
  }
  return k;
}

int rs_load_bin(const char* path, int64_t* n_out, void* dst, int64_t capacity, void* stream) {
  // gen.py:210-236: "<Q" count, then count "<i8" values (this code assumes a
  // little-endian host, as every CUDA host is)
  if (!path || !n_out) return fail(RS_EINVAL, "rs_load_bin: null path or n_out");
  FILE* f = fopen(path, "rb");
  if (!f) return fail(RS_EIO, std::string("rs_load_bin: cannot open ") + path);
  uint64_t count = 0;
  if (fread(&count, 8, 1, f) != 1) {
    fclose(f);
    return fail(RS_EINVAL, std::string("rs_load_bin: missing header in ") + path);
  }
  if (count > (uint64_t)INT64_MAX / 8) {
    fclose(f);
    return fail(RS_EINVAL, "rs_load_bin: element count out of range");
  }
  *n_out = (int64_t)count;
  if (!dst) {
    fclose(f);
    return RS_OK;
  }
  if ((int64_t)count > capacity) {
    fclose(f);
    return fail(RS_EINVAL, "rs_load_bin: file holds more elements than capacity");
  }
  cudaStream_t st = reinterpret_cast<cudaStream_t>(stream);
  const size_t kChunk = (size_t)32 << 20;  // bytes per staging buffer (double-buffered)
  void* stage[2] = {nullptr, nullptr};
  cudaEvent_t ev[2] = {nullptr, nullptr};
  int rc = RS_OK;
  for (int i = 0; i < 2 && rc == RS_OK; ++i) {
    if (cudaMallocHost(&stage[i], kChunk) != cudaSuccess || cudaEventCreateWithFlags(&ev[i], cudaEventDisableTiming) != cudaSuccess)
      rc = fail(RS_ENOMEM, "rs_load_bin: pinned staging allocation failed");
  }
  size_t total = (size_t)count * 8, done = 0;
  int b = 0;
  while (rc == RS_OK && done < total) {
    size_t len = total - done < kChunk ? total - done : kChunk;
    if (cudaEventSynchronize(ev[b]) != cudaSuccess) {  // this buffer's previous copy finished
      rc = fail(RS_ECUDA, "rs_load_bin: event synchronize failed");
      break;
    }
    if (fread(stage[b], 1, len, f) != len) {
      rc = fail(RS_EINVAL, std::string("rs_load_bin: truncated data in ") + path);
      break;
    }
    if (cudaMemcpyAsync(static_cast<unsigned char*>(dst) + done, stage[b], len, cudaMemcpyHostToDevice, st) !=
            cudaSuccess ||
        cudaEventRecord(ev[b], st) != cudaSuccess) {
      rc = fail(RS_ECUDA, "rs_load_bin: host-to-device copy failed");
      break;
    }
    done += len;
    b ^= 1;
  }
  cudaStreamSynchronize(st);
  for (int i = 0; i < 2; ++i) {
    if (ev[i]) cudaEventDestroy(ev[i]);
    if (stage[i]) cudaFreeHost(stage[i]);
  }
  fclose(f);
  return rc;
}

const char* rs_last_error(void) { return g_err.c_str(); }

int rs_version(void) { return 100; }

}  // extern "C"
