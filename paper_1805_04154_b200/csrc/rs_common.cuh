// rs_common.cuh -- shared types and device helpers for the B200 run-adaptive
// mergesort (powersort / peeksort of arXiv 1805.04154).
#pragma once
#include <cstddef>
#include <cstdint>
#include <cuda_runtime.h>

namespace rs {

using pos_t = int64_t;

constexpr int kWarp = 32;
constexpr pos_t kInf = INT64_MAX / 4;

// ---- chain (min-run) phase ----
#ifndef RS_CHAIN_T
#define RS_CHAIN_T 2048
#endif
constexpr int kChainT = RS_CHAIN_T;  // positions per chain tile
constexpr int kChainThreads = 256;
#ifndef RS_CHAIN_GROUP
#define RS_CHAIN_GROUP 64
#endif
constexpr int kChainGroup = RS_CHAIN_GROUP;  // tiles per composition group
constexpr int kTableBatch = 32;    // tables staged into smem per batch

// ---- executor ----
constexpr int kExecThreads = 256;
constexpr int kMaxDepth = 64;      // depth <= max power <= 63

// Task records (u64): [63:62] kind, [61:32] tile index, [31:0] unified node id.
enum TaskKind : uint32_t { kTaskFuse = 0, kTaskLeaf = 1, kTaskMerge = 2 };
__host__ __device__ inline uint64_t make_task(uint32_t kind, uint32_t tile, uint32_t id) {
  return (uint64_t(kind) << 62) | (uint64_t(tile & 0x3fffffffu) << 32) | uint64_t(id);
}
__host__ __device__ inline uint32_t task_kind(uint64_t t) { return uint32_t(t >> 62); }
__host__ __device__ inline uint32_t task_tile(uint64_t t) { return uint32_t(t >> 32) & 0x3fffffffu; }
__host__ __device__ inline uint32_t task_id(uint64_t t) { return uint32_t(t); }

// Merge-task descriptor (48 B, one per merge task, written by the task fill
// next to its record): everything the merge producer needs after its claim in
// one round trip -- node span and split, children, their completion counts
// and buffers -- instead of a chain of dependent lookups.
struct __align__(16) MDesc {
  pos_t s_d;          // span start | node depth << 56   (positions < 2^40)
  pos_t m_cl;         // children split | bit 56 / 57: child 0 / 1 is a merge node (class 2)
  pos_t e;            // span end
  uint32_t c0, c1;    // unified child ids
  uint32_t nd0, nd1;  // children's completion counts (need)
  uint32_t j;         // node id
  uint32_t sk;        // task index within the node
};
constexpr pos_t kMdescPosMask = ((pos_t)1 << 56) - 1;
static_assert(sizeof(MDesc) == 48 && offsetof(MDesc, e) == 16 && offsetof(MDesc, nd0) == 32 &&
                  offsetof(MDesc, sk) == 44, "MDesc layout (store_merge_task writes it as three uint4)");

// Leaf modes for big (non-fused) leaves.
enum LeafMode : int { kLeafNone = 0, kLeafSwap = 1, kLeafRevCopy = 2, kLeafCopy = 3 };

// Device-resident metrics, accumulated with atomics (reference runcore.py:40-55).
constexpr unsigned long long kErrPeekCapacity = 4;  // peeksort's compact replay workspace overflowed (input restored)
struct DevMetrics {
  unsigned long long merge_cost;
  unsigned long long comparisons;
  unsigned long long runs_detected;
  unsigned long long max_stack_height;
  unsigned long long error;       // nonzero: invariant failure (maps to AssertionError); kErrPeekCapacity: RS_ECAPACITY
  unsigned long long n_leaves;    // r
  unsigned long long n_tasks;     // total executor tasks
  unsigned long long task_ctr;    // merge-executor claim counter (starts at phaseA)
  unsigned long long task_ctr_A;  // phase-A claim counter
  unsigned long long phaseA;      // number of phase-A tasks (fuse + leaf tiles)
  unsigned long long cursorA;     // phase-A slot allocator
  unsigned long long max_depth;   // deepest internal node
  unsigned long long n_merge_tasks;
  unsigned long long n_jobs;      // small-tree path: job-list entries (rs_small.cuh)
  unsigned long long merge_cost_exec;  // sum of spans of the nodes merged by the merge executor
  unsigned long long depth_tiles[kMaxDepth];
  unsigned long long depth_base[kMaxDepth];
  unsigned long long depth_cursor[kMaxDepth];
  unsigned long long instr[8];  // RS_INSTR builds: cycle counters (see rs_merge.cuh)
  unsigned long long depth_wait[kMaxDepth];  // RS_INSTR: producer dependency-wait cycles per depth
  unsigned long long prep_ts[16];            // RS_INSTR: globaltimer at each prep phase boundary
  unsigned long long prep_arr[16];           // RS_INSTR: latest block arrival at each prep barrier
  unsigned long long prep_dbg[32];           // RS_INSTR: finer timestamps inside prep phases
  unsigned int last_ctr[8];                  // 'last block done' counters of the prep kernel
  unsigned long long peek[8];                // peeksort replay counters (frontier sizes, records)
  unsigned long long peek_lev;               // peeksort: the level at which block 0 handed the replay to the grid
};

__device__ __forceinline__ unsigned long long globaltimer_ns() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}

// Debug builds (-DRS_DEBUG_CHECKS): device invariant checks that print and trap.
#ifdef RS_DEBUG_CHECKS
#define RS_CHECK(cond, ...)                                                   \
  do {                                                                        \
    if (!(cond)) {                                                            \
      printf("RS_CHECK %s:%d %s | ", __FILE__, __LINE__, #cond);              \
      printf(__VA_ARGS__);                                                    \
      printf("\n");                                                          \
      __trap();                                                               \
    }                                                                         \
  } while (0)
#else
#define RS_CHECK(cond, ...) do { } while (0)
#endif

#ifdef RS_INSTR
#define RS_TS(met, i) do { if (blockIdx.x == 0 && threadIdx.x == 0) (met)->prep_ts[i] = globaltimer_ns(); } while (0)
#define RS_DBG(met, i) do { if (threadIdx.x == 0) atomicMax(&(met)->prep_dbg[i], globaltimer_ns()); } while (0)
#define RS_TSD(met, i) do { if (threadIdx.x == 0) (met)->prep_dbg[i] = globaltimer_ns(); } while (0)
#define RS_ARR(met, i) do { __syncthreads(); if (threadIdx.x == 0) atomicMax(&(met)->prep_arr[i], globaltimer_ns()); } while (0)
#define RS_T0(v) long long v = clock64()
#define RS_ACC(met, i, v) atomicAdd(&(met)->instr[i], (unsigned long long)(clock64() - (v)))
#else
#define RS_TS(met, i)
#define RS_ARR(met, i)
#define RS_DBG(met, i)
#define RS_TSD(met, i)
#define RS_T0(v)
#define RS_ACC(met, i, v)
#endif

// Out-of-line 64-bit divisions: the inline expansion is ~70 instructions per
// call site, and the prep's phases run once per sort from a cold instruction
// cache -- code bytes are latency there.
__device__ __noinline__ uint64_t udiv64(uint64_t a, uint64_t b) { return a / b; }
__device__ __forceinline__ int64_t ceil_div64(int64_t a, int64_t b) {
  return (int64_t)udiv64((uint64_t)(a + b - 1), (uint64_t)b);
}

// Programmatic dependent launch: a kernel launched with the programmatic
// stream-serialization attribute may start while its predecessor finishes;
// pdl_wait() blocks until the predecessor grid has completed and its memory
// is visible, pdl_trigger() lets this grid's dependent start launching.
__device__ __forceinline__ void pdl_wait() { asm volatile("griddepcontrol.wait;" ::: "memory"); }
__device__ __forceinline__ void pdl_trigger() { asm volatile("griddepcontrol.launch_dependents;" ::: "memory"); }

__device__ __forceinline__ int bitlen64(uint64_t x) { return x ? 64 - __clzll((long long)x) : 0; }

template <typename T>
__device__ __forceinline__ T ldcg(const T* p) { return __ldcg(p); }

// Copy `len` elements global -> shared with U independent loads in flight per thread.
template <typename T, int U = 8>
__device__ __forceinline__ void copy_g2s(T* __restrict__ dst, const T* __restrict__ src, int len, int tid,
                                         int nthreads) {
  for (int base = tid; base < len; base += nthreads * U) {
    T v[U];
#pragma unroll
    for (int u = 0; u < U; ++u) {
      int x = base + u * nthreads;
      if (x < len) v[u] = __ldcg(src + x);
    }
#pragma unroll
    for (int u = 0; u < U; ++u) {
      int x = base + u * nthreads;
      if (x < len) dst[x] = v[u];
    }
  }
}

// True (in every thread of the block) for the block that finishes last among
// the grid's blocks on `counter`; that block then sees all others' writes.
__device__ __forceinline__ bool last_block_done(unsigned int* counter) {
  __shared__ bool s_last;
  __syncthreads();
  if (threadIdx.x == 0) {
    __threadfence();
    unsigned prev = atomicAdd(counter, 1u);
    s_last = (prev == gridDim.x - 1);
    if (s_last) __threadfence();
  }
  __syncthreads();
  return s_last;
}

// Publish completion of a CTA's global writes: call after a barrier that all
// writers passed; one thread does release-fence + relaxed add (CUTLASS-style).
__device__ __forceinline__ void release_add_u32(uint32_t* p, uint32_t v) {
  asm volatile("fence.acq_rel.gpu;\n\tred.relaxed.gpu.global.add.u32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}

__device__ __forceinline__ uint32_t ld_relaxed_u32(const uint32_t* p) {
  uint32_t v;
  asm volatile("ld.relaxed.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}
// Turns earlier relaxed loads that observed released values into acquires.
__device__ __forceinline__ void fence_acquire_gpu() { asm volatile("fence.acq_rel.gpu;" ::: "memory"); }

__device__ __forceinline__ uint32_t ld_acquire_u32(const uint32_t* p) {
  uint32_t v;
  asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}

template <typename T>
__device__ __forceinline__ T warp_sum(T v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}
template <typename T>
__device__ __forceinline__ T warp_max(T v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) { T u = __shfl_xor_sync(0xffffffffu, v, o); v = u > v ? u : v; }
  return v;
}

// Block-wide sum into thread 0 (all threads must call). smem: >= 32 slots.
template <typename T>
__device__ __forceinline__ T block_sum(T v, T* smem) {
  v = warp_sum(v);
  int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  __syncthreads();
  if (lane == 0) smem[wid] = v;
  __syncthreads();
  T s = 0;
  if (threadIdx.x == 0)
    for (int i = 0; i < (int)(blockDim.x >> 5); ++i) s += smem[i];
  return s;
}

// Exclusive block scan of u32 counts (all threads call). Returns exclusive prefix;
// *total gets the block total. smem: >= 33 u32.
__device__ __forceinline__ uint32_t block_excl_scan_u32(uint32_t v, uint32_t* smem, uint32_t* total) {
  int lane = threadIdx.x & 31, wid = threadIdx.x >> 5, nw = blockDim.x >> 5;
  uint32_t x = v;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    uint32_t y = __shfl_up_sync(0xffffffffu, x, o);
    if (lane >= o) x += y;
  }
  __syncthreads();
  if (lane == 31) smem[wid] = x;
  __syncthreads();
  if (wid == 0) {
    uint32_t s = lane < nw ? smem[lane] : 0, t = s;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      uint32_t y = __shfl_up_sync(0xffffffffu, t, o);
      if (lane >= o) t += y;
    }
    if (lane < nw) smem[lane] = t - s;
    if (lane == 31) smem[32] = t;
  }
  __syncthreads();
  uint32_t r = smem[wid] + x - v;
  *total = smem[32];
  __syncthreads();
  return r;
}

// Next set bit at position >= p inside a window of B-words held in smem.
// words[q] covers positions base + 32q .. base + 32q + 31; nz[q] = first q' >= q
// with words[q'] != 0 (nwords when none).  Returns kInf when none in window.
__device__ __forceinline__ pos_t next_set_bit(const uint32_t* words, const uint16_t* nz, int nwords,
                                              pos_t base, pos_t p) {
  pos_t rel = p - base;
  if (rel < 0) rel = 0;
  int q = int(rel >> 5);
  if (q >= nwords) return kInf;
  uint32_t wv = words[q] & (0xffffffffu << (rel & 31));
  if (wv) return base + 32 * pos_t(q) + __ffs(wv) - 1;
  if (q + 1 >= nwords) return kInf;
  int q2 = nz[q + 1];
  if (q2 >= nwords) return kInf;
  return base + 32 * pos_t(q2) + __ffs(words[q2]) - 1;
}

// ---- PTX helpers (mbarrier + 1D TMA bulk copies) ----
__device__ __forceinline__ uint32_t smem_addr(const void* p) {
  return (uint32_t)__cvta_generic_to_shared(p);
}
__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_addr(bar)), "r"(count) : "memory");
}
__device__ __forceinline__ void mbar_fence_init() {
  asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
}
__device__ __forceinline__ void mbar_arrive_tx(uint64_t* bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_addr(bar)), "r"(bytes)
               : "memory");
}
__device__ __forceinline__ void mbar_arrive(uint64_t* bar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_addr(bar)) : "memory");
}
__device__ __forceinline__ bool mbar_try_wait(uint64_t* bar, uint32_t parity) {
  uint32_t ok;
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2, %3;\n\t"
      "selp.u32 %0, 1, 0, p;\n\t}"
      : "=r"(ok)
      : "r"(smem_addr(bar)), "r"(parity), "r"(0x989680u)
      : "memory");
  return ok != 0;
}
// Non-blocking probe of a phase.
__device__ __forceinline__ bool mbar_test_wait(uint64_t* bar, uint32_t parity) {
  uint32_t ok;
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "mbarrier.test_wait.parity.shared::cta.b64 p, [%1], %2;\n\t"
      "selp.u32 %0, 1, 0, p;\n\t}"
      : "=r"(ok)
      : "r"(smem_addr(bar)), "r"(parity)
      : "memory");
  return ok != 0;
}
__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity) {
  while (!mbar_try_wait(bar, parity)) {
  }
}
__device__ __forceinline__ void tma_load_1d(void* dst, const void* src, uint32_t bytes, uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
          smem_addr(dst)),
      "l"(src), "r"(bytes), "r"(smem_addr(bar))
      : "memory");
}
// 1D bulk store smem -> global (16B-aligned addresses, size a multiple of 16)
__device__ __forceinline__ void tma_store_1d(void* gdst, const void* ssrc, uint32_t bytes) {
  asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], %2;" ::"l"(gdst), "r"(smem_addr(ssrc)),
               "r"(bytes)
               : "memory");
}
__device__ __forceinline__ void bulk_commit() { asm volatile("cp.async.bulk.commit_group;" ::: "memory"); }
// all committed bulk stores have finished READING shared memory
__device__ __forceinline__ void bulk_wait_read0() { asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory"); }
// all committed bulk stores are complete (writes performed)
__device__ __forceinline__ void bulk_wait0() { asm volatile("cp.async.bulk.wait_group 0;" ::: "memory"); }
// all but the most recent committed group are complete
__device__ __forceinline__ void bulk_wait1() { asm volatile("cp.async.bulk.wait_group 1;" ::: "memory"); }
__device__ __forceinline__ void fence_proxy_async() { asm volatile("fence.proxy.async;" ::: "memory"); }
__device__ __forceinline__ void fence_proxy_async_global() {
  asm volatile("fence.proxy.async.global;" ::: "memory");
}
__device__ __forceinline__ void fence_proxy_async_smem() {
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
}

// Issue the aligned bulk copy covering elements [e0, e1) of `base` (element
// size es) into smem at `dst`; returns bytes and the element offset of e0.
__device__ __forceinline__ uint32_t tma_window(unsigned char* dst, const void* base, pos_t e0, pos_t e1, int es,
                                               uint64_t* bar, int32_t* off) {
  if (e1 <= e0) {
    *off = 0;
    return 0;
  }
  uintptr_t a0 = reinterpret_cast<uintptr_t>(base) + (uintptr_t)e0 * es;
  uintptr_t a1 = reinterpret_cast<uintptr_t>(base) + (uintptr_t)e1 * es;
  uintptr_t g0 = a0 & ~(uintptr_t)15;
  uintptr_t g1 = (a1 + 15) & ~(uintptr_t)15;
  *off = (int32_t)((a0 - g0) / es);
  uint32_t bytes = (uint32_t)(g1 - g0);
  tma_load_1d(dst, reinterpret_cast<const void*>(g0), bytes, bar);
  return bytes;
}

}  // namespace rs
