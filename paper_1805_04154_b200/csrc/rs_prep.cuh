// rs_prep.cuh -- one cooperative kernel for everything before the executors:
// run detection + min-run chain (rs_chain.cuh), node powers and the merge tree
// (rs_tree.cuh), classification and the ordered task list (rs_exec.cuh).
// Phases are separated by grid-wide barriers instead of ~16 kernel launches.
#pragma once
#include <cooperative_groups.h>

#include "rs_chain.cuh"
#include "rs_exec.cuh"
#include "rs_small.cuh"
#include "rs_tree.cuh"

namespace rs {

struct PrepArgs {
  const void* keys;
  pos_t n;
  int w;
  int F;
  int batch, gbatch, tbatch;
  int64_t ntiles, ngroups, r_max, nchunks;
  uint32_t* ascw;
  uint2* tables;
  uint2* gtab;
  uint32_t* gentry;
  uint64_t* goff;
  uint32_t* tentry;
  uint64_t* toff;
  MC* agg;
  uint32_t* chunkdep;
  int64_t chunkdep_words;
  uint32_t* done;
  int64_t done_words;
  TreeArrays T;
  ClassifyArgs CA;
  SmallJobs jobs;   // small-tree path: job list (rs_small.cuh)
  int leaves_only;  // stop after the leaf phase (alpha-stack sorts build their tree on the host)
};

// CT: positions per chain tile (chain_tile_for(n)), a compile-time constant so
// the tile arithmetic folds (a runtime value measured 3 us slower on cfg2).
template <typename K, int CT>
__global__ void __launch_bounds__(256, 3) k_prep(PrepArgs P) {
  namespace cg = cooperative_groups;
  cg::grid_group grid = cg::this_grid();
  DevMetrics* met = P.CA.met;
#ifdef RS_INSTR
  unsigned long long t_start = globaltimer_ns();
#endif
  const int64_t gtid = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  const int64_t gthreads = (int64_t)gridDim.x * blockDim.x;
  // zero per-call state (visible to everyone after the first grid barrier)
  {
    unsigned long long* m = reinterpret_cast<unsigned long long*>(met);
    for (int64_t i = gtid; i < (int64_t)(sizeof(DevMetrics) / 8); i += gthreads) m[i] = 0;
    for (int64_t i = gtid; i < P.done_words; i += gthreads) P.done[i] = 0;
    for (int64_t i = gtid; i < P.chunkdep_words; i += gthreads) P.chunkdep[i] = 0;
  }
  // 1. pair-type bits + candidate tables (sorters.py:462-470, runcore.py:137-159)
  const K* a = reinterpret_cast<const K*>(P.keys);
  d_scan_tables_tma<K>(a, P.n, P.w, P.ascw, P.tables, P.ntiles, CT, met);
  RS_ARR(met, 1);
  grid.sync();
  RS_TS(met, 1);
#ifdef RS_INSTR
  if (blockIdx.x == 0 && threadIdx.x == 0) met->prep_ts[0] = t_start;
#endif
  // 2. compose tables per group; the last block to finish walks the groups
  for (int64_t g = blockIdx.x; g < P.ngroups; g += gridDim.x) {
    d_group_compose(P.tables, P.ntiles, P.w, P.batch, P.gtab, g);
    __syncthreads();
  }
  if (last_block_done(&met->last_ctr[0]))
    d_group_entries(P.gtab, P.ngroups, P.w, P.gbatch, P.gentry, P.goff, const_cast<pos_t*>(P.T.leaf_start), P.n,
                    P.r_max, met);
  RS_ARR(met, 2);
  grid.sync();
  RS_TS(met, 2);
  // 3. tile entries
  for (int64_t g = blockIdx.x; g < P.ngroups; g += gridDim.x) {
    d_tile_entries(P.tables, P.ntiles, P.w, P.tbatch, P.gentry, P.goff, P.tentry, P.toff, g);
    __syncthreads();
  }
  RS_ARR(met, 3);
  grid.sync();
  RS_TS(met, 3);
  // 4. emit leaves, one warp per chain tile
  {
    int nw = blockDim.x >> 5, wid = threadIdx.x >> 5;
    for (int64_t t = (int64_t)blockIdx.x * nw + wid; t < P.ntiles; t += (int64_t)gridDim.x * nw)
      d_emit_tile(P.ascw, P.n, P.w, P.tentry, P.toff, P.r_max, const_cast<pos_t*>(P.T.leaf_start),
                  const_cast<uint32_t*>(P.T.leaf_info), t, CT);
  }
  RS_ARR(met, 4);
  grid.sync();
  RS_TS(met, 4);
  if (P.leaves_only) return;
  // small trees: phases 5-9 in block 0 alone, out of shared memory (rs_small.cuh)
  // small trees (n < 2^31): phases 5-8 in block 0 out of shared memory, then
  // the whole grid writes the task records (rs_small.cuh)
  if ((int64_t)met->n_leaves <= kSmallR && P.F == 32) {
    extern __shared__ __align__(16) unsigned char smem_prep[];
    if (blockIdx.x == 0) small_tree<256>(P.T, P.CA, smem_prep, P.jobs);
    grid.sync();
    RS_TS(met, 10);
    pdl_trigger();  // k_phaseA may start launching (it waits for this grid)
    small_fill(P.CA, P.jobs, smem_prep);
    return;
  }
  // 5. node powers + ancestor-count scan (chunk aggregates); each direction's last chunk scans them
  d_scan_reduce(P.T.leaf_start, P.n, P.F, const_cast<uint64_t*>(P.T.K), const_cast<uint8_t*>(P.T.P), met, P.agg,
                P.nchunks, &met->last_ctr[3]);
  RS_ARR(met, 5);
  grid.sync();
  RS_TS(met, 5);
  // 6+7. ancestor counts -> max stack height (sorters.py:500-502), and in the
  // same phase on the other blocks: trie ranges, parents, children, spans
  // (independent of the counts; classification derives the depths)
  {
    const int b0 = scan_down_blocks((int64_t)met->n_leaves);
    if (b0 == 0 || (int)blockIdx.x < b0)
      d_scan_down(P.T.P, met, P.agg, P.nchunks, const_cast<uint8_t*>(P.T.la), const_cast<uint8_t*>(P.T.ra));
    d_tree(P.T, P.F, met, b0);
  }
  RS_ARR(met, 7);
  grid.sync();
  RS_TS(met, 7);
  // 8. classification + Metrics closed forms; the last block lays out depths
  d_classify(P.CA, P.chunkdep);
  if (last_block_done(&met->last_ctr[2])) {
    d_task_offsets(met);
    __syncthreads();
    d_order_scan(met, P.chunkdep);
  }
  RS_ARR(met, 8);
  grid.sync();
  RS_TS(met, 8);
  // 9. task records (k_phaseA may start launching: it waits for this grid to complete)
  pdl_trigger();
  d_task_fill(P.CA, P.chunkdep);
  RS_ARR(met, 9);
  grid.sync();
  RS_TS(met, 9);
#ifdef RS_INSTR
  // calibration: the cost of a bare grid barrier
  RS_ARR(met, 10);
  grid.sync();
  RS_TS(met, 10);
  RS_ARR(met, 11);
  grid.sync();
  RS_TS(met, 11);
#endif
}

}  // namespace rs
