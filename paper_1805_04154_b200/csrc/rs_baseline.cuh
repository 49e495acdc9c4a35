// rs_baseline.cuh -- the reference's baseline sorters (sorters.py:524-660) on
// the powersort executor: only the merge tree differs.
//
//   top-down   (sorters.py:524-552)  midpoint splits down to ranges of <= w
//   bottom-up  (sorters.py:555-581)  chunks of w, merge passes of doubling width
//   alpha-stack / alpha-merge (sorters.py:587-660)  runs detected and extended
//              exactly as powersort (k_prep phases 1-4), merged by the alpha
//              stack rules
//
// The trees are built on the host from (n, w) -- top-down and bottom-up are
// data-independent -- or from the device-detected leaf lengths (the alpha
// rules are a sequential scan over run lengths only); the leaves' insertion
// sorts, every merge and all Metrics counting run on the device.  Top-down and
// bottom-up spend one comparison per node on the in-order check and skip such
// merges (counted by the executor, k_merge_exec's skipchk); their stable merge
// of an in-order pair is the concatenation, so the output is unchanged.
//
// k_tree_tasks: classification + the ordered task list for a tree already in
// the workspace (the tail of k_prep / k_peek).
#pragma once
#include <cooperative_groups.h>

#include "rs_exec.cuh"

namespace rs {

__global__ void __launch_bounds__(256) k_tree_tasks(ClassifyArgs CA, uint32_t* chunkdep) {
  namespace cg = cooperative_groups;
  cg::grid_group grid = cg::this_grid();
  d_classify(CA, chunkdep);
  if (last_block_done(&CA.met->last_ctr[2])) {
    d_task_offsets(CA.met);
    __syncthreads();
    d_order_scan(CA.met, chunkdep);
  }
  grid.sync();
  pdl_trigger();  // k_phaseA may start launching (it waits for this grid)
  d_task_fill(CA, chunkdep);
}

}  // namespace rs
