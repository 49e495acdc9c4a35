/*
 * runsort_b200.h -- C ABI of the B200 run-adaptive stable mergesort.
 *
 * Drop-in boundary for the reference package's sort entry points
 * (/root/reference/pkg/src/runsort):
 *
 *   powersort(a, cfg, metrics, tags) -> Metrics      sorters.py:430-519
 *   peeksort(a, cfg, metrics, tags)  -> Metrics      sorters.py:146-361
 *   SortConfig(min_run_len, merge_kind, record_tree)  sorters.py:63-87
 *   Metrics(merge_cost, comparisons, runs_detected,
 *           max_stack_height, merge_tree)            runcore.py:40-55
 *
 * The reference is pure Python, so its "FFI" is the Python call itself; a
 * maintainer binds these symbols with ctypes.  Plain C types
 * only: device or host pointers, sizes, an opaque cudaStream_t.
 *
 * Error codes map onto the reference's exceptions:
 *   RS_EINVAL      -> ValueError      (sorters.py:81-87 config validation)
 *   RS_EINVARIANT  -> AssertionError  (sorters.py:481-482, 491-494, 508-509)
 *   RS_ENOMEM      -> MemoryError     (bench.py:125-133 memory guard)
 *   RS_ECUDA       -> RuntimeError
 *   RS_EUNSUPPORTED-> TypeError / NotImplementedError (dtype or size outside
 *                     the device path; never a silent CPU fallback)
 *   RS_EIO         -> OSError         (gen.py:226-236 load_array file errors)
 *   RS_ECAPACITY   -> (handled inside the host entry points: retry with RS_ALGO_FULL_WS)
 */
#ifndef RUNSORT_B200_H
#define RUNSORT_B200_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define RS_OK 0
#define RS_EINVAL 1
#define RS_EINVARIANT 2
#define RS_ENOMEM 3
#define RS_ECUDA 4
#define RS_EUNSUPPORTED 5
#define RS_EIO 6
#define RS_ECAPACITY 7 /* peeksort's compact workspace overflowed; input unchanged: retry with RS_ALGO_FULL_WS */

#define RS_ALGO_POWERSORT 0
#define RS_ALGO_PEEKSORT 1
/* reference baseline sorters (sorters.py:524-660) on the same executor */
#define RS_ALGO_TOP_DOWN 2
#define RS_ALGO_BOTTOM_UP 3
#define RS_ALGO_ALPHA_STACK 4
#define RS_ALGO_ALPHA_MERGE 5
/* Flag or-ed into RS_ALGO_PEEKSORT wherever `algo` is passed (rs_workspace_bytes,
 * rs_sort*, rs_fetch_metrics, rs_export_tree): size peeksort's replay arrays
 * for the worst case of n + 1 recursive calls (~290 bytes per element) instead
 * of the compact default (n / 12 + 4096 calls, ~29 bytes per element, the
 * frontier laid over the scratch buffers).  A sort whose recursion outgrows
 * the compact arrays restores the input on the device and reports
 * RS_ECAPACITY; rs_sort_host* and the Python entry points then sort again with
 * this flag themselves.  Ignored for the other algorithms. */
#define RS_ALGO_FULL_WS 0x100

#define RS_KEY_I32 1
#define RS_KEY_I64 2

#define RS_MERGE_BITONIC 0 /* exactly size comparisons per merge (runcore.py:282-301) */
#define RS_MERGE_CLASSIC 1 /* two-pointer count (runcore.py:304-326) */

/* Per-call counters, same meaning as the reference Metrics fields.  rs_sort
 * reports the values of THIS call; accumulation into a caller-held Metrics
 * (+= for counters, max for the stack height, assignment for peeksort's
 * runs_detected) is the binding's job, as in sorters.py:443-444. */
typedef struct {
  uint64_t merge_cost;
  uint64_t comparisons;
  uint64_t runs_detected;
  uint64_t max_stack_height;
} rs_metrics;

/* Optional merge-tree export for SortConfig.record_tree (opttree.py:60-75).
 * Host buffers of `capacity` entries; the tree is the min-Cartesian tree of
 * node_depth (equivalently of node_power for powersort). */
typedef struct {
  int64_t capacity;    /* in: entries available in each array */
  int64_t n_leaves;    /* out: r */
  int64_t* leaf_len;   /* out: r leaf lengths, left to right */
  uint8_t* node_power; /* out: r-1 node powers (powersort), boundary order */
  uint8_t* node_depth; /* out: r-1 node depths (root = 0), boundary order */
} rs_tree;

/* Device workspace needed by rs_sort (bytes). */
size_t rs_workspace_bytes(int algo, int key_dtype, int tag_bytes, int64_t n, int32_t min_run_len);

/* Sort `n` keys in place on the device, moving the optional `tags` payload
 * (tag_bytes = 0, 4 or 8) in lockstep.  keys/tags/workspace are device
 * pointers; the work is enqueued on `stream` (a cudaStream_t, NULL = legacy
 * default).  When `out` or `tree` is non-NULL the call synchronizes the stream
 * and fills them; otherwise it returns without waiting and rs_fetch_metrics
 * retrieves the counters later. */
int rs_sort(int algo, int key_dtype, void* keys, int tag_bytes, void* tags, int64_t n,
            int32_t min_run_len, int32_t merge_kind, void* workspace, size_t ws_bytes,
            void* stream, rs_metrics* out, rs_tree* tree);

/* rs_sort with the alpha-stack / alpha-merge growth ratio (SortConfig.alpha,
 * sorters.py:73-87; must be > 1).  rs_sort uses alpha = 2.0. */
int rs_sort_ex(int algo, int key_dtype, void* keys, int tag_bytes, void* tags, int64_t n,
               int32_t min_run_len, int32_t merge_kind, double alpha, void* workspace, size_t ws_bytes,
               void* stream, rs_metrics* out, rs_tree* tree);

/* Synchronize `stream` and read the counters of the last rs_sort that used
 * `workspace` (same n / dtypes / min_run_len). */
int rs_fetch_metrics(int algo, int key_dtype, int tag_bytes, int64_t n, int32_t min_run_len,
                     void* workspace, void* stream, rs_metrics* out);

/* Merge-tree export of the last rs_sort that used `workspace` (same algo, n,
 * dtypes, min_run_len), for SortConfig.record_tree when the caller sizes the
 * host arrays by the leaf count r instead of n: call once with
 * tree->capacity == 0 to read r into tree->n_leaves, then again with
 * capacity >= r.  Synchronizes `stream`.  Powersort and peeksort only. */
int rs_export_tree(int algo, int key_dtype, int tag_bytes, int64_t n, int32_t min_run_len, void* workspace,
                   void* stream, rs_tree* tree);

/* Host-buffer entry (what a plain ctypes binding of the reference calls with
 * numpy arrays): device memory from the stream-ordered pool, the arrays copied
 * in and out in 4 MiB chunks through pinned slots by a pool of host threads
 * (host copies overlapped with the DMAs), the sort in between.  Synchronous;
 * the caller's buffers are written only after the device reported success. */
int rs_sort_host(int algo, int key_dtype, void* keys, int tag_bytes, void* tags, int64_t n,
                 int32_t min_run_len, int32_t merge_kind, rs_metrics* out, rs_tree* tree);

/* rs_sort_host with the alpha-stack / alpha-merge growth ratio. */
int rs_sort_host_ex(int algo, int key_dtype, void* keys, int tag_bytes, void* tags, int64_t n,
                    int32_t min_run_len, int32_t merge_kind, double alpha, rs_metrics* out, rs_tree* tree);

/* Per-phase CUDA-event timing of subsequent rs_sort calls on this thread
 * (events recorded on the sort's own stream).  rs_profile_read waits for the
 * last profiled call and writes up to `cap` values: the durations in ms of
 * [0] prep (run detection, min-run chain, merge tree, task list),
 * [1] phase A (fused small subtrees + large-leaf formation), [2] the merge
 * executor, then [3] the number of elements the merge executor merged
 * (its share of merge_cost).  Returns the number of values written. */
int rs_profile(int enable);
int rs_profile_read(double* ms, int cap);

/* Diagnostics: copy up to `cap` executor cycle counters of the last rs_sort
 * that used `workspace` (nonzero only in an RS_INSTR build).  Synchronizes. */
int rs_debug_counters(int key_dtype, int tag_bytes, int64_t n, int32_t min_run_len, void* workspace,
                      uint64_t* out, int cap);

/* Largest min_run_len the device path accepts for this element type (the
 * fused-subtree capacity, lowered for 8-byte keys so that the run-detection
 * kernel's per-warp windows fit in shared memory at every n). */
int32_t rs_max_min_run_len(int key_dtype, int tag_bytes);

/* Input format of the reference's generators (gen.py:210-236 save_array /
 * load_array): a ".bin" file is a little-endian uint64 element count followed
 * by that many little-endian int64 values.  Reads the file straight into device
 * memory (pinned staging, chunked async copies on `stream`; synchronizes before
 * returning).  `*n_out` receives the count; with dst == NULL only the header is
 * read.  RS_EINVAL: truncated / malformed file or count > capacity;
 * RS_EIO: the file cannot be opened. */
int rs_load_bin(const char* path, int64_t* n_out, void* dst, int64_t capacity, void* stream);

/* ---- Arrays that span GPUs ----
 * W <= 8 sorted shards, each given by a device pointer that may be local or a
 * peer GPU's buffer mapped over NVLink (rs_ipc_open), and a range [lo, hi).
 * The global order is (key, shard index, position): the stable order of the
 * shards' concatenation in index order, as the reference's left-wins merges
 * define it (runcore.py:262-263). */
typedef struct {
  const void* keys;
  const void* tags; /* NULL when tag_bytes == 0 */
  int64_t lo, hi;
} rs_shard;

/* Exact co-rank: for each global rank targets[b] in [0, sum(hi - lo)], the
 * split out[b * w + i] = absolute position in shard i such that shard i's
 * elements [lo_i, out[b*w+i]) are exactly the first targets[b] elements of the
 * global order.  Workspace: device memory of >= ntargets * 8 * (1 + w) + 512
 * bytes.  Synchronizes `stream`. */
int rs_corank(int key_dtype, const rs_shard* shards, int w, const int64_t* targets, int ntargets,
              int64_t* out, void* workspace, size_t ws_bytes, void* stream);

/* Stable w-way merge of the shard ranges into out_keys (+ out_tags), length
 * sum(hi - lo), ties to the lower shard index.  Reads the shards through their
 * pointers (peer memory included) and writes the output once.  Asynchronous on
 * `stream`. */
size_t rs_kway_workspace_bytes(int key_dtype, int tag_bytes, const rs_shard* shards, int w);
int rs_kway_merge(int key_dtype, int tag_bytes, const rs_shard* shards, int w, void* out_keys, void* out_tags,
                  void* workspace, size_t ws_bytes, void* stream);

/* The same, fully on the device for the sharded sort (no host round trip
 * between the local sorts and the merge).  rs_corank_rank: shard i is
 * [0, dlens[i]) (dlens: device array of w lengths, e.g. an all-gather result)
 * and dsplit (device, 2 x w) receives the split vectors of rank `rank`'s output
 * range [sum dlens[0..rank), sum dlens[0..rank]) -- row 0 its start, row 1 its
 * end.  rs_kway_merge_split merges the ranges dsplit describes (shards[i].lo/hi
 * are ignored); out_len = the ranges' total length, known to the caller as its
 * own shard length.  Both asynchronous on `stream`. */
int rs_corank_rank(int key_dtype, const rs_shard* shards, int w, const int64_t* dlens, int rank,
                   int64_t* dsplit, void* stream);
size_t rs_kway_split_workspace_bytes(int key_dtype, int tag_bytes, int w, int64_t out_len);
int rs_kway_merge_split(int key_dtype, int tag_bytes, const rs_shard* shards, int w, const int64_t* dsplit,
                        int64_t out_len, void* out_keys, void* out_tags, void* workspace, size_t ws_bytes,
                        void* stream);

/* CUDA IPC for the peer-mapped shards: rs_ipc_alloc allocates `bytes` of device
 * memory and writes its 64-byte IPC handle; another process on the node maps it
 * with rs_ipc_open (peer access enabled lazily) and unmaps with rs_ipc_close;
 * the owner frees with rs_ipc_free. */
int rs_ipc_alloc(size_t bytes, void** ptr, void* handle);
int rs_ipc_open(const void* handle, void** ptr);
int rs_ipc_close(void* ptr);
int rs_ipc_free(void* ptr);

/* Thread-local message for the last non-RS_OK return. */
const char* rs_last_error(void);

/* ABI version (major * 100 + minor). */
int rs_version(void);

/* W sorted runs stored back to back in keys[0, n) (and tags) merged in place
 * into one sorted run, stable (ties to the earlier run): the executor along a
 * balanced binary tree.  run_starts: host, nruns + 1 positions from 0 to n.
 * Used by the NCCL plane of the sharded sort for the runs it received
 * (replaces a W-way merge pass; reference order: runcore.py:262-263 left-wins). */
size_t rs_merge_runs_workspace_bytes(int key_dtype, int tag_bytes, int64_t n, int nruns);
int rs_merge_runs(int key_dtype, void* keys, int tag_bytes, void* tags, int64_t n, const int64_t* run_starts,
                  int nruns, void* workspace, size_t ws_bytes, void* stream);

#ifdef __cplusplus
}
#endif
#endif /* RUNSORT_B200_H */
