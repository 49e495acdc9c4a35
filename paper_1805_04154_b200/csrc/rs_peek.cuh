// rs_peek.cuh -- peeksort on the device (reference sorters.py:146-361).
//
// The reference recursion sort(l, r, e, s, e_desc, s_desc) is replayed level by
// level: every frontier item (one recursive call) is evaluated by one thread,
// emitting its children (the next frontier), its merge node (l, mid, r, depth),
// its leaves and the reversal of a strictly descending probed run.  Scans read
// pair-type bits of the ORIGINAL keys -- a call only scans strictly inside
// (e, s), which no earlier reversal touched -- while the point comparisons at
// the known runs' ends read the keys after the previous level's reversals were
// applied, exactly like the reference (sorters.py:201-303).  Comparison counts
// follow the reference's scalar conventions (sorters.py:180-199).
//
// Afterwards leaves are compacted through a start-position bitmap, merge nodes
// are mapped onto boundary indices, and the powersort machinery (classify ->
// ordered task list -> phase A -> merge executor) runs unchanged on the tree.
#pragma once
#include <cooperative_groups.h>

#include "rs_chain.cuh"
#include "rs_exec.cuh"
#include "rs_tree.cuh"

namespace rs {

struct PeekItem {
  pos_t l, r, e, s;
  uint32_t flags;  // bit0 e_desc, bit1 s_desc, bits 8..15 depth
  uint32_t pad;
};

struct PeekArgs {
  void* keys;
  void* tags;
  int tag_bytes;
  pos_t n;
  int w;
  uint32_t* ascw;      // pair bits of the original keys (n/32 + 2 words)
  uint32_t* no_zero;   // skip summaries (skip_tree_words): level 1 bit q set if ascw[q] == ~0
  uint32_t* no_one;    // level 1 bit q set if ascw[q] == 0
  PeekItem* front[2];  // frontier ping-pong
  int64_t front_cap;
  pos_t* nodes;        // (l, mid, r, depth) x cap
  pos_t* leaves;       // (l, r, npre, depth) x cap
  pos_t* revs;         // (i, j) x cap
  int64_t rec_cap;
  uint32_t* lbits;     // leaf-start bitmap (n/32 + 2 words)
  uint32_t* wpre;      // exclusive prefix popcount per bitmap word
  uint32_t* chunk;     // chunk sums for the word scan
  int64_t words;
  TreeArrays T;
  ClassifyArgs CA;
  uint32_t* chunkdep;
  int64_t chunkdep_words;
  uint32_t* done;
  int64_t done_words;
};

// Extra per-call counters live in the metrics struct's spare fields.
struct PeekCounters {
  unsigned long long front_n[3];
  unsigned long long n_nodes, n_leaves, n_revs;
  // capacity overflow seen while evaluating level L goes to err[(L + 1) & 1],
  // which every thread reads at the top of level L + 1 (two slots, so a fast
  // thread's level-(L+1) overflow cannot reach a slow thread's level-(L+1) read)
  unsigned long long err[2];
};
static_assert(sizeof(PeekCounters) <= sizeof(((DevMetrics*)nullptr)->peek), "PeekCounters live in DevMetrics::peek");

__device__ __forceinline__ uint32_t ascword(const uint32_t* asc, int64_t q, int v) {
  uint32_t x = __ldcg(asc + q);
  return v ? x : ~x;
}

// Skip summaries, kSkipLevels deep: level 1 bit q set iff pair word q has no
// asc == v pair (the word can be skipped); level l bit i set iff level-(l-1)
// word i is all ones.  A run of length L is crossed in O(levels + L / 32^levels)
// loads instead of L / 1024 dependent loads (config 3's runs reach n / 4).
constexpr int kSkipLevels = 4;
struct SkipTree {
  const uint32_t* lv[kSkipLevels + 1];  // lv[1..kSkipLevels]
  int64_t cnt[kSkipLevels + 1];         // words per level
};
__host__ __device__ inline int64_t skip_level_words(int64_t words, int l) {
  int64_t c = words;
  for (int k = 0; k < l; ++k) c = (c + 31) / 32;
  return c;
}
__host__ __device__ inline int64_t skip_tree_words(int64_t words) {
  int64_t t = 0;
  for (int l = 1; l <= kSkipLevels; ++l) t += skip_level_words(words, l);
  return t + 8;
}
__device__ inline SkipTree make_skip_tree(const uint32_t* base, int64_t words) {
  SkipTree S;
  int64_t off = 0;
  S.lv[0] = nullptr;
  S.cnt[0] = words;
  for (int l = 1; l <= kSkipLevels; ++l) {
    S.lv[l] = base + off;
    S.cnt[l] = skip_level_words(words, l);
    off += S.cnt[l];
  }
  return S;
}

// Smallest pair word index >= w that is not skippable (kInf if none).
__device__ int64_t skip_next(const SkipTree& S, int64_t w) {
  int64_t cur = w;
  int lev = 1;
  for (;; ++lev) {
    int64_t i = cur >> 5;
    if (i >= S.cnt[lev]) return kInf;
    uint32_t m = ~__ldcg(S.lv[lev] + i) & (0xffffffffu << (cur & 31));
    if (m) { cur = (i << 5) + __ffs(m) - 1; break; }
    cur = i + 1;
    if (lev == kSkipLevels) {  // top level: linear
      for (;; ++cur) {
        if (cur >= S.cnt[lev]) return kInf;
        uint32_t mt = ~__ldcg(S.lv[lev] + cur);
        if (mt) { cur = (cur << 5) + __ffs(mt) - 1; break; }
      }
      break;
    }
  }
  for (int l = lev - 1; l >= 1; --l) {  // descend: cur is a level-l word with a zero bit
    if (cur >= S.cnt[l]) return kInf;
    uint32_t m = ~__ldcg(S.lv[l] + cur);
    cur = (cur << 5) + __ffs(m) - 1;
  }
  return cur;
}

// Largest pair word index <= w that is not skippable (-1 if none).
__device__ int64_t skip_prev(const SkipTree& S, int64_t w) {
  int64_t cur = w;
  int lev = 1;
  for (;; ++lev) {
    if (cur < 0) return -1;
    int64_t i = cur >> 5;
    int b = int(cur & 31);
    uint32_t m = ~__ldcg(S.lv[lev] + i) & (b == 31 ? 0xffffffffu : ((1u << (b + 1)) - 1));
    if (m) { cur = (i << 5) + 31 - __clz(m); break; }
    cur = i - 1;
    if (lev == kSkipLevels) {
      for (;; --cur) {
        if (cur < 0) return -1;
        uint32_t mt = ~__ldcg(S.lv[lev] + cur);
        if (mt) { cur = (cur << 5) + 31 - __clz(mt); break; }
      }
      break;
    }
  }
  for (int l = lev - 1; l >= 1; --l) {
    uint32_t m = ~__ldcg(S.lv[l] + cur);
    cur = (cur << 5) + 31 - __clz(m);
  }
  return cur;
}

// Smallest k in [p, q) with asc_k == v, else q.
__device__ pos_t next_eq(const uint32_t* asc, const SkipTree& S, pos_t p, pos_t q, int v) {
  if (p >= q) return q;
  int64_t wq = p >> 5;
  uint32_t x = ascword(asc, wq, v) & (0xffffffffu << (p & 31));
  if (!x) {
    ++wq;
    if ((wq << 5) >= q) return q;
    wq = skip_next(S, wq);
    if (wq >= kInf || (wq << 5) >= q) return q;
    x = ascword(asc, wq, v);
  }
  pos_t k = (wq << 5) + __ffs(x) - 1;
  return k < q ? k : q;
}

// Largest k in [lo, p) with asc_k == v, else lo - 1.
__device__ pos_t prev_eq(const uint32_t* asc, const SkipTree& S, pos_t p, pos_t lo, int v) {
  if (p <= lo) return lo - 1;
  pos_t last = p - 1;
  int64_t wq = last >> 5;
  int sh = 31 - int(last & 31);
  uint32_t x = ascword(asc, wq, v) & (0xffffffffu >> sh);
  if (!x) {
    if ((wq << 5) <= lo) return lo - 1;
    wq = skip_prev(S, wq - 1);
    if (wq < 0 || ((wq + 1) << 5) <= lo) return lo - 1;
    x = ascword(asc, wq, v);
  }
  pos_t k = (wq << 5) + 31 - __clz(x);
  return k >= lo ? k : lo - 1;
}

template <typename K>
struct PeekEval {
  const K* a;
  const uint32_t* asc;
  SkipTree no_zero;  // skip words without an asc == 0 pair
  SkipTree no_one;   // skip words without an asc == 1 pair
  unsigned long long comps;

  __device__ bool le(pos_t x, pos_t y) const { return __ldcg(a + x) <= __ldcg(a + y); }
  __device__ bool gt(pos_t x, pos_t y) const { return __ldcg(a + x) > __ldcg(a + y); }
  // sorters.py:180-199 (runcore.py:77-134 semantics on the original keys)
  __device__ pos_t asc_right(pos_t st, pos_t bound) {
    pos_t j = next_eq(asc, no_zero, st, bound, 0);
    comps += (unsigned long long)((j < bound) ? (j - st + 1) : (j - st));
    return j;
  }
  __device__ pos_t desc_right(pos_t st, pos_t bound) {
    pos_t j = next_eq(asc, no_one, st, bound, 1);
    comps += (unsigned long long)((j < bound) ? (j - st + 1) : (j - st));
    return j;
  }
  __device__ pos_t asc_left(pos_t st, pos_t bound) {
    pos_t k = prev_eq(asc, no_zero, st, bound, 0);
    pos_t i = k + 1 > bound ? k + 1 : bound;
    comps += (unsigned long long)((i > bound) ? (st - i + 1) : (st - i));
    return i;
  }
  __device__ pos_t desc_left(pos_t st, pos_t bound) {
    pos_t k = prev_eq(asc, no_one, st, bound, 1);
    pos_t i = k + 1 > bound ? k + 1 : bound;
    comps += (unsigned long long)((i > bound) ? (st - i + 1) : (st - i));
    return i;
  }
  // sorters.py:201-215
  __device__ pos_t extend_prefix(pos_t e, pos_t r, pos_t s, bool e_desc, bool s_desc) {
    if (e_desc || e == r) return e;
    comps += 1;
    if (gt(e, e + 1)) return e;
    if (e + 1 == s) return r;
    pos_t E = asc_right(e + 1, s - 1);
    if (E == s - 1 && !s_desc) {
      comps += 1;
      if (le(s - 1, s)) return r;
    }
    return E;
  }
  // sorters.py:217-231
  __device__ pos_t extend_suffix(pos_t s, pos_t l, pos_t e, bool s_desc, bool e_desc) {
    if (s_desc || s == l) return s;
    comps += 1;
    if (gt(s - 1, s)) return s;
    if (s - 1 == e) return l;
    pos_t S = asc_left(s - 1, e + 1);
    if (S == e + 1 && !e_desc) {
      comps += 1;
      if (le(e, e + 1)) return l;
    }
    return S;
  }
  // sorters.py:233-303; *rev set when [i..j] must be reversed
  __device__ void probe(pos_t m, pos_t l, pos_t r, pos_t e, pos_t s, bool e_desc, bool s_desc, pos_t* pi,
                        pos_t* pj, bool* idesc, bool* jdesc, bool* rev) {
    *rev = false;
    bool asc_r;
    if (m + 1 == s && s_desc) asc_r = false;
    else { comps += 1; asc_r = le(m, m + 1); }
    if (asc_r) {
      pos_t j, i;
      if (m + 1 == s) j = r;
      else {
        j = asc_right(m + 1, s - 1);
        if (j == s - 1 && !s_desc) {
          comps += 1;
          if (le(s - 1, s)) j = r;
        }
      }
      i = asc_left(m, e + 1);
      if (i == e + 1 && !e_desc) {
        comps += 1;
        if (le(e, e + 1)) i = l;
      }
      *pi = i; *pj = j; *idesc = true; *jdesc = true;
      return;
    }
    bool asc_l;
    if (m - 1 == e && e_desc) asc_l = false;
    else { comps += 1; asc_l = le(m - 1, m); }
    if (asc_l) {
      if (m - 1 == e) { *pi = l; *pj = m; *idesc = true; *jdesc = true; return; }
      pos_t i = asc_left(m - 1, e + 1);
      if (i == e + 1 && !e_desc) {
        comps += 1;
        if (le(e, e + 1)) i = l;
      }
      *pi = i; *pj = m; *idesc = true; *jdesc = true;
      return;
    }
    pos_t i, j;
    if (m - 1 > e) {
      i = desc_left(m - 1, e + 1);
      if (i == e + 1 && l == e) {
        if (e_desc) i = l;
        else { comps += 1; if (gt(e, e + 1)) i = l; }
      }
    } else if (l == e) i = l;
    else i = m;
    if (m + 1 == s) j = (s == r) ? r : s;
    else {
      j = desc_right(m + 1, s - 1);
      if (j == s - 1 && s == r) {
        if (s_desc) j = r;
        else { comps += 1; if (gt(s - 1, s)) j = r; }
      }
    }
    *pi = i; *pj = j; *idesc = false; *jdesc = false; *rev = true;
  }
};

struct PeekOut {
  PeekItem* next;
  unsigned long long* next_cnt;
  pos_t* nodes;
  unsigned long long* n_nodes;
  pos_t* leaves;
  unsigned long long* n_leaves;
  pos_t* revs;
  unsigned long long* n_revs;
  int64_t front_cap, rec_cap;
  unsigned long long* err;  // this level's overflow slot (PeekCounters::err)
  DevMetrics* met;
};

// Slot allocation on a shared counter, one atomic per group of converged lanes
// (a wide level has thousands of items hitting the same four counters).
__device__ __forceinline__ unsigned long long agg_inc(unsigned long long* ctr) {
  const unsigned mask = __activemask();
  const int lane = threadIdx.x & 31, leader = __ffs(mask) - 1;
  unsigned long long base = 0;
  if (lane == leader) base = atomicAdd(ctr, (unsigned long long)__popc(mask));
  base = __shfl_sync(mask, base, leader);
  return base + (unsigned long long)__popc(mask & ((1u << lane) - 1u));
}

__device__ __forceinline__ void peek_push(const PeekOut& O, pos_t l, pos_t r, pos_t e, pos_t s, bool ed, bool sd,
                                          uint32_t d) {
  unsigned long long k = agg_inc(O.next_cnt);
  if ((int64_t)k >= O.front_cap) { *O.err = 2; return; }
  PeekItem it;
  it.l = l; it.r = r; it.e = e; it.s = s;
  it.flags = (ed ? 1u : 0u) | (sd ? 2u : 0u) | (d << 8);
  it.pad = 0;
  O.next[k] = it;
}
__device__ __forceinline__ void peek_leaf(const PeekOut& O, pos_t l, pos_t r, pos_t npre, uint32_t d) {
  unsigned long long k = agg_inc(O.n_leaves);
  if ((int64_t)k >= O.rec_cap) { *O.err = 2; return; }
  O.leaves[4 * k] = l; O.leaves[4 * k + 1] = r; O.leaves[4 * k + 2] = npre; O.leaves[4 * k + 3] = d;
}
__device__ __forceinline__ void peek_node(const PeekOut& O, pos_t l, pos_t mid, pos_t r, uint32_t d) {
  unsigned long long k = agg_inc(O.n_nodes);
  if ((int64_t)k >= O.rec_cap) { *O.err = 2; return; }
  O.nodes[4 * k] = l; O.nodes[4 * k + 1] = mid; O.nodes[4 * k + 2] = r; O.nodes[4 * k + 3] = d;
}
__device__ __forceinline__ void peek_rev(const PeekOut& O, pos_t i, pos_t j) {
  if (j <= i) return;
  unsigned long long k = agg_inc(O.n_revs);
  if ((int64_t)k >= O.rec_cap) { *O.err = 2; return; }
  O.revs[2 * k] = i; O.revs[2 * k + 1] = j;
}

// One recursive call (sorters.py:305-349).
template <typename K>
__device__ void peek_item(PeekEval<K>& V, const PeekItem& it, int w, const PeekOut& O) {
  pos_t l = it.l, r = it.r, e = it.e, s = it.s;
  bool e_desc = it.flags & 1u, s_desc = (it.flags >> 1) & 1u;
  uint32_t d = it.flags >> 8;
  if (e == r || s == l) { peek_leaf(O, l, r, r - l + 1, d); return; }
  if (r - l + 1 <= w) { peek_leaf(O, l, r, e - l + 1, d); return; }
  pos_t m = l + (r - l) / 2;
  if (m <= e) {
    pos_t E = V.extend_prefix(e, r, s, e_desc, s_desc);
    if (E == r) { peek_leaf(O, l, r, r - l + 1, d); return; }
    peek_push(O, E + 1, r, E + 1, s, false, s_desc, d + 1);
    peek_leaf(O, l, E, E - l + 1, d + 1);
    peek_node(O, l, E + 1, r, d);
    return;
  }
  if (m >= s) {
    pos_t S = V.extend_suffix(s, l, e, s_desc, e_desc);
    if (S == l) { peek_leaf(O, l, r, r - l + 1, d); return; }
    peek_push(O, l, S - 1, e, S - 1, e_desc, false, d + 1);
    peek_leaf(O, S, r, r - S + 1, d + 1);
    peek_node(O, l, S, r, d);
    return;
  }
  pos_t i, j;
  bool idesc, jdesc, rev;
  V.probe(m, l, r, e, s, e_desc, s_desc, &i, &j, &idesc, &jdesc, &rev);
  if (rev) peek_rev(O, i, j);
  if (i == l && j == r) { peek_leaf(O, l, r, r - l + 1, d); return; }
  if (i + j >= l + r) {  // sorters.py:334, ties go left
    peek_push(O, l, i - 1, e, i - 1, e_desc, false, d + 1);
    if (s > j) peek_push(O, i, r, j, s, jdesc, s_desc, d + 1);
    else peek_push(O, i, r, j, (j + 1 < r ? j + 1 : r), jdesc, false, d + 1);
    peek_node(O, l, i, r, d);
  } else {
    peek_push(O, l, j, e, i, e_desc, idesc, d + 1);
    if (s > j + 1) peek_push(O, j + 1, r, j + 1, s, false, s_desc, d + 1);
    else peek_push(O, j + 1, r, j + 1, j + 1, false, jdesc, d + 1);
    peek_node(O, l, j + 1, r, d);
  }
}

__device__ __forceinline__ int64_t leaf_index(const uint32_t* lbits, const uint32_t* wpre, pos_t p) {
  int64_t q = p >> 5;
  uint32_t mask = (p & 31) ? (0xffffffffu >> (32 - (p & 31))) : 0u;
  return (int64_t)wpre[q] + __popc(lbits[q] & mask);
}

template <typename K, int TB>
__device__ void reverse_segments(const PeekArgs& P, const pos_t* revs, int64_t nrev) {
  using T = typename TagT<TB>::type;
  K* a = reinterpret_cast<K*>(P.keys);
  T* t = reinterpret_cast<T*>(P.tags);
  constexpr int kRevSeg = 64;  // few (long) segments: element-parallel; many: a block per segment
  if (nrev <= kRevSeg) {
    // all blocks share the swaps of every segment (a strictly descending run
    // can be n / 4 long): prefix of half-lengths in shared memory, grid-stride
    // over the swaps, binary search for the segment
    __shared__ pos_t s_pre[kRevSeg + 1];
    __shared__ pos_t s_i[kRevSeg], s_j[kRevSeg];
    for (int64_t q = threadIdx.x; q < nrev; q += blockDim.x) {
      s_i[q] = revs[2 * q];
      s_j[q] = revs[2 * q + 1];
    }
    __syncthreads();
    if (threadIdx.x < 32) {  // warp 0: exclusive scan of the half-lengths, 2 segments per lane
      const int lane = threadIdx.x;
      pos_t h0 = 2 * lane < nrev ? (s_j[2 * lane] - s_i[2 * lane] + 1) / 2 : 0;
      pos_t h1 = 2 * lane + 1 < nrev ? (s_j[2 * lane + 1] - s_i[2 * lane + 1] + 1) / 2 : 0;
      pos_t inc = h0 + h1;
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        pos_t y = __shfl_up_sync(0xffffffffu, inc, o);
        if (lane >= o) inc += y;
      }
      pos_t ex = inc - h0 - h1;
      if (2 * lane < nrev) s_pre[2 * lane] = ex;
      if (2 * lane + 1 < nrev) s_pre[2 * lane + 1] = ex + h0;
      if (lane == 31) s_pre[nrev] = inc;
    }
    __syncthreads();
    const pos_t total = s_pre[nrev];
    for (pos_t x = (pos_t)blockIdx.x * blockDim.x + threadIdx.x; x < total; x += (pos_t)gridDim.x * blockDim.x) {
      int64_t lo = 0, hi = nrev - 1;  // last q with s_pre[q] <= x
      while (lo < hi) {
        int64_t md = (lo + hi + 1) >> 1;
        if (s_pre[md] <= x) lo = md; else hi = md - 1;
      }
      pos_t i = s_i[lo], j = s_j[lo], o = x - s_pre[lo];
      K u = a[i + o], v = a[j - o];
      a[i + o] = v;
      a[j - o] = u;
      if (TB) {
        T tu = t[i + o], tv = t[j - o];
        t[i + o] = tv;
        t[j - o] = tu;
      }
    }
    __syncthreads();
    return;
  }
  // many segments: each block takes whole segments; threads swap pairs
  for (int64_t sidx = blockIdx.x; sidx < nrev; sidx += gridDim.x) {
    pos_t i = revs[2 * sidx], j = revs[2 * sidx + 1];
    pos_t half = (j - i + 1) / 2;
    for (pos_t x = threadIdx.x; x < half; x += blockDim.x) {
      K u = a[i + x], v = a[j - x];
      a[i + x] = v;
      a[j - x] = u;
      if (TB) {
        T tu = t[i + x], tv = t[j - x];
        t[i + x] = tv;
        t[j - x] = tu;
      }
    }
  }
}

constexpr int kWordChunk = 1024;  // bitmap words per scan chunk (a block scans its chunk in blockDim rounds)

template <typename K, int TB>
__global__ void __launch_bounds__(256, 2) k_peek(PeekArgs P) {
  namespace cg = cooperative_groups;
  cg::grid_group grid = cg::this_grid();
  DevMetrics* met = P.CA.met;
  PeekCounters* pc = reinterpret_cast<PeekCounters*>(&met->peek[0]);
  const int64_t gtid = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  const int64_t gthreads = (int64_t)gridDim.x * blockDim.x;
  const K* a = reinterpret_cast<const K*>(P.keys);
  const pos_t n = P.n;
  __shared__ unsigned long long sred[32];
  unsigned long long comps = 0;

  // 0. zero state; pair bits of the original keys (runcore.py:84 / :99 pairs)
  {
    unsigned long long* m = reinterpret_cast<unsigned long long*>(met);
    for (int64_t i = gtid; i < (int64_t)(sizeof(DevMetrics) / 8); i += gthreads) m[i] = 0;
    for (int64_t i = gtid; i < P.done_words; i += gthreads) P.done[i] = 0;
    for (int64_t i = gtid; i < P.chunkdep_words; i += gthreads) P.chunkdep[i] = 0;
    for (int64_t i = gtid; i < P.words; i += gthreads) P.lbits[i] = 0;
    int lane = threadIdx.x & 31;
    int64_t gw = gtid >> 5, nwarps = gthreads >> 5;
    for (int64_t q = gw; q < P.words; q += nwarps) {
      pos_t k = 32 * q + lane;
      bool bit = (k < n - 1) && (a[k] <= a[k + 1]);
      uint32_t wv = __ballot_sync(0xffffffffu, bit);
      if (lane == 0) P.ascw[q] = wv;
    }
  }
  grid.sync();
  {
    int64_t nsw = (P.words + 31) / 32;
    int lane = threadIdx.x & 31;
    int64_t gw = gtid >> 5, nwarps = gthreads >> 5;
    for (int64_t sw = gw; sw < nsw; sw += nwarps) {
      int64_t q = 32 * sw + lane;
      uint32_t x = q < P.words ? P.ascw[q] : 0u;
      uint32_t z = __ballot_sync(0xffffffffu, q < P.words && x == 0xffffffffu);
      uint32_t o = __ballot_sync(0xffffffffu, q >= P.words || x == 0u);
      if (lane == 0) { P.no_zero[sw] = z; P.no_one[sw] = o; }
    }
  }
  // higher skip levels: bit i of level l set iff level-(l-1) word i is all ones
  {
    int lane = threadIdx.x & 31;
    int64_t gw = gtid >> 5, nwarps = gthreads >> 5;
    int64_t off_prev = 0, off = skip_level_words(P.words, 1);
    for (int l = 2; l <= kSkipLevels; ++l) {
      grid.sync();
      int64_t cprev = skip_level_words(P.words, l - 1), c = skip_level_words(P.words, l);
      for (int64_t sw = gw; sw < c; sw += nwarps) {
        int64_t q = 32 * sw + lane;
        bool zf = q < cprev && P.no_zero[off_prev + q] == 0xffffffffu;
        bool of = q < cprev && P.no_one[off_prev + q] == 0xffffffffu;
        uint32_t z = __ballot_sync(0xffffffffu, zf);
        uint32_t o = __ballot_sync(0xffffffffu, of);
        if (lane == 0) { P.no_zero[off + sw] = z; P.no_one[off + sw] = o; }
      }
      off_prev = off;
      off += c;
    }
  }
  grid.sync();
  PeekEval<K> V{a, P.ascw, make_skip_tree(P.no_zero, P.words), make_skip_tree(P.no_one, P.words), 0ull};
  PeekOut O;
  O.nodes = P.nodes;
  O.n_nodes = &pc->n_nodes;
  O.leaves = P.leaves;
  O.n_leaves = &pc->n_leaves;
  O.revs = P.revs;
  O.n_revs = &pc->n_revs;
  O.front_cap = P.front_cap;
  O.rec_cap = P.rec_cap;
  O.met = met;
  if (blockIdx.x == 0) RS_DBG(met, 1);
  // 1. first run (sorters.py:177) and the root call (:351-357)
  O.err = &pc->err[0];
  if (gtid == 0) {
    O.next = P.front[0];
    O.next_cnt = &pc->front_n[0];
    pos_t e0;
    bool desc = false;
    if (n - 1 == 0) e0 = 0;
    else if (a[0] <= a[1]) e0 = V.asc_right(0, n - 1);
    else { e0 = V.desc_right(0, n - 1); desc = true; peek_rev(O, 0, e0); }
    if (e0 == n - 1) peek_leaf(O, 0, n - 1, n, 0);
    else if (n <= P.w) peek_leaf(O, 0, n - 1, e0 + 1, 0);
    else peek_push(O, 0, n - 1, e0, n - 1, !desc, false, 0);
  }
  grid.sync();
  if (blockIdx.x == 0) RS_DBG(met, 2);
  // 2. level-synchronous replay
  // Level L evaluates front[L & 1] (count front_n[L % 3]) and pushes into
  // front[(L+1) & 1] / front_n[(L+1) % 3]; front_n[(L+2) % 3] was last read at
  // level L-1, so thread 0 clears it now and one barrier per level suffices
  // (plus one after a level's reversals, whose keys the next evaluations read).
  // The first levels hold a handful of calls each and are pure latency: block 0
  // replays them alone, one call per thread, with the frontier ping-pong, its
  // counters and the record counters in shared memory (the same peek_item, its
  // PeekOut pointing at shared memory) behind __syncthreads instead of grid
  // barriers, until a level has more calls than the block has threads, a
  // reversal is pending (all blocks share the swaps) or a record array is
  // full.  Then it writes frontier and counters back and the grid continues.
  {
    constexpr int kTopCap = 512;  // calls per shared-memory frontier (a level of <= 256 pushes <= 512)
    extern __shared__ __align__(16) unsigned char smem_peek[];  // k_peek's dynamic shared memory (kFillSmem), free until the task fill
    static_assert(2 * kTopCap * sizeof(PeekItem) <= (size_t)kFillSmem, "shared-memory frontier fits the fill staging area");
    __shared__ unsigned long long s_fn[2], s_nn, s_nl, s_nr, s_err2[2];
    if (blockIdx.x == 0) {
      PeekItem* sf[2] = {reinterpret_cast<PeekItem*>(smem_peek), reinterpret_cast<PeekItem*>(smem_peek) + kTopCap};
      const unsigned long long c0 = *(volatile unsigned long long*)&pc->front_n[0];
      if (threadIdx.x == 0) {
        s_fn[0] = c0;
        s_fn[1] = 0;
        s_nn = pc->n_nodes;
        s_nl = pc->n_leaves;
        s_nr = pc->n_revs;
        s_err2[0] = pc->err[0];
        s_err2[1] = 0;
      }
      for (unsigned long long x = threadIdx.x; x < c0 && x < (unsigned long long)kTopCap; x += blockDim.x) sf[0][x] = P.front[0][x];
      __syncthreads();
      PeekOut T = O;
      T.n_nodes = &s_nn;
      T.n_leaves = &s_nl;
      T.n_revs = &s_nr;
      T.front_cap = kTopCap;
      int tl = 0;
      for (;;) {
        const unsigned long long cnt = s_fn[tl & 1];
        if (cnt == 0 || cnt > (unsigned long long)blockDim.x || s_nr != 0 || s_err2[tl & 1] != 0) break;
        T.next = sf[(tl + 1) & 1];
        T.next_cnt = &s_fn[(tl + 1) & 1];
        T.err = &s_err2[(tl + 1) & 1];
        if (threadIdx.x < cnt) peek_item<K>(V, sf[tl & 1][threadIdx.x], P.w, T);
        __syncthreads();
        if (threadIdx.x == 0) s_fn[tl & 1] = 0;  // this level's slot is the one after next
        ++tl;
        __syncthreads();
      }
      // hand over level tl: frontier, its counters (the next two slots empty), records, errors
      const unsigned long long cnt = s_fn[tl & 1];
      for (unsigned long long x = threadIdx.x; x < cnt; x += blockDim.x) P.front[tl & 1][x] = sf[tl & 1][x];
      if (threadIdx.x == 0) {
        pc->front_n[tl % 3] = cnt;
        pc->front_n[(tl + 1) % 3] = 0;
        pc->front_n[(tl + 2) % 3] = 0;
        pc->n_nodes = s_nn;
        pc->n_leaves = s_nl;
        pc->n_revs = s_nr;
        pc->err[tl & 1] = s_err2[tl & 1];
        pc->err[(tl + 1) & 1] = 0;
        met->peek_lev = (unsigned long long)tl;
      }
    }
    grid.sync();
  }
  int lev = (int)*(volatile unsigned long long*)&met->peek_lev;
  unsigned long long rev_done = 0;
  constexpr int kRevBatches = 256;  // reversal batches (one per level that reversed something)
  __shared__ unsigned long long s_revb[kRevBatches];
  int nbatch = 0;
  for (;;) {
    if (*(volatile unsigned long long*)&pc->err[lev & 1]) {
      // The frontier or a record array is full (compact workspace, rs_workspace_bytes
      // without RS_ALGO_FULL_WS).  Put the keys back as they came -- the
      // reversals applied so far are disjoint strictly descending runs, so
      // reversing them again restores the input -- and leave every task count
      // at zero: phase A and the merge executor find nothing to do, and the
      // host reports RS_ECAPACITY (the caller sorts again with the full workspace).
      // A later level's chain may end on the first element of an earlier
      // level's (reversed) run, so the batches are undone last first; within
      // a level the calls' ranges, hence their reversals, are disjoint.
      __syncthreads();
      for (int b = (nbatch < kRevBatches ? nbatch : kRevBatches) - 1; b >= 0; --b) {
        const unsigned long long b0 = s_revb[b], b1 = b + 1 < nbatch ? s_revb[b + 1] : rev_done;
        reverse_segments<K, TB>(P, P.revs + 2 * b0, (int64_t)(b1 - b0));
        grid.sync();
      }
      // more levels than batch slots (beyond any tree the executor takes): not restored
      if (gtid == 0) met->error = nbatch <= kRevBatches ? kErrPeekCapacity : 2;
      return;
    }
    O.err = &pc->err[(lev + 1) & 1];
    unsigned long long nrev = *(volatile unsigned long long*)&pc->n_revs;
    if (nrev > rev_done) {
      if (threadIdx.x == 0 && nbatch < kRevBatches) s_revb[nbatch] = rev_done;  // batch starts, for the undo
      ++nbatch;
      reverse_segments<K, TB>(P, P.revs + 2 * rev_done, (int64_t)(nrev - rev_done));
      rev_done = nrev;
      grid.sync();
    }
    unsigned long long cnt = *(volatile unsigned long long*)&pc->front_n[lev % 3];
    if (cnt == 0) break;
    if (gtid == 0) pc->front_n[(lev + 2) % 3] = 0;
    O.next = P.front[(lev + 1) & 1];
    O.next_cnt = &pc->front_n[(lev + 1) % 3];
    const PeekItem* items = P.front[lev & 1];
    for (int64_t x = gtid; x < (int64_t)cnt; x += gthreads) peek_item<K>(V, items[x], P.w, O);
    grid.sync();
    ++lev;
  }
  grid.sync();
#ifdef RS_INSTR
  if (gtid == 0) met->prep_arr[15] = (unsigned long long)lev;  // replay levels
#endif
  if (blockIdx.x == 0) RS_DBG(met, 3);
  // 3. leaf-start bitmap and its word prefix popcount
  unsigned long long R = pc->n_leaves;
  unsigned long long NN = pc->n_nodes;
  for (int64_t k = gtid; k < (int64_t)R; k += gthreads) {
    pos_t l = P.leaves[4 * k];
    atomicOr(P.lbits + (l >> 5), 1u << (l & 31));
  }
  grid.sync();
  int64_t nchunks = (P.words + kWordChunk - 1) / kWordChunk;
  for (int64_t c = blockIdx.x; c < nchunks; c += gridDim.x) {
    unsigned long long s = 0;
    for (int64_t q = c * kWordChunk + threadIdx.x; q < (c + 1) * kWordChunk && q < P.words; q += blockDim.x)
      s += __popc(P.lbits[q]);
    s = block_sum(s, sred);
    if (threadIdx.x == 0) P.chunk[c] = (uint32_t)s;
    __syncthreads();
  }
  grid.sync();
  if (blockIdx.x == 0) {  // exclusive scan of the chunk sums: block scans of blockDim chunks
    __shared__ uint32_t s_cs[40];
    uint32_t carry = 0;
    for (int64_t c0 = 0; c0 < nchunks; c0 += blockDim.x) {
      int64_t c = c0 + threadIdx.x;
      uint32_t v = c < nchunks ? P.chunk[c] : 0u;
      uint32_t tot;
      uint32_t ex = block_excl_scan_u32(v, s_cs, &tot);
      if (c < nchunks) P.chunk[c] = carry + ex;
      carry += tot;
    }
  }
  grid.sync();
  {
    __shared__ uint32_t s_scan[40];
    for (int64_t c = blockIdx.x; c < nchunks; c += gridDim.x) {
      uint32_t base = P.chunk[c];
      for (int64_t q0 = c * kWordChunk; q0 < (c + 1) * kWordChunk && q0 < P.words; q0 += blockDim.x) {
        int64_t q = q0 + threadIdx.x;
        uint32_t v = q < P.words && q < (c + 1) * kWordChunk ? __popc(P.lbits[q]) : 0u;
        uint32_t tot;
        uint32_t ex = block_excl_scan_u32(v, s_scan, &tot);
        if (q < P.words && q < (c + 1) * kWordChunk) P.wpre[q] = base + ex;
        base += tot;
      }
    }
  }
  grid.sync();
  if (blockIdx.x == 0) RS_DBG(met, 4);
  // 4. leaves and nodes onto leaf / boundary indices
  TreeArrays& T = P.T;
  pos_t* leaf_start = const_cast<pos_t*>(T.leaf_start);
  uint32_t* leaf_info = const_cast<uint32_t*>(T.leaf_info);
  for (int64_t k = gtid; k < (int64_t)R; k += gthreads) {
    pos_t l = P.leaves[4 * k], r = P.leaves[4 * k + 1], npre = P.leaves[4 * k + 2];
    int64_t idx = leaf_index(P.lbits, P.wpre, l);
    leaf_start[idx] = l;
    uint32_t nl = npre >= r - l + 1 ? (uint32_t)P.w : (uint32_t)npre;
    leaf_info[idx] = nl;
    T.leaf_depth[idx] = (uint8_t)P.leaves[4 * k + 3];
  }
  for (int64_t k = gtid; k < (int64_t)NN; k += gthreads) {
    pos_t l = P.nodes[4 * k], mid = P.nodes[4 * k + 1], r = P.nodes[4 * k + 2];
    int64_t j = leaf_index(P.lbits, P.wpre, mid);
    T.node_s[j] = l;
    T.node_e[j] = r + 1;
    T.node_a[j] = (int32_t)leaf_index(P.lbits, P.wpre, l);
    T.node_b[j] = (int32_t)((r + 1 >= n ? (int64_t)R : leaf_index(P.lbits, P.wpre, r + 1)) - 1);
    T.depth[j] = (uint8_t)P.nodes[4 * k + 3];
  }
  if (gtid == 0) {
    leaf_start[R] = n;
    met->n_leaves = R;
    met->runs_detected = R;  // sorters.py:358: merges + 1
    if (NN + 1 != R) met->error = 3;
  }
  comps = block_sum(comps + V.comps, sred);
  if (threadIdx.x == 0 && comps) atomicAdd(&met->comparisons, comps);
  grid.sync();
  if (blockIdx.x == 0) RS_DBG(met, 5);
  // 5. parents and children from depths (a child's parent is the deeper of the
  //    boundaries at its span's two ends)
  for (int64_t i = gtid; i < (int64_t)R; i += gthreads) {
    {
      int64_t par = -1;
      int side = 0;
      bool hasL = i >= 1, hasR = i + 1 <= (int64_t)R - 1;
      if (hasL && hasR) {
        if (T.depth[i] > T.depth[i + 1]) { par = i; side = 1; } else { par = i + 1; side = 0; }
      } else if (hasL) { par = i; side = 1; }
      else if (hasR) { par = i + 1; side = 0; }
      uint32_t lid = T.leaf_base + (uint32_t)i;
      T.parent[lid] = (int32_t)par;
      if (par >= 0) T.child[2 * par + side] = lid;
    }
    if (i >= 1) {
      int64_t j = i, aa = T.node_a[j], bb = T.node_b[j];
      int64_t par = -1;
      int side = 0;
      bool hasL = aa >= 1, hasR = bb + 1 <= (int64_t)R - 1;
      if (hasL && hasR) {
        if (T.depth[aa] > T.depth[bb + 1]) { par = aa; side = 1; } else { par = bb + 1; side = 0; }
      } else if (hasL) { par = aa; side = 1; }
      else if (hasR) { par = bb + 1; side = 0; }
      T.parent[j] = (int32_t)par;
      if (par >= 0) T.child[2 * par + side] = (uint32_t)j;
    }
  }
  grid.sync();
  if (blockIdx.x == 0) RS_DBG(met, 6);
  // 6. classification (no detection term: peeksort counted its scans above),
  //    ordered task list -- shared with powersort.
  d_classify(P.CA, P.chunkdep);
  if (last_block_done(&met->last_ctr[2])) {
    d_task_offsets(met);
    __syncthreads();
    d_order_scan(met, P.chunkdep);
  }
  grid.sync();
  pdl_trigger();  // k_phaseA may start launching (it waits for this grid)
  d_task_fill(P.CA, P.chunkdep);
}

}  // namespace rs
