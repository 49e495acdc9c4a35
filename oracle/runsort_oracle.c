/*
 * runsort_oracle.c -- TEST INFRASTRUCTURE ONLY.
 *
 * A plain-C, single-threaded restatement of the reference package's
 * powersort / peeksort (arXiv 1805.04154, Python package `runsort`), used as
 * the parity checker for the CUDA path and as the CPU baseline in bench.py.
 * Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline /
 * --impl reference legs may load it.  The product path never calls it.
 *
 * Pinned against the reference itself: tests/golden/make_golden.py imports
 * the reference from /root/reference/pkg/src and commits its outputs and
 * Metrics as fixtures; tests/test_oracle.py checks this file against them.
 *
 * Every routine cites the reference line it restates
 * (paths relative to /root/reference/pkg/src/runsort/).
 *
 * Keys: int32 or int64 (signed compare).  Tags: opaque 0/4/8-byte payloads
 * moved in lockstep with the keys (runcore.py:3-6).
 */
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

typedef struct {
    uint64_t merge_cost;       /* runcore.py:51 */
    uint64_t comparisons;      /* runcore.py:52 */
    uint64_t runs_detected;    /* runcore.py:53 */
    uint64_t max_stack_height; /* runcore.py:54 */
} orc_metrics;

/* ------------------------------------------------------------------ tags */

typedef struct {
    unsigned char *p;
    int bytes; /* 0, 4 or 8 */
} tagv;

static inline void tag_swap(tagv t, int64_t i, int64_t j) {
    if (t.bytes == 4) {
        uint32_t *q = (uint32_t *)t.p, x = q[i];
        q[i] = q[j]; q[j] = x;
    } else if (t.bytes == 8) {
        uint64_t *q = (uint64_t *)t.p, x = q[i];
        q[i] = q[j]; q[j] = x;
    }
}

static inline void tag_copy(unsigned char *dst, int64_t di, const unsigned char *src,
                            int64_t si, int bytes) {
    if (bytes == 4) ((uint32_t *)dst)[di] = ((const uint32_t *)src)[si];
    else if (bytes == 8) ((uint64_t *)dst)[di] = ((const uint64_t *)src)[si];
}

/* -------------------------------------------------------- node power (int) */

static int bitlen_u64(uint64_t x) { return x ? 64 - __builtin_clzll(x) : 0; }

/* sorters.py:376-392 node_power_def, 1-based runs, any n (128-bit shifts). */
int orc_node_power_def(int64_t s1, int64_t e1, int64_t s2, int64_t e2, int64_t n) {
    if (!(1 <= s1 && s1 <= e1 && e1 < s2 && s2 <= e2 && e2 <= n)) return -1;
    int64_t n1 = e1 - s1 + 1, n2 = e2 - s2 + 1;
    unsigned __int128 a2 = (unsigned __int128)(2 * (s1 - 1) + n1);
    unsigned __int128 b2 = (unsigned __int128)(2 * (s2 - 1) + n2);
    unsigned __int128 two_n = (unsigned __int128)(2 * n);
    int level = 1;
    while ((a2 << level) / two_n == (b2 << level) / two_n) level++;
    return level;
}

/* sorters.py:414-423 _node_power0: 0-based adjacent runs. */
static int node_power0(int64_t s1, int64_t e1, int64_t s2, int64_t e2, int64_t n) {
    if (n < ((int64_t)1 << 31)) {
        uint64_t l = (uint64_t)(s1 + s2), r = (uint64_t)(s2 + e2 + 1);
        uint64_t two_n = 2 * (uint64_t)n;
        uint64_t afix = (l << 31) / two_n, bfix = (r << 31) / two_n;
        return 32 - bitlen_u64(afix ^ bfix);
    }
    return orc_node_power_def(s1 + 1, e1 + 1, s2 + 1, e2 + 1, n);
}

/* --------------------------------------------------- per-key-type kernels */

#define DEFINE_ORACLE(SFX, KT)                                                          \
                                                                                        \
/* runcore.py:70-74 reverse_range */                                                   \
static void reverse_##SFX(KT *a, tagv t, int64_t i, int64_t j) {                        \
    while (i < j) {                                                                     \
        KT x = a[i]; a[i] = a[j]; a[j] = x;                                             \
        tag_swap(t, i, j);                                                              \
        i++; j--;                                                                       \
    }                                                                                   \
}                                                                                       \
                                                                                        \
/* runcore.py:77-89: largest j <= hi with a[i..j] weakly increasing */                 \
static int64_t scan_asc_##SFX(const KT *a, int64_t i, int64_t hi) {                     \
    int64_t j = i;                                                                      \
    while (j < hi && a[j] <= a[j + 1]) j++;                                             \
    return j;                                                                           \
}                                                                                       \
/* runcore.py:92-104: largest j <= hi with a[i..j] strictly decreasing */              \
static int64_t scan_desc_##SFX(const KT *a, int64_t i, int64_t hi) {                    \
    int64_t j = i;                                                                      \
    while (j < hi && a[j] > a[j + 1]) j++;                                              \
    return j;                                                                           \
}                                                                                       \
/* runcore.py:107-119: smallest k >= lo with a[k..i] weakly increasing */              \
static int64_t scan_asc_left_##SFX(const KT *a, int64_t i, int64_t lo) {                \
    int64_t k = i;                                                                      \
    while (k > lo && a[k - 1] <= a[k]) k--;                                             \
    return k;                                                                           \
}                                                                                       \
/* runcore.py:122-134: smallest k >= lo with a[k..i] strictly decreasing */            \
static int64_t scan_desc_left_##SFX(const KT *a, int64_t i, int64_t lo) {               \
    int64_t k = i;                                                                      \
    while (k > lo && a[k - 1] > a[k]) k--;                                              \
    return k;                                                                           \
}                                                                                       \
                                                                                        \
/* runcore.py:137-159 find_run_right; returns end, sets *desc */                       \
static int64_t find_run_right_##SFX(KT *a, tagv t, int64_t i, int64_t hi,               \
                                    orc_metrics *m, int *desc) {                        \
    *desc = 0;                                                                          \
    if (i == hi) return i;                                                              \
    int64_t j;                                                                          \
    if (a[i] <= a[i + 1]) {                                                             \
        j = scan_asc_##SFX(a, i, hi);                                                   \
        m->comparisons += (uint64_t)((j < hi) ? (j - i + 1) : (j - i));                 \
        return j;                                                                       \
    }                                                                                   \
    j = scan_desc_##SFX(a, i, hi);                                                      \
    m->comparisons += (uint64_t)((j < hi) ? (j - i + 1) : (j - i));                     \
    reverse_##SFX(a, t, i, j);                                                          \
    *desc = 1;                                                                          \
    return j;                                                                           \
}                                                                                       \
                                                                                        \
/* runcore.py:215-248 insertionsort_presorted: stable straight insertion with a      \
 * presorted prefix; inserting v past g greater elements costs g+1 comparisons,      \
 * or g when it runs off the left end (runcore.py:237-244). */                         \
static void insertion_##SFX(KT *a, tagv t, int64_t lo, int64_t hi, int64_t npre,        \
                            orc_metrics *m) {                                           \
    int64_t len = hi - lo + 1;                                                          \
    if (npre < 1) npre = 1;                                                             \
    if (len <= 1 || npre >= len) return;                                                \
    uint64_t comps = 0;                                                                 \
    for (int64_t i = lo + npre; i <= hi; i++) {                                         \
        KT v = a[i];                                                                    \
        uint64_t tv = 0;                                                                \
        if (t.bytes == 4) tv = ((uint32_t *)t.p)[i];                                    \
        else if (t.bytes == 8) tv = ((uint64_t *)t.p)[i];                               \
        int64_t j = i - 1;                                                              \
        while (j >= lo) {                                                               \
            comps++;                                                                    \
            if (v < a[j]) {                                                             \
                a[j + 1] = a[j];                                                        \
                tag_copy(t.p, j + 1, t.p, j, t.bytes);                                  \
                j--;                                                                    \
            } else break;                                                               \
        }                                                                               \
        a[j + 1] = v;                                                                   \
        if (t.bytes == 4) ((uint32_t *)t.p)[j + 1] = (uint32_t)tv;                      \
        else if (t.bytes == 8) ((uint64_t *)t.p)[j + 1] = tv;                           \
    }                                                                                   \
    m->comparisons += comps;                                                            \
}                                                                                       \
                                                                                        \
/* runcore.py:251-279 _stable_merge: left run wins ties.  Left run staged in buf. */   \
static void merge_##SFX(KT *a, tagv t, int64_t l, int64_t mid, int64_t r, KT *buf,      \
                        unsigned char *tbuf, int classic, orc_metrics *m) {             \
    int64_t size = r - l + 1;                                                           \
    if (classic) {                                                                      \
        /* runcore.py:319-324: slots of the last left / last right element */           \
        KT lastL = a[mid - 1], lastR = a[r];                                            \
        int64_t lo = mid, hi = r + 1; /* #right < lastL */                              \
        while (lo < hi) { int64_t md = lo + (hi - lo) / 2;                              \
            if (a[md] < lastL) lo = md + 1; else hi = md; }                             \
        int64_t pos_left = (mid - 1 - l) + (lo - mid);                                  \
        lo = l; hi = mid; /* #left <= lastR */                                          \
        while (lo < hi) { int64_t md = lo + (hi - lo) / 2;                              \
            if (a[md] <= lastR) lo = md + 1; else hi = md; }                            \
        int64_t pos_right = (r - mid) + (lo - l);                                       \
        m->comparisons += (uint64_t)((pos_left < pos_right ? pos_left : pos_right) + 1);\
    } else {                                                                            \
        m->comparisons += (uint64_t)size; /* runcore.py:299-301 */                      \
    }                                                                                   \
    m->merge_cost += (uint64_t)size;                                                    \
    int64_t nl = mid - l;                                                               \
    memcpy(buf, a + l, (size_t)nl * sizeof(KT));                                        \
    if (t.bytes) memcpy(tbuf, t.p + (size_t)l * t.bytes, (size_t)nl * t.bytes);         \
    int64_t i = 0, j = mid, k = l;                                                      \
    while (i < nl && j <= r) {                                                          \
        if (buf[i] <= a[j]) { a[k] = buf[i]; tag_copy(t.p, k, tbuf, i, t.bytes); i++; } \
        else { a[k] = a[j]; tag_copy(t.p, k, t.p, j, t.bytes); j++; }                   \
        k++;                                                                            \
    }                                                                                   \
    while (i < nl) { a[k] = buf[i]; tag_copy(t.p, k, tbuf, i, t.bytes); i++; k++; }     \
}                                                                                       \
                                                                                        \
/* sorters.py:430-519 powersort.  Optional outputs: node powers in boundary order   \
 * (r-1 entries) and leaf starts (r entries), written while count < cap. */            \
static int64_t powersort_##SFX(KT *a, tagv t, int64_t n, int32_t w, int classic,        \
                               orc_metrics *m, int32_t *powers_out,                     \
                               int64_t *leaf_starts_out, int64_t cap) {                 \
    if (n <= 1) { m->runs_detected = (uint64_t)n; return n; } /* :445-450 */            \
    KT *buf = (KT *)malloc((size_t)n * sizeof(KT));                                     \
    unsigned char *tbuf = t.bytes ? (unsigned char *)malloc((size_t)n * t.bytes) : 0;   \
    int max_power = bitlen_u64((uint64_t)n); /* :455 */                                 \
    int64_t run_start[72], run_end[72];                                                 \
    for (int i = 0; i <= max_power; i++) { run_start[i] = -1; run_end[i] = -1; }        \
    int top = 0;                                                                        \
    uint64_t occupied = 0;                                                              \
    int64_t nleaves = 0;                                                                \
    /* detect(): sorters.py:462-470 */                                                  \
    int64_t s1 = 0, e1, s2, e2;                                                         \
    {                                                                                   \
        int desc; int64_t end = find_run_right_##SFX(a, t, 0, n - 1, m, &desc);         \
        m->runs_detected += 1;                                                          \
        int64_t len = end + 1;                                                          \
        if (len < w) { end = (w - 1 < n - 1) ? (w - 1) : (n - 1);                       \
                       insertion_##SFX(a, t, 0, end, len, m); }                         \
        e1 = end;                                                                       \
        if (leaf_starts_out && nleaves < cap) leaf_starts_out[nleaves] = 0;             \
        nleaves++;                                                                      \
    }                                                                                   \
    while (e1 < n - 1) { /* :474-504 */                                                 \
        s2 = e1 + 1;                                                                    \
        int desc; int64_t end = find_run_right_##SFX(a, t, s2, n - 1, m, &desc);        \
        m->runs_detected += 1;                                                          \
        int64_t len = end - s2 + 1;                                                     \
        if (len < w) { int64_t cap_end = s2 + w - 1;                                    \
                       end = cap_end < n - 1 ? cap_end : n - 1;                         \
                       insertion_##SFX(a, t, s2, end, len, m); }                        \
        e2 = end;                                                                       \
        if (leaf_starts_out && nleaves < cap) leaf_starts_out[nleaves] = s2;            \
        int p = node_power0(s1, e1, s2, e2, n);                                         \
        if (powers_out && nleaves - 1 < cap) powers_out[nleaves - 1] = p;               \
        nleaves++;                                                                      \
        for (int level = top; level > p; level--) {                                     \
            if (run_start[level] < 0) continue;                                         \
            if (run_end[level] + 1 != s1) { free(buf); free(tbuf); return -2; }         \
            merge_##SFX(a, t, run_start[level], s1, e1, buf, tbuf, classic, m);         \
            s1 = run_start[level];                                                      \
            run_start[level] = -1;                                                      \
            occupied--;                                                                 \
        }                                                                               \
        if (run_start[p] >= 0) { free(buf); free(tbuf); return -3; } /* :491-494 */     \
        run_start[p] = s1; run_end[p] = e1;                                             \
        occupied++;                                                                     \
        if (occupied > m->max_stack_height) m->max_stack_height = occupied;             \
        top = p;                                                                        \
        s1 = s2; e1 = e2;                                                               \
    }                                                                                   \
    for (int level = top; level > 0; level--) { /* :505-516 */                          \
        if (run_start[level] < 0) continue;                                             \
        if (run_end[level] + 1 != s1) { free(buf); free(tbuf); return -2; }             \
        merge_##SFX(a, t, run_start[level], s1, n - 1, buf, tbuf, classic, m);          \
        s1 = run_start[level];                                                          \
        run_start[level] = -1;                                                          \
        occupied--;                                                                     \
    }                                                                                   \
    free(buf); free(tbuf);                                                              \
    return nleaves;                                                                     \
}                                                                                       \
                                                                                        \
/* ---- elementary baselines, sorters.py:524-581 ---- */                              \
/* top_down_mergesort (sorters.py:524-552): midpoint split, insertion sort of      \
 * ranges of <= w elements, one comparison to skip an in-order merge. */             \
static void td_sort_##SFX(KT *a, tagv t, int64_t l, int64_t r, int32_t w, KT *buf,      \
                          unsigned char *tbuf, int classic, orc_metrics *m) {           \
    if (r - l + 1 <= w) { insertion_##SFX(a, t, l, r, 1, m); return; }                 \
    int64_t mid = l + (r - l) / 2;                                                      \
    td_sort_##SFX(a, t, l, mid, w, buf, tbuf, classic, m);                              \
    td_sort_##SFX(a, t, mid + 1, r, w, buf, tbuf, classic, m);                          \
    m->comparisons += 1;                                                                \
    if (a[mid] <= a[mid + 1]) return;                                                   \
    merge_##SFX(a, t, l, mid + 1, r, buf, tbuf, classic, m);                            \
}                                                                                       \
/* bottom_up_mergesort (sorters.py:555-581): insertion-sorted chunks of w, then     \
 * passes of doubling width with the same skip check. */                               \
static void bu_sort_##SFX(KT *a, tagv t, int64_t n, int32_t w, KT *buf,                 \
                          unsigned char *tbuf, int classic, orc_metrics *m) {           \
    if (w > 1)                                                                          \
        for (int64_t c = 0; c < n; c += w)                                              \
            insertion_##SFX(a, t, c, (c + w < n ? c + w : n) - 1, 1, m);                \
    for (int64_t width = w; width < n; width *= 2) {                                    \
        for (int64_t l = 0; l < n - width; l += 2 * width) {                            \
            int64_t mid = l + width;                                                    \
            int64_t r = l + 2 * width - 1 < n - 1 ? l + 2 * width - 1 : n - 1;          \
            m->comparisons += 1;                                                        \
            if (a[mid - 1] <= a[mid]) continue;                                         \
            merge_##SFX(a, t, l, mid, r, buf, tbuf, classic, m);                        \
        }                                                                               \
    }                                                                                   \
}                                                                                       \
/* _stack_natural_sort (sorters.py:587-635): detect + extend runs like powersort,  \
 * push, merge the top two while len_below < alpha * len_top (alpha-merge also      \
 * merges the top two before the push while the top is shorter than the new run),   \
 * finally merge the stack bottom-up, left to right. */                                \
static int64_t alpha_sort_##SFX(KT *a, tagv t, int64_t n, int32_t w, int classic,       \
                                double alpha, int pre_push, orc_metrics *m) {           \
    if (n <= 1) { m->runs_detected = (uint64_t)n; return 0; }                           \
    KT *buf = (KT *)malloc((size_t)n * sizeof(KT));                                     \
    unsigned char *tbuf = t.bytes ? (unsigned char *)malloc((size_t)n * t.bytes) : 0;   \
    int64_t cap = 64, h = 0;                                                            \
    int64_t *ss = (int64_t *)malloc(cap * sizeof(int64_t));                             \
    int64_t *se = (int64_t *)malloc(cap * sizeof(int64_t));                             \
    int64_t pos = 0;                                                                    \
    while (pos < n) {                                                                   \
        int desc; int64_t e = find_run_right_##SFX(a, t, pos, n - 1, m, &desc);         \
        m->runs_detected += 1;                                                          \
        int64_t len = e - pos + 1;                                                      \
        if (len < w) { e = (pos + w - 1 < n - 1) ? pos + w - 1 : n - 1;                 \
                       insertion_##SFX(a, t, pos, e, len, m); }                         \
        int64_t s = pos;                                                                \
        if (pre_push)                                                                   \
            while (h >= 2 && se[h - 1] - ss[h - 1] + 1 < e - s + 1) {                   \
                merge_##SFX(a, t, ss[h - 2], ss[h - 1], se[h - 1], buf, tbuf, classic, m); \
                se[h - 2] = se[h - 1]; h--;                                             \
            }                                                                           \
        if (h == cap) { cap *= 2; ss = (int64_t *)realloc(ss, cap * sizeof(int64_t));   \
                        se = (int64_t *)realloc(se, cap * sizeof(int64_t)); }           \
        ss[h] = s; se[h] = e; h++;                                                      \
        while (h >= 2) {                                                                \
            int64_t lb = se[h - 2] - ss[h - 2] + 1, lt = se[h - 1] - ss[h - 1] + 1;     \
            if ((double)lb < alpha * (double)lt) {                                      \
                merge_##SFX(a, t, ss[h - 2], ss[h - 1], se[h - 1], buf, tbuf, classic, m); \
                se[h - 2] = se[h - 1]; h--;                                             \
            } else break;                                                               \
        }                                                                               \
        if ((uint64_t)h > m->max_stack_height) m->max_stack_height = (uint64_t)h;       \
        pos = e + 1;                                                                    \
    }                                                                                   \
    for (int64_t k = 1; k < h; k++) /* cleanup: bottom-up, left to right */             \
        merge_##SFX(a, t, ss[0], ss[k], se[k], buf, tbuf, classic, m);                  \
    free(ss); free(se); free(buf); free(tbuf);                                          \
    return 0;                                                                           \
}                                                                                       \
static int64_t baseline_##SFX(int algo, KT *a, tagv t, int64_t n, int32_t w,            \
                              int classic, double alpha, orc_metrics *m) {              \
    if (algo == 4 || algo == 5) return alpha_sort_##SFX(a, t, n, w, classic, alpha, algo == 5, m); \
    if (n <= 1) return 0;                                                               \
    KT *buf = (KT *)malloc((size_t)n * sizeof(KT));                                     \
    unsigned char *tbuf = t.bytes ? (unsigned char *)malloc((size_t)n * t.bytes) : 0;   \
    if (algo == 2) td_sort_##SFX(a, t, 0, n - 1, w, buf, tbuf, classic, m);             \
    else bu_sort_##SFX(a, t, n, w, buf, tbuf, classic, m);                              \
    free(buf); free(tbuf);                                                              \
    return 0;                                                                           \
}                                                                                       \
                                                                                        \
/* ---- peeksort, sorters.py:146-361 ---- */                                           \
typedef struct {                                                                        \
    KT *a; tagv t; KT *buf; unsigned char *tbuf; int classic; int32_t w;                \
    orc_metrics *m; int64_t merges;                                                     \
    int64_t *merges_out; int64_t cap; /* (l, mid, r, depth) quadruples */               \
} peek_##SFX;                                                                           \
                                                                                        \
static void peek_merge_##SFX(peek_##SFX *P, int64_t l, int64_t mid, int64_t r,          \
                             int64_t depth) {                                           \
    merge_##SFX(P->a, P->t, l, mid, r, P->buf, P->tbuf, P->classic, P->m);              \
    if (P->merges_out && P->merges < P->cap) {                                          \
        P->merges_out[4 * P->merges + 0] = l;                                           \
        P->merges_out[4 * P->merges + 1] = mid;                                         \
        P->merges_out[4 * P->merges + 2] = r;                                           \
        P->merges_out[4 * P->merges + 3] = depth;                                       \
    }                                                                                   \
    P->merges++;                                                                        \
}                                                                                       \
/* sorters.py:180-199: scans with the scalar pair-count convention */                  \
static int64_t pk_asc_right_##SFX(peek_##SFX *P, int64_t st, int64_t bound) {           \
    int64_t j = scan_asc_##SFX(P->a, st, bound);                                        \
    P->m->comparisons += (uint64_t)((j < bound) ? (j - st + 1) : (j - st));             \
    return j;                                                                           \
}                                                                                       \
static int64_t pk_asc_left_##SFX(peek_##SFX *P, int64_t st, int64_t bound) {            \
    int64_t i = scan_asc_left_##SFX(P->a, st, bound);                                   \
    P->m->comparisons += (uint64_t)((i > bound) ? (st - i + 1) : (st - i));             \
    return i;                                                                           \
}                                                                                       \
static int64_t pk_desc_right_##SFX(peek_##SFX *P, int64_t st, int64_t bound) {          \
    int64_t j = scan_desc_##SFX(P->a, st, bound);                                       \
    P->m->comparisons += (uint64_t)((j < bound) ? (j - st + 1) : (j - st));             \
    return j;                                                                           \
}                                                                                       \
static int64_t pk_desc_left_##SFX(peek_##SFX *P, int64_t st, int64_t bound) {           \
    int64_t i = scan_desc_left_##SFX(P->a, st, bound);                                  \
    P->m->comparisons += (uint64_t)((i > bound) ? (st - i + 1) : (st - i));             \
    return i;                                                                           \
}                                                                                       \
/* sorters.py:201-215 extend_prefix */                                                 \
static int64_t pk_ext_prefix_##SFX(peek_##SFX *P, int64_t e, int64_t r, int64_t s,      \
                                   int e_desc, int s_desc) {                            \
    KT *a = P->a;                                                                       \
    if (e_desc || e == r) return e;                                                     \
    P->m->comparisons += 1;                                                             \
    if (a[e] > a[e + 1]) return e;                                                      \
    if (e + 1 == s) return r;                                                           \
    int64_t E = pk_asc_right_##SFX(P, e + 1, s - 1);                                    \
    if (E == s - 1 && !s_desc) {                                                        \
        P->m->comparisons += 1;                                                         \
        if (a[s - 1] <= a[s]) return r;                                                 \
    }                                                                                   \
    return E;                                                                           \
}                                                                                       \
/* sorters.py:217-231 extend_suffix */                                                 \
static int64_t pk_ext_suffix_##SFX(peek_##SFX *P, int64_t s, int64_t l, int64_t e,      \
                                   int s_desc, int e_desc) {                            \
    KT *a = P->a;                                                                       \
    if (s_desc || s == l) return s;                                                     \
    P->m->comparisons += 1;                                                             \
    if (a[s - 1] > a[s]) return s;                                                      \
    if (s - 1 == e) return l;                                                           \
    int64_t S = pk_asc_left_##SFX(P, s - 1, e + 1);                                     \
    if (S == e + 1 && !e_desc) {                                                        \
        P->m->comparisons += 1;                                                         \
        if (a[e] <= a[e + 1]) return l;                                                 \
    }                                                                                   \
    return S;                                                                           \
}                                                                                       \
/* sorters.py:233-303 probe: returns run [*pi..*pj] around m with descent flags */     \
static void pk_probe_##SFX(peek_##SFX *P, int64_t m, int64_t l, int64_t r, int64_t e,   \
                           int64_t s, int e_desc, int s_desc, int64_t *pi,              \
                           int64_t *pj, int *idesc, int *jdesc) {                       \
    KT *a = P->a;                                                                       \
    int asc_right;                                                                      \
    if (m + 1 == s && s_desc) asc_right = 0;                                            \
    else { P->m->comparisons += 1; asc_right = a[m] <= a[m + 1]; }                      \
    if (asc_right) {                                                                    \
        int64_t j, i;                                                                   \
        if (m + 1 == s) j = r;                                                          \
        else {                                                                          \
            j = pk_asc_right_##SFX(P, m + 1, s - 1);                                    \
            if (j == s - 1 && !s_desc) {                                                \
                P->m->comparisons += 1;                                                 \
                if (a[s - 1] <= a[s]) j = r;                                            \
            }                                                                           \
        }                                                                               \
        i = pk_asc_left_##SFX(P, m, e + 1);                                             \
        if (i == e + 1 && !e_desc) {                                                    \
            P->m->comparisons += 1;                                                     \
            if (a[e] <= a[e + 1]) i = l;                                                \
        }                                                                               \
        *pi = i; *pj = j; *idesc = 1; *jdesc = 1;                                       \
        return;                                                                         \
    }                                                                                   \
    int asc_left;                                                                       \
    if (m - 1 == e && e_desc) asc_left = 0;                                             \
    else { P->m->comparisons += 1; asc_left = a[m - 1] <= a[m]; }                       \
    if (asc_left) {                                                                     \
        if (m - 1 == e) { *pi = l; *pj = m; *idesc = 1; *jdesc = 1; return; }           \
        int64_t i = pk_asc_left_##SFX(P, m - 1, e + 1);                                 \
        if (i == e + 1 && !e_desc) {                                                    \
            P->m->comparisons += 1;                                                     \
            if (a[e] <= a[e + 1]) i = l;                                                \
        }                                                                               \
        *pi = i; *pj = m; *idesc = 1; *jdesc = 1;                                       \
        return;                                                                         \
    }                                                                                   \
    int64_t i, j;                                                                       \
    if (m - 1 > e) {                                                                    \
        i = pk_desc_left_##SFX(P, m - 1, e + 1);                                        \
        if (i == e + 1 && l == e) {                                                     \
            if (e_desc) i = l;                                                          \
            else { P->m->comparisons += 1; if (a[e] > a[e + 1]) i = l; }                \
        }                                                                               \
    } else if (l == e) i = l;                                                           \
    else i = m;                                                                         \
    if (m + 1 == s) j = (s == r) ? r : s;                                               \
    else {                                                                              \
        j = pk_desc_right_##SFX(P, m + 1, s - 1);                                       \
        if (j == s - 1 && s == r) {                                                     \
            if (s_desc) j = r;                                                          \
            else { P->m->comparisons += 1; if (a[s - 1] > a[s]) j = r; }                \
        }                                                                               \
    }                                                                                   \
    reverse_##SFX(a, P->t, i, j);                                                       \
    *pi = i; *pj = j; *idesc = 0; *jdesc = 0;                                           \
}                                                                                       \
/* sorters.py:305-349 sort(l, r, e, s, e_desc, s_desc) */                              \
static void pk_sort_##SFX(peek_##SFX *P, int64_t l, int64_t r, int64_t e, int64_t s,    \
                          int e_desc, int s_desc, int64_t depth) {                      \
    if (e == r || s == l) return;                                                       \
    if (r - l + 1 <= P->w) {                                                            \
        insertion_##SFX(P->a, P->t, l, r, e - l + 1, P->m);                             \
        return;                                                                         \
    }                                                                                   \
    int64_t m = l + (r - l) / 2;                                                        \
    if (m <= e) {                                                                       \
        int64_t E = pk_ext_prefix_##SFX(P, e, r, s, e_desc, s_desc);                    \
        if (E == r) return;                                                             \
        pk_sort_##SFX(P, E + 1, r, E + 1, s, 0, s_desc, depth + 1);                     \
        peek_merge_##SFX(P, l, E + 1, r, depth);                                        \
        return;                                                                         \
    }                                                                                   \
    if (m >= s) {                                                                       \
        int64_t S = pk_ext_suffix_##SFX(P, s, l, e, s_desc, e_desc);                    \
        if (S == l) return;                                                             \
        pk_sort_##SFX(P, l, S - 1, e, S - 1, e_desc, 0, depth + 1);                     \
        peek_merge_##SFX(P, l, S, r, depth);                                            \
        return;                                                                         \
    }                                                                                   \
    int64_t i, j; int idesc, jdesc;                                                     \
    pk_probe_##SFX(P, m, l, r, e, s, e_desc, s_desc, &i, &j, &idesc, &jdesc);           \
    if (i == l && j == r) return;                                                       \
    if (i + j >= l + r) { /* :334, ties go left */                                      \
        pk_sort_##SFX(P, l, i - 1, e, i - 1, e_desc, 0, depth + 1);                     \
        if (s > j) pk_sort_##SFX(P, i, r, j, s, jdesc, s_desc, depth + 1);             \
        else pk_sort_##SFX(P, i, r, j, (j + 1 < r ? j + 1 : r), jdesc, 0, depth + 1);   \
        peek_merge_##SFX(P, l, i, r, depth);                                            \
    } else {                                                                            \
        pk_sort_##SFX(P, l, j, e, i, e_desc, idesc, depth + 1);                         \
        if (s > j + 1) pk_sort_##SFX(P, j + 1, r, j + 1, s, 0, s_desc, depth + 1);      \
        else pk_sort_##SFX(P, j + 1, r, j + 1, j + 1, 0, jdesc, depth + 1);             \
        peek_merge_##SFX(P, l, j + 1, r, depth);                                        \
    }                                                                                   \
}                                                                                       \
/* sorters.py:146-361 peeksort driver.  Returns #merges; merges_out gets           \
 * (l, mid, r, depth) per merge in execution (post-)order. */                          \
static int64_t peeksort_##SFX(KT *a, tagv t, int64_t n, int32_t w, int classic,         \
                              orc_metrics *m, int64_t *merges_out, int64_t cap) {       \
    if (n <= 1) { m->runs_detected = (uint64_t)n; return 0; } /* :169-173 */            \
    peek_##SFX P;                                                                       \
    P.a = a; P.t = t; P.classic = classic; P.w = w; P.m = m; P.merges = 0;              \
    P.merges_out = merges_out; P.cap = cap;                                             \
    P.buf = (KT *)malloc((size_t)n * sizeof(KT));                                       \
    P.tbuf = t.bytes ? (unsigned char *)malloc((size_t)n * t.bytes) : 0;                \
    int first_desc;                                                                     \
    int64_t e0 = find_run_right_##SFX(a, t, 0, n - 1, m, &first_desc); /* :177 */       \
    if (e0 == n - 1) { /* single run */ }                                               \
    else if (n <= w) insertion_##SFX(a, t, 0, n - 1, e0 + 1, m);                        \
    else pk_sort_##SFX(&P, 0, n - 1, e0, n - 1, !first_desc, 0, 0);                     \
    m->runs_detected = (uint64_t)(P.merges + 1); /* :358 (assignment) */                \
    free(P.buf); free(P.tbuf);                                                          \
    return P.merges;                                                                    \
}

DEFINE_ORACLE(i32, int32_t)
DEFINE_ORACLE(i64, int64_t)

/* ------------------------------------------------------------ C ABI (test) */

/* key_kind: 0 = int32, 1 = int64.  Returns #leaves (>= 0) or < 0 on an
 * invariant failure (the reference raises AssertionError, sorters.py:481-494). */
int64_t orc_powersort(int key_kind, void *keys, int tag_bytes, void *tags, int64_t n,
                      int32_t min_run_len, int32_t classic, orc_metrics *m,
                      int32_t *powers_out, int64_t *leaf_starts_out, int64_t cap) {
    tagv t = {(unsigned char *)tags, tags ? tag_bytes : 0};
    if (key_kind == 0)
        return powersort_i32((int32_t *)keys, t, n, min_run_len, classic, m, powers_out,
                             leaf_starts_out, cap);
    return powersort_i64((int64_t *)keys, t, n, min_run_len, classic, m, powers_out,
                         leaf_starts_out, cap);
}

int64_t orc_peeksort(int key_kind, void *keys, int tag_bytes, void *tags, int64_t n,
                     int32_t min_run_len, int32_t classic, orc_metrics *m,
                     int64_t *merges_out, int64_t cap) {
    tagv t = {(unsigned char *)tags, tags ? tag_bytes : 0};
    if (key_kind == 0)
        return peeksort_i32((int32_t *)keys, t, n, min_run_len, classic, m, merges_out, cap);
    return peeksort_i64((int64_t *)keys, t, n, min_run_len, classic, m, merges_out, cap);
}

/* algo: 2 top-down, 3 bottom-up, 4 alpha-stack, 5 alpha-merge (sorters.py:524-660).
 * Returns 0, or < 0 on a bad algo code. */
int64_t orc_baseline(int algo, int key_kind, void *keys, int tag_bytes, void *tags, int64_t n,
                     int32_t min_run_len, int32_t classic, double alpha, orc_metrics *m) {
    if (algo < 2 || algo > 5) return -1;
    tagv t = {(unsigned char *)tags, tags ? tag_bytes : 0};
    if (key_kind == 0)
        return baseline_i32(algo, (int32_t *)keys, t, n, min_run_len, classic, alpha, m);
    return baseline_i64(algo, (int64_t *)keys, t, n, min_run_len, classic, alpha, m);
}

int orc_node_power0(int64_t s1, int64_t e1, int64_t s2, int64_t e2, int64_t n) {
    return node_power0(s1, e1, s2, e2, n);
}
