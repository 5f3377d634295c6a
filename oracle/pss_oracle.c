/*
 * oracle/pss_oracle.c -- TEST INFRASTRUCTURE ONLY.
 *
 * A plain, slow, obviously correct CPU implementation of Parallel Space Saving (Cafaro,
 * Pulimeno, Epicoco, Aloisio; arXiv 1606.04669), written from PAPER.md. It exists to check the
 * CUDA path (paper_1606_04669_b200/) and shares no code with it. Only tests/, __graft_entry__.smoke()
 * and bench.py's cpu_baseline / --impl reference legs may load it. Nothing here is tuned: lookups
 * are linear scans over the k counters, the minimum is found by a linear scan, COMBINE matches by
 * linear scan and orders with the C library's qsort.
 *
 * All arithmetic is integer. Keys are widened to uint64 (ordering of u32 keys is unchanged).
 * Readings of the paper (R1..R12) are the ones listed in DESIGN.md / SURVEY.md section 8(c).
 *
 * Pins: tests/test_oracle_pins.py checks every function below against worked examples
 * (tests/golden/), closed forms, textbook special cases (numpy unique/histograms) and the paper's
 * guarantees checked exhaustively on tiny inputs. No function here is "parity unpinned".
 */
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

static uint64_t key_at(const void* A, int key_bytes, uint64_t i) {
  return key_bytes == 4 ? (uint64_t)((const uint32_t*)A)[i] : ((const uint64_t*)A)[i];
}

/*
 * Block decomposition, Algorithm 1 lines 3-4: left = floor(r n / p),
 * right = floor((r+1) n / p) - 1. Returned as the half-open range [lo, hi) = [left, right + 1).
 * 128-bit products (reading R10); p > n gives empty ranges.
 */
void orc_bounds(uint64_t n, uint32_t p, uint32_t r, uint64_t* lo, uint64_t* hi) {
  *lo = (uint64_t)(((unsigned __int128)r * n) / p);
  *hi = (uint64_t)(((unsigned __int128)(r + 1u) * n) / p);
}

/*
 * Sequential Space Saving with k counters over A[lo..hi) (Algorithm 1 line 5,
 * PAPER.md:96): "When processing an item which is already monitored by a counter, its estimated
 * frequency is incremented by one. ... If a counter is available, it will be in charge of
 * monitoring the item and its estimated frequency is set to one. Otherwise ... the counter
 * storing the item with minimum frequency is incremented by one. Then the monitored item is
 * evicted from the counter and replaced by the new item."
 *   R1: the evicted counter is the lowest count, then the lowest slot index.
 *   R2: free counters are taken in slot order 0, 1, ..., k-1.
 *   R3: err = 0 on fill, err = m (the evicted minimum) on eviction (Metwally's epsilon).
 * Output: slots 0..size-1 in slot order. Returns size.
 */
/* Compiled twice by gcc (AVX2 and baseline x86-64, chosen at load time) only so that the full-size
 * parity tests finish in minutes; the C below is the same for both. */
#if defined(__GNUC__) && defined(__x86_64__) && !defined(__clang__)
__attribute__((target_clones("arch=x86-64-v3", "default")))
#endif
uint32_t orc_space_saving(const void* A, int key_bytes, uint64_t lo, uint64_t hi, uint32_t k,
                          uint64_t* items, uint64_t* counts, uint64_t* errs) {
  uint32_t size = 0;
  for (uint64_t i = lo; i < hi; ++i) {
    uint64_t x = key_at(A, key_bytes, i);
    uint32_t s;
    for (s = 0; s < size; ++s)
      if (items[s] == x) break;
    if (s < size) { /* monitored: incremented by one */
      counts[s] += 1;
    } else if (size < k) { /* a counter is available */
      items[size] = x;
      counts[size] = 1;
      errs[size] = 0;
      size += 1;
    } else { /* all occupied: the minimum counter (lowest slot on ties) */
      uint64_t m = counts[0];
      for (uint32_t t = 1; t < k; ++t)
        if (counts[t] < m) m = counts[t];
      uint32_t v = 0;
      while (counts[v] != m) ++v;
      items[v] = x;
      errs[v] = m;
      counts[v] = m + 1;
    }
  }
  return size;
}

/*
 * MIN(S): Algorithm 2 lines 2-3 read m = S[0].f, the minimum of all of the
 * frequencies of a summary that has "exactly k counters". Reading R4: an
 * unoccupied counter has frequency 0, so m = 0 unless all k counters are occupied.
 */
uint64_t orc_min(const uint64_t* counts, uint32_t size, uint32_t k) {
  if (size < k) return 0;
  uint64_t m = counts[0];
  for (uint32_t t = 1; t < size; ++t)
    if (counts[t] < m) m = counts[t];
  return m;
}

typedef struct {
  uint64_t item, count, err;
} counter_t;

/* canonical order, reading R5: count descending, then item ascending */
static int canon_cmp(const void* a, const void* b) {
  const counter_t* x = (const counter_t*)a;
  const counter_t* y = (const counter_t*)b;
  if (x->count != y->count) return x->count > y->count ? -1 : 1;
  if (x->item != y->item) return x->item < y->item ? -1 : 1;
  return 0;
}

/* sort a summary into canonical order in place (R5) */
void orc_canonical(uint64_t* items, uint64_t* counts, uint64_t* errs, uint32_t size) {
  counter_t* c = (counter_t*)malloc(sizeof(counter_t) * (size ? size : 1));
  for (uint32_t i = 0; i < size; ++i) c[i] = (counter_t){items[i], counts[i], errs[i]};
  qsort(c, size, sizeof(counter_t), canon_cmp);
  for (uint32_t i = 0; i < size; ++i) {
    items[i] = c[i].item;
    counts[i] = c[i].count;
    errs[i] = c[i].err;
  }
  free(c);
}

/*
 * COMBINE(S1, S2, k), Algorithm 2 (prose PAPER.md:112-115):
 *   m1, m2 = minima (lines 2-3, reading R4);
 *   for each counter of S1: if S2.Find(item) -> f1 + f2, S2.Remove; else f1 + m2 (lines 4-13);
 *   for each remaining counter of S2: f2 + m1 (lines 14-18);
 *   Prune(k): "only the k counters with the greatest frequencies are kept" (line 19).
 * Errors (reading R3): matched e1 + e2, S1-only e1 + m2, S2-only e2 + m1.
 * Ties at rank k and the output order: canonical order (reading R5). Returns the output size.
 */
uint32_t orc_combine(const uint64_t* it1, const uint64_t* c1, const uint64_t* e1, uint32_t n1,
                     const uint64_t* it2, const uint64_t* c2, const uint64_t* e2, uint32_t n2,
                     uint32_t k, uint64_t* out_items, uint64_t* out_counts, uint64_t* out_errs) {
  uint64_t m1 = orc_min(c1, n1, k);
  uint64_t m2 = orc_min(c2, n2, k);
  counter_t* sc = (counter_t*)malloc(sizeof(counter_t) * (n1 + n2 + 1));
  char* removed = (char*)calloc(n2 + 1, 1);
  uint32_t nc = 0;
  for (uint32_t i = 0; i < n1; ++i) {
    uint32_t j;
    for (j = 0; j < n2; ++j)
      if (!removed[j] && it2[j] == it1[i]) break;
    if (j < n2) {
      sc[nc++] = (counter_t){it1[i], c1[i] + c2[j], e1[i] + e2[j]};
      removed[j] = 1;
    } else {
      sc[nc++] = (counter_t){it1[i], c1[i] + m2, e1[i] + m2};
    }
  }
  for (uint32_t j = 0; j < n2; ++j)
    if (!removed[j]) sc[nc++] = (counter_t){it2[j], c2[j] + m1, e2[j] + m1};
  qsort(sc, nc, sizeof(counter_t), canon_cmp);
  uint32_t out = nc < k ? nc : k;
  for (uint32_t i = 0; i < out; ++i) {
    out_items[i] = sc[i].item;
    out_counts[i] = sc[i].count;
    out_errs[i] = sc[i].err;
  }
  free(sc);
  free(removed);
  return out;
}

/*
 * ParallelReduction(local, k, COMBINE) (Algorithm 1 line 7). Reading R6: a fixed
 * balanced binary tree, level by level, nodes (2i, 2i+1) merged, an odd last node carried up
 * unchanged. Leaves are given as [P][k] arrays with sizes[P]. The root is returned in canonical
 * order (R5). Returns the root size.
 */
uint32_t orc_tree(const uint64_t* items, const uint64_t* counts, const uint64_t* errs,
                  const uint32_t* sizes, uint32_t P, uint32_t k, uint64_t* root_items,
                  uint64_t* root_counts, uint64_t* root_errs) {
  size_t cap = (size_t)P * k + 1;
  uint64_t* ci = (uint64_t*)malloc(cap * 8);
  uint64_t* cc = (uint64_t*)malloc(cap * 8);
  uint64_t* ce = (uint64_t*)malloc(cap * 8);
  uint32_t* cs = (uint32_t*)malloc(sizeof(uint32_t) * (P + 1));
  uint64_t* ni = (uint64_t*)malloc(cap * 8);
  uint64_t* nn = (uint64_t*)malloc(cap * 8);
  uint64_t* ne = (uint64_t*)malloc(cap * 8);
  uint32_t* ns = (uint32_t*)malloc(sizeof(uint32_t) * (P + 1));
  memcpy(ci, items, (size_t)P * k * 8);
  memcpy(cc, counts, (size_t)P * k * 8);
  memcpy(ce, errs, (size_t)P * k * 8);
  memcpy(cs, sizes, sizeof(uint32_t) * P);
  uint32_t cur = P;
  while (cur > 1) {
    uint32_t nxt = 0;
    for (uint32_t i = 0; i + 1 < cur; i += 2, ++nxt) {
      size_t a = (size_t)i * k, b = (size_t)(i + 1) * k, o = (size_t)nxt * k;
      ns[nxt] = orc_combine(ci + a, cc + a, ce + a, cs[i], ci + b, cc + b, ce + b, cs[i + 1], k,
                            ni + o, nn + o, ne + o);
    }
    if (cur & 1u) { /* odd last node carried up unchanged */
      size_t a = (size_t)(cur - 1) * k, o = (size_t)nxt * k;
      memcpy(ni + o, ci + a, (size_t)k * 8);
      memcpy(nn + o, cc + a, (size_t)k * 8);
      memcpy(ne + o, ce + a, (size_t)k * 8);
      ns[nxt] = cs[cur - 1];
      ++nxt;
    }
    uint64_t* t;
    t = ci; ci = ni; ni = t;
    t = cc; cc = nn; nn = t;
    t = ce; ce = ne; ne = t;
    uint32_t* ts = cs; cs = ns; ns = ts;
    cur = nxt;
  }
  uint32_t size = P ? cs[0] : 0;
  memcpy(root_items, ci, (size_t)size * 8);
  memcpy(root_counts, cc, (size_t)size * 8);
  memcpy(root_errs, ce, (size_t)size * 8);
  orc_canonical(root_items, root_counts, root_errs, size);
  free(ci); free(cc); free(ce); free(cs);
  free(ni); free(nn); free(ne); free(ns);
  return size;
}

/*
 * Pruned(global, n, k) at rank 0 (Algorithm 1 lines 8-9): "removing all of the
 * items below the threshold required for an item to be frequent"; the threshold is
 * f >= floor(n/k) + 1. Candidates keep root order (reading R7/R8).
 */
uint64_t orc_threshold(uint64_t n, uint32_t k) { return n / k + 1; }

uint32_t orc_prune(const uint64_t* items, const uint64_t* counts, uint32_t size, uint64_t n,
                   uint32_t k, uint64_t* cand) {
  uint64_t thr = orc_threshold(n, k);
  uint32_t nc = 0;
  for (uint32_t i = 0; i < size; ++i)
    if (counts[i] >= thr) cand[nc++] = items[i];
  return nc;
}

static int u64_cmp(const void* a, const void* b) {
  uint64_t x = *(const uint64_t*)a, y = *(const uint64_t*)b;
  return x < y ? -1 : (x > y ? 1 : 0);
}

/*
 * Off-line verification ("a parallel scan of the input can be used to determine the
 * actual frequent items"): exact[j] = #{i : A[i] = cand[j]}. One pass over A; each key is looked
 * up by binary search in a sorted copy of the candidate list (qsort), counts go back to the
 * candidates' own positions.
 */
void orc_verify(const void* A, int key_bytes, uint64_t n, const uint64_t* cand, uint32_t nc,
                uint64_t* exact) {
  uint64_t* sorted = (uint64_t*)malloc(8 * (nc + 1));
  uint64_t* cnt = (uint64_t*)calloc(nc + 1, 8);
  memcpy(sorted, cand, 8 * (size_t)nc);
  qsort(sorted, nc, 8, u64_cmp);
  for (uint64_t i = 0; i < n; ++i) {
    uint64_t x = key_at(A, key_bytes, i);
    uint32_t lo = 0, hi = nc;
    while (lo < hi) {
      uint32_t mid = lo + (hi - lo) / 2;
      if (sorted[mid] < x) lo = mid + 1; else hi = mid;
    }
    if (lo < nc && sorted[lo] == x) cnt[lo] += 1;
  }
  for (uint32_t j = 0; j < nc; ++j) {
    uint64_t* p = (uint64_t*)bsearch(&cand[j], sorted, nc, 8, u64_cmp);
    /* duplicates in cand share one sorted entry: find its first position */
    while (p > sorted && p[-1] == cand[j]) --p;
    exact[j] = cnt[p - sorted];
  }
  free(sorted);
  free(cnt);
}

/*
 * The k-majority answer after verification: the candidates whose exact count
 * reaches floor(n/k) + 1, ordered by (exact count desc, item asc). Returns its length.
 */
uint32_t orc_result(const uint64_t* cand, const uint64_t* exact, uint32_t nc, uint64_t n,
                    uint32_t k, uint64_t* out_items, uint64_t* out_counts) {
  uint64_t thr = orc_threshold(n, k);
  counter_t* r = (counter_t*)malloc(sizeof(counter_t) * (nc + 1));
  uint32_t len = 0;
  for (uint32_t j = 0; j < nc; ++j)
    if (exact[j] >= thr) r[len++] = (counter_t){cand[j], exact[j], 0};
  qsort(r, len, sizeof(counter_t), canon_cmp);
  for (uint32_t j = 0; j < len; ++j) {
    out_items[j] = r[j].item;
    out_counts[j] = r[j].count;
  }
  free(r);
  return len;
}
