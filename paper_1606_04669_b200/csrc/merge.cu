// merge.cu -- K2/K3: COMBINE (Algorithm 2) on a fixed balanced binary merge
// tree (ParallelReduction, Algorithm 1 line 7; reading R6), and Pruned (Algorithm 1
// lines 8-9).
//
// One CTA per COMBINE. Both summaries are staged in shared memory; S2's items are indexed by a
// small hash table so each S1 counter finds its match in O(1) (Find/Remove of Alg. 2 l.5-7);
// unmatched counters get the other summary's minimum (R4: 0 for an unfull summary); Prune(k)
// orders the <= 2k counters by (count desc, item asc) and keeps the first k (R5). The ordering is
// a bitonic network over NT threads x EPT elements held in registers: exchanges between elements
// of one thread stay in registers, exchanges within a warp use shuffles, and only the strides of
// 32*EPT elements and more go through shared memory. Outputs are in canonical order.
#include <cstdio>
#include <cstdlib>

#include "common.cuh"

namespace pss {

struct NodeRef {  // a batch of summaries, structure of arrays
  const void* items;
  const uint32_t* counts;
  const uint32_t* errs;
  const uint32_t* sizes;
};
struct NodeOut {
  void* items;
  uint32_t* counts;
  uint32_t* errs;
  uint32_t* sizes;
};

struct CombArgs {
  NodeRef a, b;
  NodeOut o;
  uint32_t k;
  uint32_t a_mul, a_add, b_mul, b_add;  // left node = blk*a_mul + a_add, right = blk*b_mul + b_add
  uint32_t nblocks;                     // output nodes
  uint32_t nright;                      // blocks < nright have a right node
  uint32_t canon_single;                // a block without right node: 1 = canonicalize, 0 = copy
  uint32_t sort_out;                    // 1 = canonical order, 0 = top-k set (internal node)
  unsigned char* gscratch;              // per-CTA scratch when it does not fit shared memory
  size_t gstride;
  size_t o_ucnt, o_uerr, o_dead, o_ht, o_x;
  uint32_t logH2;
  uint32_t NP;  // sort width
  uint32_t no_x;  // the working set has no exchange buffer (tree kernel of large summaries)
};

struct MLayout {
  size_t ukey, ucnt, uerr, dead, ht, x, total;
  uint32_t logH2, NP;
};

// NP = sort width (power of two >= 2k); x = exchange buffer for the shared-memory sort passes
static MLayout m_layout(uint32_t k, int kb, uint32_t NP) {
  MLayout L;
  const size_t U = 2 * (size_t)k;
  L.NP = NP;
  L.logH2 = ceil_log2(2ull * k);
  Bump b;
  L.ukey = b.take<unsigned char>(U * kb);
  L.ucnt = b.take<uint32_t>(U);
  L.uerr = b.take<uint32_t>(U);
  L.dead = b.take<uint8_t>(k);
  L.ht = b.take<uint32_t>((size_t)1 << L.logH2);
  L.x = b.take<unsigned char>((size_t)NP * (8 + kb));
  L.total = b.bytes();
  return L;
}

#ifdef PSS_MSTATS  // debug build only (tools/merge_stats.py): per-phase SM cycles of a COMBINE
__device__ unsigned long long g_m_stats[16][16];  // [ceil_log2(nblocks)][phase]
}  // namespace pss
extern "C" int pss_debug_mstats(unsigned long long* out, int reset) {
  cudaMemcpyFromSymbol(out, pss::g_m_stats, sizeof(pss::g_m_stats));
  if (reset) {
    static unsigned long long z[16][16] = {};
    cudaMemcpyToSymbol(pss::g_m_stats, z, sizeof(z));
  }
  return (int)cudaGetLastError();
}
namespace pss {
__device__ __forceinline__ void m_tick(int ph, uint32_t lv) {
  __shared__ long long prev;
  if (threadIdx.x == 0) {
    const long long t = clock64();
    if (ph >= 0) atomicAdd(&g_m_stats[lv & 15][ph], (unsigned long long)(t - prev));
    prev = t;
  }
}
#else
__device__ __forceinline__ void m_tick(int, uint32_t) {}
#endif


template <int NT>
__device__ __forceinline__ uint32_t block_reduce(uint32_t v, uint32_t* red, bool is_min) {
  v = is_min ? __reduce_min_sync(PSS_FULL, v) : __reduce_add_sync(PSS_FULL, v);
  constexpr int NW = NT / 32;
  __syncthreads();
  if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = v;
  __syncthreads();
  uint32_t r = is_min ? 0xffffffffu : 0u;
#pragma unroll
  for (int i = 0; i < NW; ++i) r = is_min ? min(r, red[i]) : r + red[i];
  __syncthreads();
  return r;
}

// sort element: (hi = ~count, lo = item) ascending == canonical order; idx = union position
template <typename KT>
struct SE {
  uint32_t hi;
  KT lo;
  uint32_t idx;
};
template <typename KT>
__device__ __forceinline__ bool se_less(const SE<KT>& a, const SE<KT>& b) {
  return a.hi < b.hi || (a.hi == b.hi && (a.lo < b.lo || (a.lo == b.lo && a.idx < b.idx)));
}
template <typename KT>
__device__ __forceinline__ SE<KT> se_shfl_xor(const SE<KT>& e, int m) {
  SE<KT> r;
  r.hi = __shfl_xor_sync(PSS_FULL, e.hi, m);
  r.lo = __shfl_xor_sync(PSS_FULL, e.lo, m);
  r.idx = __shfl_xor_sync(PSS_FULL, e.idx, m);
  return r;
}

// bitonic sort of NT*EPT elements, element i = t*EPT + j held by thread t in v[j]
template <typename KT, int NT, int EPT>
__device__ __forceinline__ void bitonic(SE<KT> (&v)[EPT], uint32_t* xhi, KT* xlo, uint32_t* xidx) {
  constexpr uint32_t NP = NT * EPT;
  const uint32_t t = threadIdx.x;
#pragma unroll 1
  for (uint32_t size = 2; size <= NP; size <<= 1) {
#pragma unroll 1
    for (uint32_t stride = size >> 1; stride > 0; stride >>= 1) {
      if (stride < EPT) {  // partner in the same thread (compile-time register indices)
#pragma unroll
        for (int s = 1; s < EPT; s <<= 1) {
          if ((uint32_t)s == stride) {
#pragma unroll
            for (int j = 0; j < EPT; ++j) {
              const int jp = j ^ s;
              if (jp > j) {
                const uint32_t i = t * EPT + j;
                const bool asc = (i & size) == 0;
                if (se_less(v[jp], v[j]) == asc) {
                  const SE<KT> tmp = v[j];
                  v[j] = v[jp];
                  v[jp] = tmp;
                }
              }
            }
          }
        }
      } else if (stride < 32u * EPT) {  // partner in the same warp
        const int lm = (int)(stride / EPT);
#pragma unroll
        for (int j = 0; j < EPT; ++j) {
          const uint32_t i = t * EPT + j;
          const SE<KT> o = se_shfl_xor(v[j], lm);
          const bool asc = (i & size) == 0;
          const bool lower = (i & stride) == 0;
          const bool take_min = lower == asc;
          const bool o_less = se_less(o, v[j]);
          if (o_less == take_min) v[j] = o;
        }
      } else {  // through shared memory
#pragma unroll
        for (int j = 0; j < EPT; ++j) {
          const uint32_t i = t * EPT + j;
          xhi[i] = v[j].hi;
          xlo[i] = v[j].lo;
          xidx[i] = v[j].idx;
        }
        __syncthreads();
#pragma unroll
        for (int j = 0; j < EPT; ++j) {
          const uint32_t i = t * EPT + j;
          const uint32_t p = i ^ stride;
          SE<KT> o;
          o.hi = xhi[p];
          o.lo = xlo[p];
          o.idx = xidx[p];
          const bool asc = (i & size) == 0;
          const bool take_min = ((i & stride) == 0) == asc;
          if (se_less(o, v[j]) == take_min) v[j] = o;
        }
        __syncthreads();
      }
    }
  }
}

// bitonic sort of NP (power of two) elements held in shared memory (large k)
template <typename KT, int NT>
__device__ __forceinline__ void bitonic_smem(uint32_t NP, uint32_t* xhi, KT* xlo, uint32_t* xidx) {
  for (uint32_t size = 2; size <= NP; size <<= 1) {
    for (uint32_t stride = size >> 1; stride > 0; stride >>= 1) {
      for (uint32_t i = threadIdx.x; i < NP / 2; i += NT) {
        const uint32_t p = 2 * i - (i & (stride - 1));
        const uint32_t q = p + stride;
        const bool asc = (p & size) == 0;
        const SE<KT> ep{xhi[p], xlo[p], xidx[p]};
        const SE<KT> eq{xhi[q], xlo[q], xidx[q]};
        if (se_less(eq, ep) == asc) {
          xhi[p] = eq.hi;
          xlo[p] = eq.lo;
          xidx[p] = eq.idx;
          xhi[q] = ep.hi;
          xlo[q] = ep.lo;
          xidx[q] = ep.idx;
        }
      }
      __syncthreads();
    }
  }
}

// One radix-select pass over 8-bit digits: hist[0..256) holds the digit histogram of the
// elements still in play; finds the digit d at which the running count (from the top digit down
// when `from_top`, else from digit 0 up) reaches `need`, and the count strictly before d in that
// order. Result in hist[256] (d) and hist[257] (count before). Warp 0 only.
__device__ __forceinline__ void radix_pick(uint32_t* hist, uint32_t need, bool from_top) {
  const uint32_t lane = threadIdx.x & 31u;
  // lane l owns 8 consecutive digits in the scan order
  uint32_t h[8];
  uint32_t s = 0;
#pragma unroll
  for (int j = 0; j < 8; ++j) {
    const uint32_t dig = from_top ? 255u - (lane * 8 + j) : lane * 8 + j;
    h[j] = hist[dig];
    s += h[j];
  }
  uint32_t incl = s;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const uint32_t t = __shfl_up_sync(PSS_FULL, incl, o);
    if (lane >= (uint32_t)o) incl += t;
  }
  const uint32_t excl = incl - s;
  if (excl < need && need <= incl) {
    uint32_t run = excl;
#pragma unroll
    for (int j = 0; j < 8; ++j) {
      if (run < need && need <= run + h[j]) {
        hist[256] = from_top ? 255u - (lane * 8 + j) : lane * 8 + j;
        hist[257] = run;
      }
      run += h[j];
    }
  }
}

// counters tied at the threshold count ranked by brute force (each against all) up to this many
constexpr uint32_t TIE_RANK_MAX = 128;

// warp-aggregated append: lanes with `take` get consecutive positions from *ctr (one atomic per
// warp); returns this lane's position (undefined if !take). All lanes of the warp must call it.
__device__ __forceinline__ uint32_t warp_append(uint32_t* ctr, bool take) {
  const uint32_t b = __ballot_sync(PSS_FULL, take);
  if (!b) return 0;
  const uint32_t lead = (uint32_t)(__ffs(b) - 1);
  uint32_t off = 0;
  if ((threadIdx.x & 31u) == lead) off = atomicAdd(ctr, (uint32_t)__popc(b));
  off = __shfl_sync(PSS_FULL, off, lead);
  return off + (uint32_t)__popc(b & lanemask_lt());
}

// Prune(k) for an internal tree node: the k greatest counters by (count desc, item asc) as a
// set, in no particular order (COMBINE does not depend on the order of its inputs).
//   1. live count and live min/max count (one block reduction);
//   2. threshold count C by radix select on 8-bit digits, from the highest digit in which the
//      live minimum and maximum differ (the digits above are common to all counters);
//   3. the counters with count == C are compacted into a list (tl = union index, tkey = item);
//      if more of them are tied than still needed, the threshold item K is the need-th smallest
//      item of the list: by brute-force ranking for short lists, else by radix select on it;
//   4. the selected counters are appended to the output (warp-aggregated positions).
template <typename KT, int NT>
__device__ void select_topk_write(uint32_t N, uint32_t n1, uint32_t k, const KT* ukey,
                                  const uint32_t* ucnt, const uint32_t* uerr, const uint8_t* dead,
                                  uint32_t* hist, uint32_t* red, uint32_t* tl, KT* tkey, KT* oi,
                                  uint32_t* oc, uint32_t* oe, uint32_t* osize, uint32_t lv) {
  constexpr int NW = NT / 32;
  __shared__ KT kres;
  const uint32_t tid = threadIdx.x, lane = tid & 31u, warp = tid >> 5;
  // tkey == nullptr: the tied items are read through their indices (the tree kernel of large
  // summaries keeps no tkey array and puts tl over the hash table, free by now)
  auto tie_key = [&](uint32_t j) -> KT { return tkey ? tkey[j] : ukey[tl[j]]; };
  uint32_t live = 0, mn = 0xffffffffu, mx = 0;
  for (uint32_t i = tid; i < N; i += NT) {
    if (i >= n1 && dead[i - n1]) continue;
    const uint32_t c = ucnt[i];
    ++live;
    mn = min(mn, c);
    mx = max(mx, c);
  }
  live = __reduce_add_sync(PSS_FULL, live);
  mn = __reduce_min_sync(PSS_FULL, mn);
  mx = __reduce_max_sync(PSS_FULL, mx);
  __syncthreads();
  if (lane == 0) {
    red[warp] = live;
    red[NW + warp] = mn;
    red[2 * NW + warp] = mx;
  }
  if (tid == 0) {
    hist[258] = 0;
    hist[259] = 0;
  }
  // radix passes alternate between two histograms: a pass clears the next one while it fills
  // its own, so a pass needs two barriers instead of four
  uint32_t* const hb = hist + 260;
  uint32_t pb = 0;
  for (uint32_t b = tid; b < 256; b += NT) hb[b] = 0;
  __syncthreads();
  uint32_t Lv = 0;
  mn = 0xffffffffu;
  mx = 0;
#pragma unroll
  for (int w = 0; w < NW; ++w) {
    Lv += red[w];
    mn = min(mn, red[NW + w]);
    mx = max(mx, red[2 * NW + w]);
  }
  m_tick(5, lv);
  const bool all = Lv <= k;
  uint32_t need = k;
  uint32_t C = 0;       // threshold count
  KT K = (KT)0;         // threshold item among count == C (inclusive)
  bool all_eq = true;   // take every counter with count == C
  if (!all) {
    if (mn == mx) {
      C = mn;
    } else {
      const int top = 31 - __clz(mn ^ mx);
      int shift = top / 8 * 8;
      uint32_t mask = shift >= 24 ? 0u : ~((1u << (shift + 8)) - 1u);
      C = mn & mask;
      for (; shift >= 0; shift -= 8, ++pb) {
        uint32_t* const cur = hb + 258 * (pb & 1u);
        uint32_t* const nxt = hb + 258 * ((pb + 1) & 1u);
        for (uint32_t b = tid; b < 256; b += NT) nxt[b] = 0;
        for (uint32_t i = tid; i < N; i += NT) {
          if (i >= n1 && dead[i - n1]) continue;
          const uint32_t c = ucnt[i];
          if ((c & mask) == C) atomicAdd(&cur[(c >> shift) & 255u], 1u);
        }
        __syncthreads();
        if (tid < 32) radix_pick(cur, need, true);
        __syncthreads();
        need -= cur[257];
        C |= cur[256] << shift;
        mask |= 255u << shift;
      }
    }
    m_tick(6, lv);
    // the counters with count == C, `need` of which are taken (the smallest items)
    for (uint32_t base = warp * 32; base < N; base += NT) {
      const uint32_t i = base + lane;
      const bool t = i < N && !(i >= n1 && dead[i - n1]) && ucnt[i] == C;
      const uint32_t o = warp_append(&hist[259], t);
      if (t) {
        tl[o] = i;
        if (tkey) tkey[o] = ukey[i];
      }
    }
    __syncthreads();
    const uint32_t E = hist[259];
    all_eq = E == need;
    if (!all_eq) {
      if (E <= TIE_RANK_MAX) {  // items in the union are distinct: ranks are exact
        for (uint32_t j = tid; j < E; j += NT) {
          const KT x = tie_key(j);
          uint32_t r = 0;
          for (uint32_t u = 0; u < E; ++u) r += tie_key(u) < x;
          if (r == need - 1) kres = x;
        }
        __syncthreads();
        K = kres;
      } else {
        KT kmask = 0;
        for (int shift = 8 * (int)sizeof(KT) - 8; shift >= 0; shift -= 8, ++pb) {
          uint32_t* const cur = hb + 258 * (pb & 1u);
          uint32_t* const nxt = hb + 258 * ((pb + 1) & 1u);
          for (uint32_t b = tid; b < 256; b += NT) nxt[b] = 0;
          for (uint32_t j = tid; j < E; j += NT) {
            const KT x = tie_key(j);
            if ((x & kmask) == K) atomicAdd(&cur[(uint32_t)(x >> shift) & 255u], 1u);
          }
          __syncthreads();
          if (tid < 32) radix_pick(cur, need, false);
          __syncthreads();
          need -= cur[257];
          K |= (KT)cur[256] << shift;
          kmask |= (KT)255 << shift;
        }
      }
    }
  }
  m_tick(7, lv);
  for (uint32_t base = warp * 32; base < N; base += NT) {
    const uint32_t i = base + lane;
    const bool lvv = i < N && !(i >= n1 && dead[i - n1]);
    const uint32_t c = lvv ? ucnt[i] : 0u;
    const bool tk = lvv && (all || c > C || (c == C && (all_eq || ukey[i] <= K)));
    const uint32_t o = warp_append(&hist[258], tk);
    if (tk) {
      oi[o] = ukey[i];
      oc[o] = c;
      oe[o] = uerr[i];
    }
  }
  __syncthreads();
  if (tid == 0) *osize = hist[258];
  m_tick(8, lv);
}

// loads of summaries: read-only path for inputs written by earlier launches (CG = false), L2
// (bypassing L1, which is not coherent across SMs) for nodes written by other CTAs of the same
// launch (CG = true)
template <bool CG, typename T>
__device__ __forceinline__ T ldx(const T* p) {
  if constexpr (CG)
    return __ldcg(p);
  else
    return __ldg(p);
}

// shared-memory views of one COMBINE's working set
template <typename KT>
struct CombSmem {
  KT* ukey;
  uint32_t* ucnt;
  uint32_t* uerr;
  uint8_t* dead;
  uint32_t* ht;
  uint32_t* xhi;
  uint32_t* xidx;
  KT* xlo;
  uint32_t* tl;  // Prune(k)'s list of counters tied at the threshold: indices, items
  KT* tkey;
  uint32_t* red;
  uint32_t* hist;
};
template <typename KT>
__device__ __forceinline__ CombSmem<KT> comb_smem(const CombArgs& a, unsigned char* base,
                                                  uint32_t* red, uint32_t* hist) {
  CombSmem<KT> m;
  m.ukey = reinterpret_cast<KT*>(base);
  m.ucnt = reinterpret_cast<uint32_t*>(base + a.o_ucnt);
  m.uerr = reinterpret_cast<uint32_t*>(base + a.o_uerr);
  m.dead = reinterpret_cast<uint8_t*>(base + a.o_dead);
  m.ht = reinterpret_cast<uint32_t*>(base + a.o_ht);
  m.xhi = reinterpret_cast<uint32_t*>(base + a.o_x);
  m.xidx = m.xhi + a.NP;
  m.xlo = reinterpret_cast<KT*>(m.xidx + a.NP);
  m.tl = a.no_x ? m.ht : m.xidx;  // no exchange buffer: the hash table's space, indices only
  m.tkey = a.no_x ? nullptr : m.xlo;
  m.red = red;
  m.hist = hist;
  return m;
}

// One COMBINE (Alg. 2): node li of `ina` with node ri of `inb` (if has_r) into node blk of `o`.
// EPT > 0: the root sort keeps EPT elements per thread in registers; EPT == 0: shared-memory sort
template <typename KT, int NT, int EPT, bool CG>
__device__ void combine_node(const CombArgs& a, const NodeRef& ina, uint32_t li,
                             const NodeRef& inb, uint32_t ri, bool has_r, const NodeOut& o,
                             uint32_t blk, const CombSmem<KT>& sm, uint32_t lv) {
  const uint32_t NP = a.NP;
  const uint32_t k = a.k;
  const uint32_t tid = threadIdx.x;
  KT* const ukey = sm.ukey;
  uint32_t* const ucnt = sm.ucnt;
  uint32_t* const uerr = sm.uerr;
  uint8_t* const dead = sm.dead;
  uint32_t* const ht = sm.ht;
  uint32_t* const xhi = sm.xhi;
  uint32_t* const xidx = sm.xidx;
  KT* const xlo = sm.xlo;
  uint32_t* const red = sm.red;
  uint32_t* const hist = sm.hist;
  (void)NP;
  (void)xhi;
  const uint32_t n1 = ldx<CG>(ina.sizes + li);
  const uint32_t n2 = has_r ? ldx<CG>(inb.sizes + ri) : 0u;
  const KT* i1 = reinterpret_cast<const KT*>(ina.items) + (size_t)li * k;
  const uint32_t* c1 = ina.counts + (size_t)li * k;
  const uint32_t* e1 = ina.errs + (size_t)li * k;
  KT* oi = reinterpret_cast<KT*>(o.items) + (size_t)blk * k;
  uint32_t* oc = o.counts + (size_t)blk * k;
  uint32_t* oe = o.errs + (size_t)blk * k;

  if (!has_r && !a.canon_single) {  // odd last node carried up unchanged (R6)
    for (uint32_t t = tid; t < n1; t += NT) {
      oi[t] = ldx<CG>(i1 + t);
      oc[t] = ldx<CG>(c1 + t);
      oe[t] = ldx<CG>(e1 + t);
    }
    if (tid == 0) o.sizes[blk] = n1;
    return;
  }
  const KT* i2 = has_r ? reinterpret_cast<const KT*>(inb.items) + (size_t)ri * k : nullptr;
  const uint32_t* c2 = has_r ? inb.counts + (size_t)ri * k : nullptr;
  const uint32_t* e2 = has_r ? inb.errs + (size_t)ri * k : nullptr;
  // S2's index: sized from S2's actual size (load <= 1/2), at most the planned capacity, so that
  // unfull summaries (large k) clear and probe a table of their own size
  uint32_t lh = 5;
  while (lh < a.logH2 && (1u << lh) < 2u * n2) ++lh;
  const uint32_t H2 = 1u << lh, hmask = H2 - 1u;

  // stage S1 -> u[0, n1), S2 -> u[n1, n1 + n2); minima (Alg. 2 l.2-3, R4). The loads of
  // both summaries are issued before their stores.
  uint32_t mn1 = 0xffffffffu, mn2 = 0xffffffffu;
  for (uint32_t t = tid; t < max(n1, n2); t += NT) {
    const bool h1 = t < n1, h2 = t < n2;
    KT x1 = 0, x2 = 0;
    uint32_t cc1 = 0, ee1 = 0, cc2 = 0, ee2 = 0;
    if (h1) {
      x1 = ldx<CG>(i1 + t);
      cc1 = ldx<CG>(c1 + t);
      ee1 = ldx<CG>(e1 + t);
    }
    if (h2) {
      x2 = ldx<CG>(i2 + t);
      cc2 = ldx<CG>(c2 + t);
      ee2 = ldx<CG>(e2 + t);
    }
    if (h1) {
      ukey[t] = x1;
      ucnt[t] = cc1;
      uerr[t] = ee1;
      mn1 = min(mn1, cc1);
    }
    if (h2) {
      ukey[n1 + t] = x2;
      ucnt[n1 + t] = cc2;
      uerr[n1 + t] = ee2;
      dead[t] = 0;
      mn2 = min(mn2, cc2);
    }
  }
  for (uint32_t h = tid; h < H2; h += NT) ht[h] = 0xffffffffu;
  mn1 = __reduce_min_sync(PSS_FULL, mn1);
  mn2 = __reduce_min_sync(PSS_FULL, mn2);
  __syncthreads();
  if ((tid & 31u) == 0) {
    red[tid >> 5] = mn1;
    red[NT / 32 + (tid >> 5)] = mn2;
  }
  __syncthreads();
  uint32_t m1r = 0xffffffffu, m2r = 0xffffffffu;
#pragma unroll
  for (int w = 0; w < NT / 32; ++w) {
    m1r = min(m1r, red[w]);
    m2r = min(m2r, red[NT / 32 + w]);
  }
  const uint32_t m1 = n1 == k ? m1r : 0u;
  const uint32_t m2 = n2 == k ? m2r : 0u;
  m_tick(0, lv);
  // index S2's items (Find of Alg. 2 l.5)
  for (uint32_t t = tid; t < n2; t += NT) {
    uint32_t h = hslot(ukey[n1 + t], lh);
    while (atomicCAS(&ht[h], 0xffffffffu, t) != 0xffffffffu) h = (h + 1u) & hmask;
  }
  __syncthreads();
  m_tick(1, lv);
  // counters of S1: matched -> f1 + f2 and Remove from S2; else f1 + m2 (Alg. 2 l.4-13)
  for (uint32_t t = tid; t < n1; t += NT) {
    const KT x = ukey[t];
    uint32_t h = hslot(x, lh);
    uint32_t j;
    while ((j = ht[h]) != 0xffffffffu && ukey[n1 + j] != x) h = (h + 1u) & hmask;
    if (j != 0xffffffffu) {
      ucnt[t] += ucnt[n1 + j];
      uerr[t] += uerr[n1 + j];
      dead[j] = 1;
    } else {
      ucnt[t] += m2;
      uerr[t] += m2;
    }
  }
  __syncthreads();
  m_tick(2, lv);
  // remaining counters of S2: f2 + m1 (Alg. 2 l.14-18)
  for (uint32_t t = tid; t < n2; t += NT)
    if (!dead[t]) {
      ucnt[n1 + t] += m1;
      uerr[n1 + t] += m1;
    }
  __syncthreads();
  m_tick(3, lv);
  // Prune(k) (Alg. 2 l.19): order by (count desc, item asc), keep the first k (R5)
  const uint32_t N = n1 + n2;
  if (!a.sort_out) {  // internal tree node: the top-k set
    select_topk_write<KT, NT>(N, n1, k, ukey, ucnt, uerr, dead, hist, red, sm.tl, sm.tkey, oi, oc,
                              oe, o.sizes + blk, lv);
    if (tid == 0) {
#ifdef PSS_MSTATS
      atomicAdd(&g_m_stats[lv & 15][15], 1ull);
#endif
    }
    return;
  }
  if constexpr (EPT > 0) {
    SE<KT> v[EPT];
    uint32_t live = 0;
#pragma unroll
    for (int j = 0; j < EPT; ++j) {
      const uint32_t i = tid * EPT + j;
      const bool valid = i < N && !(i >= n1 && dead[i - n1]);
      v[j].hi = valid ? ~ucnt[i] : 0xffffffffu;  // valid counts are >= 1: ~count < all-ones
      v[j].lo = valid ? ukey[i] : (KT)0;
      v[j].idx = valid ? i : 0xffffffffu;
      live += valid;
    }
    const uint32_t Lv = block_reduce<NT>(live, red, false);
    bitonic<KT, NT, EPT>(v, xhi, xlo, xidx);
    const uint32_t outn = min(Lv, k);
#pragma unroll
    for (int j = 0; j < EPT; ++j) {
      const uint32_t i = tid * EPT + j;
      if (i < outn) {
        const uint32_t u = v[j].idx;
        oi[i] = ukey[u];
        oc[i] = ucnt[u];
        oe[i] = uerr[u];
      }
    }
    if (tid == 0) o.sizes[blk] = outn;
  } else {
    uint32_t live = 0;
    for (uint32_t i = tid; i < NP; i += NT) {
      const bool valid = i < N && !(i >= n1 && dead[i - n1]);
      xhi[i] = valid ? ~ucnt[i] : 0xffffffffu;
      xlo[i] = valid ? ukey[i] : (KT)0;
      xidx[i] = valid ? i : 0xffffffffu;
      live += valid;
    }
    const uint32_t Lv = block_reduce<NT>(live, red, false);
    bitonic_smem<KT, NT>(NP, xhi, xlo, xidx);
    const uint32_t outn = min(Lv, k);
    for (uint32_t i = tid; i < outn; i += NT) {
      const uint32_t u = xidx[i];
      oi[i] = ukey[u];
      oc[i] = ucnt[u];
      oe[i] = uerr[u];
    }
    if (tid == 0) o.sizes[blk] = outn;
  }
}

template <typename KT, bool G, int NT, int EPT>
__global__ void __launch_bounds__(NT) combine_kernel(const CombArgs a) {
  extern __shared__ __align__(128) unsigned char smem[];
  __shared__ uint32_t red[3 * (NT / 32)];
  __shared__ uint32_t hist[260 + 2 * 258];
  unsigned char* base = G ? a.gscratch + (size_t)blockIdx.x * a.gstride : smem;
  const CombSmem<KT> sm = comb_smem<KT>(a, base, red, hist);
  const uint32_t lv = ceil_log2(a.nblocks);
  for (uint32_t blk = blockIdx.x; blk < a.nblocks; blk += gridDim.x) {
    m_tick(-1, lv);
    const uint32_t li = blk * a.a_mul + a.a_add;
    const bool has_r = blk < a.nright;
    const uint32_t ri = blk * a.b_mul + a.b_add;
    combine_node<KT, NT, EPT, false>(a, a.a, li, a.b, ri, has_r, a.o, blk, sm, lv);
    __syncthreads();
  }
}

// The internal levels of the tree in one persistent launch: CTAs take COMBINE tasks in level
// order from a queue (task t = node t of the concatenated levels); a task waits until its
// children's done flags are set, then runs and sets its own. Children always have smaller task
// ids and are held by running CTAs, so there is no deadlock whatever the residency; levels
// overlap, and there are no launch boundaries between them.
struct TreeArgs {
  CombArgs a;        // k, table sizes, shared-memory offsets
  NodeRef leaves;
  NodeOut nodes;     // every internal node, indexed by task id
  uint32_t nlev;     // internal levels
  uint32_t off[33];  // first task of each level; off[nlev] = number of tasks
  uint32_t cin[32];  // input nodes of each level
  uint32_t* flags;   // per task: 1 once its node is written
  uint32_t* queue;
  const uint32_t* leaf_flags;  // non-null: leaf r is ready once leaf_flags[r] != 0 (K1 overlap)
};

template <typename KT, int NT>
__global__ void __launch_bounds__(NT, 1536 / NT) tree_kernel(const TreeArgs ta) {
  extern __shared__ __align__(128) unsigned char smem[];
  __shared__ uint32_t red[3 * (NT / 32)];
  __shared__ uint32_t hist[260 + 2 * 258];
  __shared__ uint32_t task;
  const CombSmem<KT> sm = comb_smem<KT>(ta.a, smem, red, hist);
  const uint32_t ntasks = ta.off[ta.nlev];
  const NodeRef nodes_in{ta.nodes.items, ta.nodes.counts, ta.nodes.errs, ta.nodes.sizes};
  while (true) {
    if (threadIdx.x == 0) task = atomicAdd(ta.queue, 1u);
    __syncthreads();
    const uint32_t t = task;
    if (t >= ntasks) break;
    uint32_t j = 0;
    while (t >= ta.off[j + 1]) ++j;
    const uint32_t i = t - ta.off[j];
    const bool has_r = 2 * i + 1 < ta.cin[j];
    const NodeRef& in = j == 0 ? ta.leaves : nodes_in;
    const uint32_t base = j == 0 ? 0u : ta.off[j - 1];
    if (threadIdx.x == 0 && (j > 0 || ta.leaf_flags)) {  // acquire the children
      const uint32_t* fl = (j > 0 ? ta.flags + base : ta.leaf_flags) + 2 * i;
      while (ld_acquire(fl) == 0 || (has_r && ld_acquire(fl + 1) == 0)) __nanosleep(64);
    }
    __syncthreads();
    CombArgs a = ta.a;
    a.sort_out = 0;
    a.canon_single = 0;
    combine_node<KT, NT, 0, true>(a, in, base + 2 * i, in, base + 2 * i + 1, has_r, ta.nodes, t,
                                  sm, j);
    __syncthreads();
    if (threadIdx.x == 0) {  // release the node
      __threadfence();
      st_release(ta.flags + t, 1u);
    }
  }
  // launched as a programmatic dependent of K1: complete only after K1 has (stream order for
  // whatever follows)
  if (ta.leaf_flags) pdl_wait_prerequisites();
}

// ------------------------------------------------------------------------------ host side
struct MPlan {
  bool g;
  int nt, ept;
  MLayout L;
  size_t smem;
  int grid_cap;
};

static MPlan m_plan(int kb, uint32_t k, const DevInfo& d) {
  MPlan p;
  uint32_t NP = 1u << ceil_log2(2ull * k);
  if (NP < 256) NP = 256;
  const char* nts = std::getenv("PSS_DEBUG_MERGE_NT");  // experiment hook
  const uint32_t ntmax = nts ? (uint32_t)std::atoi(nts) : 512u;
  p.nt = (int)std::min<uint32_t>(ntmax, NP / 2);
  if (NP / p.nt > 8) p.nt = (int)std::min<uint32_t>(1024, NP / 2);
  p.ept = (int)(NP / p.nt);
  p.L = m_layout(k, kb, NP);
  p.g = p.L.total > (size_t)d.smem_optin - 2048;
  p.smem = p.g ? 0 : p.L.total;
  p.grid_cap = p.g ? 2 * d.sms : 1 << 30;
  return p;
}

static void fill_comb_args(CombArgs& a, int, uint32_t k, const MPlan& p, void* ws) {
  a.k = k;
  a.gscratch = p.g ? static_cast<unsigned char*>(ws) : nullptr;
  a.gstride = p.L.total;
  a.o_ucnt = p.L.ucnt;
  a.o_uerr = p.L.uerr;
  a.o_dead = p.L.dead;
  a.o_ht = p.L.ht;
  a.o_x = p.L.x;
  a.logH2 = p.L.logH2;
  a.NP = p.L.NP;
  a.no_x = 0;
}

template <typename KT, bool G, int NT, int EPT>
static void launch_comb(const CombArgs& a, int grid, size_t smem, cudaStream_t s) {
  auto kern = combine_kernel<KT, G, NT, EPT>;
  if (!G) allow_max_smem(kern, dev_info());
  kern<<<grid, NT, G ? 0 : smem, s>>>(a);
}

template <typename KT, bool G>
static bool dispatch_comb(const CombArgs& a, int grid, const MPlan& p, cudaStream_t s) {
  switch (p.nt * 100 + p.ept) {
    case 128 * 100 + 2: launch_comb<KT, G, 128, 2>(a, grid, p.smem, s); return true;
    case 256 * 100 + 2: launch_comb<KT, G, 256, 2>(a, grid, p.smem, s); return true;
    case 512 * 100 + 2: launch_comb<KT, G, 512, 2>(a, grid, p.smem, s); return true;
    case 512 * 100 + 4: launch_comb<KT, G, 512, 4>(a, grid, p.smem, s); return true;
    case 512 * 100 + 8: launch_comb<KT, G, 512, 8>(a, grid, p.smem, s); return true;
    case 256 * 100 + 4: launch_comb<KT, G, 256, 4>(a, grid, p.smem, s); return true;
    case 256 * 100 + 8: launch_comb<KT, G, 256, 8>(a, grid, p.smem, s); return true;
    case 1024 * 100 + 2: launch_comb<KT, G, 1024, 2>(a, grid, p.smem, s); return true;
    case 1024 * 100 + 4: launch_comb<KT, G, 1024, 4>(a, grid, p.smem, s); return true;
    case 1024 * 100 + 8: launch_comb<KT, G, 1024, 8>(a, grid, p.smem, s); return true;
  }
  if (p.nt == 1024 && p.ept > 8) {
    launch_comb<KT, G, 1024, 0>(a, grid, p.smem, s);
    return true;
  }
  return false;
}

// ---- canonical order (R5: count descending, then item ascending) of one summary by ranks, for
// summaries too large for a CTA's shared memory (k beyond ~2000). A summary holds distinct
// items, so the canonical order is a permutation: the rank of counter i is the number of
// counters before it; a 2-D grid (counter tiles x slices of the summary) adds partial ranks,
// then each counter is written at its rank. Replaces the single-CTA bitonic sort over global
// scratch (C4-k20000: 2.2 ms for the root).
constexpr int RK_NT = 256, RK_SLICE = 1024;
template <typename KT>
__global__ void __launch_bounds__(RK_NT) rank_partial_kernel(const KT* items,
                                                             const uint32_t* counts,
                                                             const uint32_t* size_p,
                                                             uint32_t* rank) {
  __shared__ KT sx[RK_NT];
  __shared__ uint32_t sc[RK_NT];
  const uint32_t size = *size_p;
  const uint32_t i = blockIdx.x * RK_NT + threadIdx.x;
  const uint32_t j0 = blockIdx.y * RK_SLICE, j1 = min(size, j0 + RK_SLICE);
  if (blockIdx.x * RK_NT >= size || j0 >= size) return;
  const bool act = i < size;
  const uint32_t c = act ? counts[i] : 0u;
  const KT x = act ? items[i] : KT(0);
  uint32_t r = 0;
  for (uint32_t t = j0; t < j1; t += RK_NT) {
    __syncthreads();
    if (t + threadIdx.x < j1) {
      sx[threadIdx.x] = items[t + threadIdx.x];
      sc[threadIdx.x] = counts[t + threadIdx.x];
    }
    __syncthreads();
    const uint32_t m = min((uint32_t)RK_NT, j1 - t);
    for (uint32_t u = 0; u < m; ++u) r += canon_before(sc[u], sx[u], c, x);
  }
  if (act && r) atomicAdd(&rank[i], r);
}
template <typename KT>
__global__ void rank_scatter_kernel(const KT* items, const uint32_t* counts, const uint32_t* errs,
                                    const uint32_t* size_p, const uint32_t* rank, KT* oi,
                                    uint32_t* oc, uint32_t* oe, uint32_t* osize) {
  const uint32_t size = *size_p;
  const uint32_t i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i == 0) *osize = size;
  if (i >= size) return;
  const uint32_t r = rank[i];
  oi[r] = items[i];
  oc[r] = counts[i];
  oe[r] = errs[i];
}
// in = one summary (<= k counters), out = the same counters in canonical order; rank: k words
static cudaError_t canon_rank_sort(int kb, uint32_t k, NodeRef in, NodeOut out, uint32_t* rank,
                                   cudaStream_t s) {
  cudaError_t e = cudaMemsetAsync(rank, 0, (size_t)k * sizeof(uint32_t), s);
  if (e != cudaSuccess) return e;
  const dim3 grid((k + RK_NT - 1) / RK_NT, (k + RK_SLICE - 1) / RK_SLICE);
  const int sg = (int)((k + 255) / 256);
  if (kb == 4) {
    rank_partial_kernel<uint32_t><<<grid, RK_NT, 0, s>>>(
        static_cast<const uint32_t*>(in.items), in.counts, in.sizes, rank);
    rank_scatter_kernel<uint32_t><<<sg, 256, 0, s>>>(
        static_cast<const uint32_t*>(in.items), in.counts, in.errs, in.sizes, rank,
        static_cast<uint32_t*>(out.items), out.counts, out.errs, out.sizes);
  } else {
    rank_partial_kernel<uint64_t><<<grid, RK_NT, 0, s>>>(
        static_cast<const uint64_t*>(in.items), in.counts, in.sizes, rank);
    rank_scatter_kernel<uint64_t><<<sg, 256, 0, s>>>(
        static_cast<const uint64_t*>(in.items), in.counts, in.errs, in.sizes, rank,
        static_cast<uint64_t*>(out.items), out.counts, out.errs, out.sizes);
  }
  return cudaGetLastError();
}
// bytes of the unsorted-root staging + ranks (large-k path only)
static size_t rank_tmp_bytes(int kb, uint32_t k) {
  return align_up((size_t)k * kb, 256) + 2 * align_up((size_t)k * 4, 256) + 256 +
         align_up((size_t)k * 4, 256);
}
struct RankTmp {
  NodeOut node;
  uint32_t* rank;
};
static RankTmp rank_tmp(void* base, int kb, uint32_t k) {
  unsigned char* w = static_cast<unsigned char*>(base);
  RankTmp t;
  size_t o = 0;
  t.node.items = w + o;
  o += align_up((size_t)k * kb, 256);
  t.node.counts = reinterpret_cast<uint32_t*>(w + o);
  o += align_up((size_t)k * 4, 256);
  t.node.errs = reinterpret_cast<uint32_t*>(w + o);
  o += align_up((size_t)k * 4, 256);
  t.node.sizes = reinterpret_cast<uint32_t*>(w + o);
  o += 256;
  t.rank = reinterpret_cast<uint32_t*>(w + o);
  return t;
}

static size_t scratch_bytes(int kb, uint32_t k, const DevInfo& d);
static cudaError_t combine_run(int kb, uint32_t k, CombArgs a, void* ws, cudaStream_t s,
                               const DevInfo& d) {
  MPlan p = m_plan(kb, k, d);
  if (p.g && a.sort_out && a.nblocks == 1) {
    // large k: the set by the level kernel's radix selection, the order by ranks (the staging
    // node and ranks follow the COMBINE scratch in ws)
    const RankTmp t = rank_tmp(static_cast<unsigned char*>(ws) + align_up(scratch_bytes(kb, k, d), 256), kb, k);
    const NodeOut final_out = a.o;
    if (a.canon_single && a.nright == 0) {  // COMBINE(S, empty): S itself, reordered
      return canon_rank_sort(kb, k, a.a, final_out, t.rank, s);
    }
    a.o = t.node;
    a.sort_out = 0;
    a.canon_single = 0;
    cudaError_t e = combine_run(kb, k, a, ws, s, d);
    if (e != cudaSuccess) return e;
    return canon_rank_sort(kb, k, NodeRef{t.node.items, t.node.counts, t.node.errs, t.node.sizes},
                           final_out, t.rank, s);
  }
  fill_comb_args(a, kb, k, p, ws);
  if (a.nblocks == 0) return cudaSuccess;
  const int grid = (int)std::min<uint32_t>(a.nblocks, (uint32_t)p.grid_cap);
  bool ok;
  if (kb == 4)
    ok = p.g ? dispatch_comb<uint32_t, true>(a, grid, p, s) : dispatch_comb<uint32_t, false>(a, grid, p, s);
  else
    ok = p.g ? dispatch_comb<uint64_t, true>(a, grid, p, s) : dispatch_comb<uint64_t, false>(a, grid, p, s);
  if (!ok) return cudaErrorInvalidConfiguration;
  return cudaGetLastError();
}

static size_t scratch_bytes(int kb, uint32_t k, const DevInfo& d) {
  MPlan p = m_plan(kb, k, d);
  return p.g ? p.L.total * (size_t)p.grid_cap : 0;
}

size_t combine_ws(int kb, uint32_t k, uint32_t, const DevInfo& d) {
  return align_up(scratch_bytes(kb, k, d), 256) + 256 +
         (m_plan(kb, k, d).g ? rank_tmp_bytes(kb, k) : 0);
}

cudaError_t combine_launch(int kb, uint32_t k, uint32_t count, const void* a_items,
                           const uint32_t* a_counts, const uint32_t* a_errs,
                           const uint32_t* a_sizes, const void* b_items, const uint32_t* b_counts,
                           const uint32_t* b_errs, const uint32_t* b_sizes, void* o_items,
                           uint32_t* o_counts, uint32_t* o_errs, uint32_t* o_sizes, void* ws,
                           cudaStream_t s, const DevInfo& d) {
  CombArgs a{};
  a.a = {a_items, a_counts, a_errs, a_sizes};
  a.b = {b_items, b_counts, b_errs, b_sizes};
  a.o = {o_items, o_counts, o_errs, o_sizes};
  a.a_mul = 1;
  a.a_add = 0;
  a.b_mul = 1;
  a.b_add = 0;
  a.nblocks = count;
  a.nright = count;
  a.canon_single = 1;
  a.sort_out = 1;
  return combine_run(kb, k, a, ws, s, d);
}

// the fixed tree: internal levels (every COMBINE except the root), their first task ids and
// input counts; c_final = nodes entering the root COMBINE (1 only when P == 1)
struct TreePlan {
  uint32_t nlev = 0, ntasks = 0, c_final = 0;
  uint32_t off[33] = {};
  uint32_t cin[32] = {};
};
static TreePlan tree_plan(uint32_t P) {
  TreePlan t;
  uint32_t c = P;
  while (true) {
    const uint32_t cout = (c + 1) / 2;
    if (cout <= 1) break;
    t.off[t.nlev] = t.ntasks;
    t.cin[t.nlev] = c;
    t.ntasks += cout;
    ++t.nlev;
    c = cout;
  }
  t.off[t.nlev] = t.ntasks;
  t.c_final = c;
  return t;
}

// workspace of pss_merge: every internal node (task order), sizes, done flags, the task queue,
// and the global scratch of COMBINEs that do not fit shared memory
struct TreeWs {
  size_t items, counts, errs, sizes, flags, queue, scratch, total;
};
static TreeWs tree_ws(int kb, uint32_t k, uint32_t P, const DevInfo& d) {
  const TreePlan t = tree_plan(P);
  const size_t nn = std::max<uint32_t>(t.ntasks, 1);
  TreeWs w;
  Bump b;
  w.items = b.take<unsigned char>(nn * k * kb);
  w.counts = b.take<uint32_t>(nn * k);
  w.errs = b.take<uint32_t>(nn * k);
  w.sizes = b.take<uint32_t>(nn);
  w.flags = b.take<uint32_t>(nn);
  w.queue = b.take<uint32_t>(1);
  w.scratch = b.take<unsigned char>(align_up(scratch_bytes(kb, k, d), 256) +
                                     (m_plan(kb, k, d).g ? rank_tmp_bytes(kb, k) : 0));
  w.total = b.bytes();
  return w;
}

size_t merge_ws(int kb, uint32_t k, uint32_t P, const DevInfo& d) {
  return tree_ws(kb, k, P, d).total;
}

template <typename KT>
#ifndef PSS_TREE_NT
#define PSS_TREE_NT 512
#endif
static cudaError_t launch_tree(const TreeArgs& ta, const MPlan& p, const DevInfo& d,
                               cudaStream_t s) {
  constexpr int NT = PSS_TREE_NT;
  auto kern = tree_kernel<KT, NT>;
  allow_max_smem(kern, d);
  int nb = 0;
  if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&nb, kern, NT, p.smem) != cudaSuccess ||
      nb < 1)
    nb = 1;
  // Internal nodes need the exchange buffer only for Prune(k)'s tie list. When it costs
  // residency (k around 2000: one CTA per SM), the list goes over the hash table instead
  // (indices only) and the buffer is dropped: 2-3 CTAs per SM.
  size_t smem = p.smem;
  TreeArgs tb = ta;
  if (nb < 1536 / NT) {
    int nb2 = 0;
    if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&nb2, kern, NT, p.L.x) == cudaSuccess &&
        nb2 > nb) {
      nb = nb2;
      smem = p.L.x;
      tb.a.no_x = 1;
    }
  }
  const int grid = (int)std::min<uint64_t>(ta.off[ta.nlev], (uint64_t)nb * d.sms);
  if (!ta.leaf_flags) {
    kern<<<grid, NT, smem, s>>>(tb);
    return cudaGetLastError();
  }
  // overlapping K1: a programmatic dependent launch (K1 triggers it at its start; the tree's CTAs
  // are placed as K1's persistent CTAs exit and wait for their leaves through leaf_flags)
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(grid);
  cfg.blockDim = dim3(NT);
  cfg.dynamicSmemBytes = smem;
  cfg.stream = s;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  return cudaLaunchKernelEx(&cfg, kern, tb);
}

bool merge_tree_overlaps(int kb, uint32_t k, uint32_t P, const DevInfo& d) {
  return P >= 4 && !m_plan(kb, k, d).g && tree_plan(P).nlev > 0;
}

cudaError_t merge_tree_reset(int kb, uint32_t k, uint32_t P, void* ws, cudaStream_t s,
                             const DevInfo& d) {
  const TreeWs L = tree_ws(kb, k, P, d);
  unsigned char* w = static_cast<unsigned char*>(ws);
  return cudaMemsetAsync(w + L.flags, 0, (L.queue - L.flags) + sizeof(uint32_t), s);
}

cudaError_t merge_tree_launch(int kb, uint32_t k, uint32_t P, const void* items,
                              const uint32_t* counts, const uint32_t* errs, const uint32_t* sizes,
                              void* r_items, uint32_t* r_counts, uint32_t* r_errs,
                              uint32_t* r_sizes, void* ws, cudaStream_t s, const DevInfo& d,
                              const uint32_t* leaf_flags) {
  unsigned char* w = static_cast<unsigned char*>(ws);
  const TreeWs L = tree_ws(kb, k, P, d);
  if (leaf_flags && !merge_tree_overlaps(kb, k, P, d)) leaf_flags = nullptr;
  const TreePlan t = tree_plan(P);
  NodeOut nodes{w + L.items, reinterpret_cast<uint32_t*>(w + L.counts),
                reinterpret_cast<uint32_t*>(w + L.errs), reinterpret_cast<uint32_t*>(w + L.sizes)};
  void* scratch = w + L.scratch;
  NodeRef leaves{items, counts, errs, sizes};
  NodeOut root{r_items, r_counts, r_errs, r_sizes};
  if (P == 1) {  // root = the only leaf, in canonical order = COMBINE(S, empty)
    CombArgs a{};
    a.a = leaves;
    a.b = leaves;
    a.o = root;
    a.a_mul = 1;
    a.b_mul = 1;
    a.nblocks = 1;
    a.nright = 0;
    a.canon_single = 1;
    a.sort_out = 1;
    return combine_run(kb, k, a, scratch, s, d);
  }
  const MPlan p = m_plan(kb, k, d);
  if (t.nlev > 0) {
    if (!p.g) {  // all internal levels in one persistent launch
      cudaError_t e = cudaSuccess;
      if (!leaf_flags)  // else cleared before K1 (merge_tree_reset)
        e = cudaMemsetAsync(w + L.flags, 0, (L.queue - L.flags) + sizeof(uint32_t), s);
      if (e != cudaSuccess) return e;
      TreeArgs ta{};
      fill_comb_args(ta.a, kb, k, p, nullptr);
      ta.leaves = leaves;
      ta.nodes = nodes;
      ta.nlev = t.nlev;
      for (uint32_t i = 0; i <= t.nlev; ++i) ta.off[i] = t.off[i];
      for (uint32_t i = 0; i < t.nlev; ++i) ta.cin[i] = t.cin[i];
      ta.flags = reinterpret_cast<uint32_t*>(w + L.flags);
      ta.queue = reinterpret_cast<uint32_t*>(w + L.queue);
      ta.leaf_flags = leaf_flags;
      e = kb == 4 ? launch_tree<uint32_t>(ta, p, d, s) : launch_tree<uint64_t>(ta, p, d, s);
      if (e != cudaSuccess) return e;
    } else {  // summaries too large for shared memory: one launch per level
      for (uint32_t lv = 0; lv < t.nlev; ++lv) {
        CombArgs a{};
        a.a = lv == 0 ? leaves
                      : NodeRef{nodes.items, nodes.counts, nodes.errs, nodes.sizes};
        a.b = a.a;
        a.o = NodeOut{static_cast<unsigned char*>(nodes.items) + (size_t)t.off[lv] * k * kb,
                      nodes.counts + (size_t)t.off[lv] * k, nodes.errs + (size_t)t.off[lv] * k,
                      nodes.sizes + t.off[lv]};
        const uint32_t base = lv == 0 ? 0u : t.off[lv - 1];
        a.a_mul = 2;
        a.a_add = base;
        a.b_mul = 2;
        a.b_add = base + 1;
        a.nblocks = t.off[lv + 1] - t.off[lv];
        a.nright = t.cin[lv] / 2;
        a.canon_single = 0;
        a.sort_out = 0;
        const cudaError_t e = combine_run(kb, k, a, scratch, s, d);
        if (e != cudaSuccess) return e;
      }
    }
  }
  // the root (canonical order, R5)
  CombArgs a{};
  const uint32_t base = t.nlev == 0 ? 0u : t.off[t.nlev - 1];
  a.a = t.nlev == 0 ? leaves : NodeRef{nodes.items, nodes.counts, nodes.errs, nodes.sizes};
  a.b = a.a;
  a.o = root;
  a.a_mul = 2;
  a.a_add = base;
  a.b_mul = 2;
  a.b_add = base + 1;
  a.nblocks = 1;
  a.nright = t.c_final / 2;
  a.canon_single = 0;
  a.sort_out = 1;
  return combine_run(kb, k, a, scratch, s, d);
}

// ---- K3: Pruned(global, n, k) -- the root is in canonical order, so candidates are a prefix
template <typename KT>
__global__ void __launch_bounds__(256) prune_kernel(const KT* items, const uint32_t* counts,
                                                    const uint32_t* sizes, uint64_t thr,
                                                    KT* cand, uint32_t* n_cand) {
  __shared__ uint32_t red[8];
  const uint32_t size = sizes[0];
  uint32_t c = 0;
  for (uint32_t t = threadIdx.x; t < size; t += 256) {
    if ((uint64_t)counts[t] >= thr) {
      cand[t] = items[t];
      ++c;
    }
  }
  c = __reduce_add_sync(PSS_FULL, c);
  if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = c;
  __syncthreads();
  if (threadIdx.x == 0) {
    uint32_t t = 0;
    for (int i = 0; i < 8; ++i) t += red[i];
    *n_cand = t;
  }
}

cudaError_t prune_launch(int kb, uint32_t k, const void* items, const uint32_t* counts,
                         const uint32_t* sizes, uint64_t n, void* cand, uint32_t* n_cand,
                         cudaStream_t s) {
  const uint64_t thr = n / k + 1;  // floor(n/k) + 1
  if (kb == 4)
    prune_kernel<uint32_t><<<1, 256, 0, s>>>(static_cast<const uint32_t*>(items), counts, sizes,
                                              thr, static_cast<uint32_t*>(cand), n_cand);
  else
    prune_kernel<uint64_t><<<1, 256, 0, s>>>(static_cast<const uint64_t*>(items), counts, sizes,
                                              thr, static_cast<uint64_t*>(cand), n_cand);
  return cudaGetLastError();
}

}  // namespace pss
