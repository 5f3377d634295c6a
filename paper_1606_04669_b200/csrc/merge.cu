// merge.cu -- K2/K3: COMBINE (Algorithm 2) on a fixed balanced binary merge
// tree (ParallelReduction, Algorithm 1 line 7; reading R6), and Pruned (Algorithm 1
// lines 8-9).
//
// One CTA per COMBINE. Both summaries are staged in shared memory; S2's items are indexed by a
// small hash table so each S1 counter finds its match in O(1) (Find/Remove of Alg. 2 l.5-7);
// unmatched counters get the other summary's minimum (R4: 0 for an unfull summary); Prune(k)
// orders the <= 2k counters by (count desc, item asc) with a shared-memory bitonic network and
// keeps the first k (R5). Outputs are in canonical order.
#include "common.cuh"

namespace pss {

constexpr int MT = 512;  // threads per merge CTA

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
  unsigned char* gscratch;              // per-CTA scratch when it does not fit shared memory
  size_t gstride;
  size_t o_ucnt, o_uerr, o_dead, o_ht, o_shi, o_slo, o_sidx;
  uint32_t logH2, NPmax;
};

struct MLayout {
  size_t ukey, ucnt, uerr, dead, ht, shi, slo, sidx, total;
  uint32_t logH2, NPmax;
};

static MLayout m_layout(uint32_t k, int kb) {
  MLayout L;
  const size_t U = 2 * (size_t)k;
  L.NPmax = 1u << ceil_log2(U);
  L.logH2 = ceil_log2(2ull * k);
  Bump b;
  L.ukey = b.take<unsigned char>(U * kb);
  L.ucnt = b.take<uint32_t>(U);
  L.uerr = b.take<uint32_t>(U);
  L.dead = b.take<uint8_t>(k);
  L.ht = b.take<uint32_t>((size_t)1 << L.logH2);
  L.shi = b.take<uint32_t>(L.NPmax);
  L.slo = b.take<unsigned char>((size_t)L.NPmax * kb);
  L.sidx = b.take<uint32_t>(L.NPmax);
  L.total = b.bytes();
  return L;
}

__device__ __forceinline__ uint32_t block_min(uint32_t v, uint32_t* red) {
  v = __reduce_min_sync(PSS_FULL, v);
  const int w = threadIdx.x >> 5, nw = blockDim.x >> 5;
  __syncthreads();
  if ((threadIdx.x & 31) == 0) red[w] = v;
  __syncthreads();
  uint32_t r = 0xffffffffu;
  for (int i = 0; i < nw; ++i) r = min(r, red[i]);
  __syncthreads();
  return r;
}

template <typename KT, bool G>
__global__ void __launch_bounds__(MT) combine_kernel(const CombArgs a) {
  extern __shared__ __align__(128) unsigned char smem[];
  __shared__ uint32_t red[MT / 32];
  const uint32_t k = a.k;
  const int tid = threadIdx.x;
  unsigned char* base = G ? a.gscratch + (size_t)blockIdx.x * a.gstride : smem;
  KT* ukey = reinterpret_cast<KT*>(base);
  uint32_t* ucnt = reinterpret_cast<uint32_t*>(base + a.o_ucnt);
  uint32_t* uerr = reinterpret_cast<uint32_t*>(base + a.o_uerr);
  uint8_t* dead = reinterpret_cast<uint8_t*>(base + a.o_dead);
  uint32_t* ht = reinterpret_cast<uint32_t*>(base + a.o_ht);
  uint32_t* shi = reinterpret_cast<uint32_t*>(base + a.o_shi);
  KT* slo = reinterpret_cast<KT*>(base + a.o_slo);
  uint32_t* sidx = reinterpret_cast<uint32_t*>(base + a.o_sidx);
  const uint32_t H2 = 1u << a.logH2, hmask = H2 - 1u;

  for (uint32_t blk = blockIdx.x; blk < a.nblocks; blk += gridDim.x) {
    const uint32_t li = blk * a.a_mul + a.a_add;
    const bool has_r = blk < a.nright;
    const uint32_t ri = blk * a.b_mul + a.b_add;
    const uint32_t n1 = a.a.sizes[li];
    const uint32_t n2 = has_r ? a.b.sizes[ri] : 0u;
    const KT* i1 = reinterpret_cast<const KT*>(a.a.items) + (size_t)li * k;
    const uint32_t* c1 = a.a.counts + (size_t)li * k;
    const uint32_t* e1 = a.a.errs + (size_t)li * k;
    KT* oi = reinterpret_cast<KT*>(a.o.items) + (size_t)blk * k;
    uint32_t* oc = a.o.counts + (size_t)blk * k;
    uint32_t* oe = a.o.errs + (size_t)blk * k;

    if (!has_r && !a.canon_single) {  // odd last node carried up unchanged (R6)
      for (uint32_t t = tid; t < n1; t += MT) {
        oi[t] = i1[t];
        oc[t] = c1[t];
        oe[t] = e1[t];
      }
      if (tid == 0) a.o.sizes[blk] = n1;
      continue;
    }
    const KT* i2 = has_r ? reinterpret_cast<const KT*>(a.b.items) + (size_t)ri * k : nullptr;
    const uint32_t* c2 = has_r ? a.b.counts + (size_t)ri * k : nullptr;
    const uint32_t* e2 = has_r ? a.b.errs + (size_t)ri * k : nullptr;

    // stage S1 -> u[0, n1), S2 -> u[n1, n1 + n2); minima (Alg. 2 l.2-3, R4)
    uint32_t mn1 = 0xffffffffu, mn2 = 0xffffffffu;
    for (uint32_t t = tid; t < n1; t += MT) {
      ukey[t] = i1[t];
      ucnt[t] = c1[t];
      uerr[t] = e1[t];
      mn1 = min(mn1, c1[t]);
    }
    for (uint32_t t = tid; t < n2; t += MT) {
      ukey[n1 + t] = i2[t];
      ucnt[n1 + t] = c2[t];
      uerr[n1 + t] = e2[t];
      dead[t] = 0;
      mn2 = min(mn2, c2[t]);
    }
    for (uint32_t h = tid; h < H2; h += MT) ht[h] = 0xffffffffu;
    const uint32_t m1r = block_min(mn1, red);
    const uint32_t m2r = block_min(mn2, red);
    const uint32_t m1 = n1 == k ? m1r : 0u;
    const uint32_t m2 = n2 == k ? m2r : 0u;
    // index S2's items (Find of Alg. 2 l.5)
    for (uint32_t t = tid; t < n2; t += MT) {
      uint32_t h = hslot(ukey[n1 + t], a.logH2);
      while (atomicCAS(&ht[h], 0xffffffffu, t) != 0xffffffffu) h = (h + 1u) & hmask;
    }
    __syncthreads();
    // counters of S1: matched -> f1 + f2 and Remove from S2; else f1 + m2 (Alg. 2 l.4-13)
    for (uint32_t t = tid; t < n1; t += MT) {
      const KT x = ukey[t];
      uint32_t h = hslot(x, a.logH2);
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
    // remaining counters of S2: f2 + m1 (Alg. 2 l.14-18)
    for (uint32_t t = tid; t < n2; t += MT)
      if (!dead[t]) {
        ucnt[n1 + t] += m1;
        uerr[n1 + t] += m1;
      }
    __syncthreads();
    // Prune(k) (Alg. 2 l.19): order by (count desc, item asc), keep the first k (R5)
    const uint32_t N = n1 + n2;
    const uint32_t NP = N <= 1 ? 1u : 1u << ceil_log2(N);
    uint32_t live = 0;
    for (uint32_t t = tid; t < NP; t += MT) {
      const bool valid = t < N && !(t >= n1 && dead[t - n1]);
      shi[t] = valid ? ~ucnt[t] : 0xffffffffu;  // valid counts are >= 1, so ~count < all-ones
      slo[t] = valid ? ukey[t] : (KT)0;
      sidx[t] = valid ? t : 0xffffffffu;
      live += valid;
    }
    live = __reduce_add_sync(PSS_FULL, live);
    __syncthreads();
    if ((tid & 31) == 0) red[tid >> 5] = live;
    __syncthreads();
    uint32_t L = 0;
    for (int i = 0; i < MT / 32; ++i) L += red[i];
    __syncthreads();
    for (uint32_t size = 2; size <= NP; size <<= 1) {
      for (uint32_t stride = size >> 1; stride > 0; stride >>= 1) {
        for (uint32_t i = tid; i < NP / 2; i += MT) {
          const uint32_t p = 2 * i - (i & (stride - 1));
          const uint32_t q = p + stride;
          const bool up = (p & size) == 0;
          const uint32_t hp = shi[p], hq = shi[q];
          const KT lp = slo[p], lq = slo[q];
          const bool gt = hp > hq || (hp == hq && (lp > lq || (lp == lq && sidx[p] > sidx[q])));
          if (gt == up) {
            shi[p] = hq;
            shi[q] = hp;
            slo[p] = lq;
            slo[q] = lp;
            const uint32_t t = sidx[p];
            sidx[p] = sidx[q];
            sidx[q] = t;
          }
        }
        __syncthreads();
      }
    }
    const uint32_t outn = min(L, k);
    for (uint32_t t = tid; t < outn; t += MT) {
      const uint32_t j = sidx[t];
      oi[t] = ukey[j];
      oc[t] = ucnt[j];
      oe[t] = uerr[j];
    }
    if (tid == 0) a.o.sizes[blk] = outn;
    __syncthreads();
  }
}

// ------------------------------------------------------------------------------ host side
struct MPlan {
  bool g;
  MLayout L;
  size_t smem;
  int grid_cap;
};

static MPlan m_plan(int kb, uint32_t k, const DevInfo& d) {
  MPlan p;
  p.L = m_layout(k, kb);
  p.g = p.L.total > (size_t)d.smem_optin - 1024;
  p.smem = p.g ? 0 : p.L.total;
  p.grid_cap = p.g ? 2 * d.sms : 1 << 30;
  return p;
}

static cudaError_t combine_run(int kb, uint32_t k, CombArgs a, void* ws, cudaStream_t s,
                               const DevInfo& d) {
  MPlan p = m_plan(kb, k, d);
  a.k = k;
  a.gscratch = p.g ? static_cast<unsigned char*>(ws) : nullptr;
  a.gstride = p.L.total;
  a.o_ucnt = p.L.ucnt;
  a.o_uerr = p.L.uerr;
  a.o_dead = p.L.dead;
  a.o_ht = p.L.ht;
  a.o_shi = p.L.shi;
  a.o_slo = p.L.slo;
  a.o_sidx = p.L.sidx;
  a.logH2 = p.L.logH2;
  a.NPmax = p.L.NPmax;
  if (a.nblocks == 0) return cudaSuccess;
  const int grid = (int)std::min<uint32_t>(a.nblocks, (uint32_t)p.grid_cap);
  if (kb == 4) {
    if (p.g) {
      combine_kernel<uint32_t, true><<<grid, MT, 0, s>>>(a);
    } else {
      cudaFuncSetAttribute(combine_kernel<uint32_t, false>,
                           cudaFuncAttributeMaxDynamicSharedMemorySize, (int)p.smem);
      combine_kernel<uint32_t, false><<<grid, MT, p.smem, s>>>(a);
    }
  } else {
    if (p.g) {
      combine_kernel<uint64_t, true><<<grid, MT, 0, s>>>(a);
    } else {
      cudaFuncSetAttribute(combine_kernel<uint64_t, false>,
                           cudaFuncAttributeMaxDynamicSharedMemorySize, (int)p.smem);
      combine_kernel<uint64_t, false><<<grid, MT, p.smem, s>>>(a);
    }
  }
  return cudaGetLastError();
}

static size_t scratch_bytes(int kb, uint32_t k, const DevInfo& d) {
  MPlan p = m_plan(kb, k, d);
  return p.g ? p.L.total * (size_t)p.grid_cap : 0;
}

size_t combine_ws(int kb, uint32_t k, uint32_t, const DevInfo& d) {
  return align_up(scratch_bytes(kb, k, d), 256) + 256;
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
  return combine_run(kb, k, a, ws, s, d);
}

// level buffers: A holds ceil(P/2) nodes, B ceil(P/4) nodes (levels alternate A, B, A, ...)
size_t merge_ws(int kb, uint32_t k, uint32_t P, const DevInfo& d) {
  Bump b;
  const size_t nA = (P + 1) / 2, nB = (P + 3) / 4;
  b.take<unsigned char>(nA * k * kb);
  b.take<uint32_t>(nA * k);
  b.take<uint32_t>(nA * k);
  b.take<uint32_t>(nA);
  b.take<unsigned char>(nB * k * kb);
  b.take<uint32_t>(nB * k);
  b.take<uint32_t>(nB * k);
  b.take<uint32_t>(nB);
  b.take<unsigned char>(scratch_bytes(kb, k, d));
  return b.bytes();
}

cudaError_t merge_tree_launch(int kb, uint32_t k, uint32_t P, const void* items,
                              const uint32_t* counts, const uint32_t* errs, const uint32_t* sizes,
                              void* r_items, uint32_t* r_counts, uint32_t* r_errs,
                              uint32_t* r_sizes, void* ws, cudaStream_t s, const DevInfo& d) {
  unsigned char* w = static_cast<unsigned char*>(ws);
  Bump b;
  const size_t nA = (P + 1) / 2, nB = (P + 3) / 4;
  NodeOut bufA, bufB;
  bufA.items = w + b.take<unsigned char>(nA * k * kb);
  bufA.counts = reinterpret_cast<uint32_t*>(w + b.take<uint32_t>(nA * k));
  bufA.errs = reinterpret_cast<uint32_t*>(w + b.take<uint32_t>(nA * k));
  bufA.sizes = reinterpret_cast<uint32_t*>(w + b.take<uint32_t>(nA));
  bufB.items = w + b.take<unsigned char>(nB * k * kb);
  bufB.counts = reinterpret_cast<uint32_t*>(w + b.take<uint32_t>(nB * k));
  bufB.errs = reinterpret_cast<uint32_t*>(w + b.take<uint32_t>(nB * k));
  bufB.sizes = reinterpret_cast<uint32_t*>(w + b.take<uint32_t>(nB));
  void* scratch = w + b.take<unsigned char>(scratch_bytes(kb, k, d));

  NodeRef cur{items, counts, errs, sizes};
  NodeOut root{r_items, r_counts, r_errs, r_sizes};
  if (P == 1) {  // root = the only leaf, in canonical order = COMBINE(S, empty)
    CombArgs a{};
    a.a = cur;
    a.b = cur;
    a.o = root;
    a.a_mul = 1;
    a.b_mul = 1;
    a.nblocks = 1;
    a.nright = 0;
    a.canon_single = 1;
    return combine_run(kb, k, a, scratch, s, d);
  }
  uint32_t c = P;
  int level = 0;
  while (c > 1) {
    const uint32_t cout = (c + 1) / 2;
    NodeOut out = cout == 1 ? root : (level % 2 == 0 ? bufA : bufB);
    CombArgs a{};
    a.a = cur;
    a.b = cur;
    a.o = out;
    a.a_mul = 2;
    a.a_add = 0;
    a.b_mul = 2;
    a.b_add = 1;
    a.nblocks = cout;
    a.nright = c / 2;
    a.canon_single = 0;
    cudaError_t e = combine_run(kb, k, a, scratch, s, d);
    if (e != cudaSuccess) return e;
    cur = NodeRef{out.items, out.counts, out.errs, out.sizes};
    c = cout;
    ++level;
  }
  return cudaSuccess;
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
