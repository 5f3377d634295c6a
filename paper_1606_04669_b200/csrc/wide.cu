// wide.cu -- summaries with 64-bit counts and errors ("wide") for the levels of the fixed tree
// above the leaves when the summarized stream may exceed 2^31 items: the top levels over several
// ranks' subtree roots (the paper's MPI reduction P:159) and the on-line stream's
// upper tree (R14, P:195 streams of 29 10^9 items).
//
// Reading R9 bounds f_hat <= N + N/k < 2^32 only for N <= 2^31 items; above the leaves a summary
// can cover more, so these COMBINEs (Algorithm 2, readings R3-R6) keep counts
// and errors in 64 bits. One CTA per COMBINE: both summaries are staged, S2's items indexed by an
// open-addressing table (Find/Remove of Alg. 2), unmatched counters get the other side's minimum
// (R4), and the union is sorted canonically (count descending, item ascending, R5) by a bitonic
// network over indices, the first k kept. These levels are few (log2 of the ranks, or of the
// stream's leaves) and their summaries small, so one simple kernel serves all of them.
#include <cstdlib>

#include "common.cuh"

namespace pss {

constexpr int W_NT = 512;
constexpr uint32_t W_EMPTY = 0xffffffffu;

struct WRef {
  const void* items;
  const uint64_t* counts;
  const uint64_t* errs;
  const uint32_t* sizes;
};
struct WOut {
  void* items;
  uint64_t* counts;
  uint64_t* errs;
  uint32_t* sizes;
};

struct WArgs {
  WRef a, b;
  WOut o;
  uint32_t k;
  uint32_t nblocks, nright;  // COMBINE i of a level: inputs a[i*a_mul+a_add], b[i*b_mul+b_add]
  uint32_t a_mul, a_add, b_mul, b_add;
  int canon_single;  // a single input (no b) is sorted canonically instead of copied
  unsigned char* gscratch;  // per-CTA scratch in global memory (else shared memory)
  size_t gstride;
  uint32_t NP, logH;        // sort length (power of two >= 2k), index table size 2^logH
};

struct WLayout {
  size_t key, cnt, err, dead, ht, idx, total;
};
__host__ __device__ inline WLayout w_layout(int kb, uint32_t NP, uint32_t H) {
  WLayout L;
  size_t o = 0;
  auto take = [&](size_t bytes) {
    const size_t r = o;
    o = (o + bytes + 15) & ~(size_t)15;
    return r;
  };
  L.key = take((size_t)NP * kb);
  L.cnt = take((size_t)NP * 8);
  L.err = take((size_t)NP * 8);
  L.dead = take(NP);
  L.ht = take((size_t)H * 4);
  L.idx = take((size_t)NP * 4);
  L.total = o;
  return L;
}

template <typename KT>
__global__ void __launch_bounds__(W_NT) wide_combine_kernel(const WArgs a) {
  extern __shared__ __align__(16) unsigned char smem[];
  __shared__ unsigned long long red[2 * (W_NT / 32)];
  __shared__ uint32_t nlive[W_NT / 32];
  const uint32_t tid = threadIdx.x, lane = tid & 31u, warp = tid >> 5;
  unsigned char* base = a.gscratch ? a.gscratch + (size_t)blockIdx.x * a.gstride : smem;
  const WLayout L = w_layout((int)sizeof(KT), a.NP, 1u << a.logH);
  KT* ukey = reinterpret_cast<KT*>(base + L.key);
  uint64_t* ucnt = reinterpret_cast<uint64_t*>(base + L.cnt);
  uint64_t* uerr = reinterpret_cast<uint64_t*>(base + L.err);
  uint8_t* dead = reinterpret_cast<uint8_t*>(base + L.dead);
  uint32_t* ht = reinterpret_cast<uint32_t*>(base + L.ht);
  uint32_t* idx = reinterpret_cast<uint32_t*>(base + L.idx);
  const uint32_t k = a.k, H = 1u << a.logH, hmask = H - 1u;

  for (uint32_t blk = blockIdx.x; blk < a.nblocks; blk += gridDim.x) {
    const uint32_t li = blk * a.a_mul + a.a_add;
    const bool has_r = blk < a.nright;
    const uint32_t ri = blk * a.b_mul + a.b_add;
    const uint32_t n1 = a.a.sizes[li];
    const uint32_t n2 = has_r ? a.b.sizes[ri] : 0u;
    const KT* i1 = reinterpret_cast<const KT*>(a.a.items) + (size_t)li * k;
    const uint64_t* c1 = a.a.counts + (size_t)li * k;
    const uint64_t* e1 = a.a.errs + (size_t)li * k;
    KT* oi = reinterpret_cast<KT*>(a.o.items) + (size_t)blk * k;
    uint64_t* oc = a.o.counts + (size_t)blk * k;
    uint64_t* oe = a.o.errs + (size_t)blk * k;
    if (!has_r && !a.canon_single) {  // odd last node carried up unchanged (R6)
      for (uint32_t t = tid; t < n1; t += W_NT) {
        oi[t] = i1[t];
        oc[t] = c1[t];
        oe[t] = e1[t];
      }
      if (tid == 0) a.o.sizes[blk] = n1;
      __syncthreads();
      continue;
    }
    const KT* i2 = has_r ? reinterpret_cast<const KT*>(a.b.items) + (size_t)ri * k : nullptr;
    const uint64_t* c2 = has_r ? a.b.counts + (size_t)ri * k : nullptr;
    const uint64_t* e2 = has_r ? a.b.errs + (size_t)ri * k : nullptr;
    // stage S1 -> u[0, n1), S2 -> u[n1, n1 + n2); minima (Alg. 2 l.2-3, R4)
    unsigned long long mn1 = ~0ull, mn2 = ~0ull;
    for (uint32_t t = tid; t < n1; t += W_NT) {
      ukey[t] = i1[t];
      ucnt[t] = c1[t];
      uerr[t] = e1[t];
      mn1 = min(mn1, (unsigned long long)c1[t]);
    }
    for (uint32_t t = tid; t < n2; t += W_NT) {
      ukey[n1 + t] = i2[t];
      ucnt[n1 + t] = c2[t];
      uerr[n1 + t] = e2[t];
      dead[t] = 0;
      mn2 = min(mn2, (unsigned long long)c2[t]);
    }
    for (uint32_t h = tid; h < H; h += W_NT) ht[h] = W_EMPTY;
#pragma unroll
    for (int o = 16; o; o >>= 1) {
      mn1 = min(mn1, __shfl_xor_sync(PSS_FULL, mn1, o));
      mn2 = min(mn2, __shfl_xor_sync(PSS_FULL, mn2, o));
    }
    if (lane == 0) {
      red[warp] = mn1;
      red[W_NT / 32 + warp] = mn2;
    }
    __syncthreads();
    unsigned long long m1r = ~0ull, m2r = ~0ull;
#pragma unroll
    for (int w = 0; w < W_NT / 32; ++w) {
      m1r = min(m1r, red[w]);
      m2r = min(m2r, red[W_NT / 32 + w]);
    }
    const uint64_t m1 = n1 == k ? m1r : 0u;  // R4: 0 unless all k counters are occupied
    const uint64_t m2 = n2 == k ? m2r : 0u;
    // index S2's items (Find of Alg. 2 l.5)
    for (uint32_t t = tid; t < n2; t += W_NT) {
      uint32_t h = hslot(ukey[n1 + t], a.logH);
      while (atomicCAS(&ht[h], W_EMPTY, t) != W_EMPTY) h = (h + 1u) & hmask;
    }
    __syncthreads();
    // S1's counters: matched -> f1 + f2 (Remove from S2); else f1 + m2 (Alg. 2 l.4-13)
    for (uint32_t t = tid; t < n1; t += W_NT) {
      const KT x = ukey[t];
      uint32_t h = hslot(x, a.logH);
      uint32_t j;
      while ((j = ht[h]) != W_EMPTY && ukey[n1 + j] != x) h = (h + 1u) & hmask;
      if (j != W_EMPTY) {
        ucnt[t] += ucnt[n1 + j];
        uerr[t] += uerr[n1 + j];
        dead[j] = 1;
      } else {
        ucnt[t] += m2;
        uerr[t] += m2;
      }
    }
    __syncthreads();
    // S2's remaining counters: f2 + m1 (Alg. 2 l.14-18)
    const uint32_t N = n1 + n2;
    uint32_t live = 0;
    for (uint32_t t = tid; t < n2; t += W_NT)
      if (!dead[t]) {
        ucnt[n1 + t] += m1;
        uerr[n1 + t] += m1;
      }
    __syncthreads();
    // Prune(k) (Alg. 2 l.19): canonical order (count desc, item asc, R5), the first k kept
    uint32_t NPs = 2;
    while (NPs < N) NPs <<= 1;
    for (uint32_t i = tid; i < NPs; i += W_NT) {
      const bool valid = i < N && !(i >= n1 && dead[i - n1]);
      idx[i] = valid ? i : W_EMPTY;
      live += valid;
    }
    live = __reduce_add_sync(PSS_FULL, live);
    if (lane == 0) nlive[warp] = live;
    __syncthreads();
    auto before = [&](uint32_t x, uint32_t y) {  // x precedes y; unused entries go last
      if (y == W_EMPTY) return x != W_EMPTY;
      if (x == W_EMPTY) return false;
      return ucnt[x] > ucnt[y] || (ucnt[x] == ucnt[y] && ukey[x] < ukey[y]);
    };
    for (uint32_t size = 2; size <= NPs; size <<= 1) {
      for (uint32_t stride = size >> 1; stride; stride >>= 1) {
        for (uint32_t t = tid; t < NPs / 2; t += W_NT) {
          const uint32_t lo = 2 * stride * (t / stride) + (t % stride), hi = lo + stride;
          const bool up = (lo & size) == 0;
          const uint32_t x = idx[lo], y = idx[hi];
          if (before(y, x) == up) {
            idx[lo] = y;
            idx[hi] = x;
          }
        }
        __syncthreads();
      }
    }
    uint32_t Lv = 0;
#pragma unroll
    for (int w = 0; w < W_NT / 32; ++w) Lv += nlive[w];
    const uint32_t outn = min(Lv, k);
    for (uint32_t i = tid; i < outn; i += W_NT) {
      const uint32_t u = idx[i];
      oi[i] = ukey[u];
      oc[i] = ucnt[u];
      oe[i] = uerr[u];
    }
    if (tid == 0) a.o.sizes[blk] = outn;
    __syncthreads();
  }
}

template <typename KT>
__global__ void widen_kernel(const KT* items, const uint32_t* counts, const uint32_t* errs,
                             const uint32_t* sizes, uint32_t k, uint32_t count, KT* wi,
                             uint64_t* wc, uint64_t* we, uint32_t* ws) {
  const uint64_t total = (uint64_t)count * k;
  for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < total;
       i += (uint64_t)gridDim.x * blockDim.x) {
    const uint32_t s = (uint32_t)(i / k);
    if (i - (uint64_t)s * k < sizes[s]) {
      wi[i] = items[i];
      wc[i] = counts[i];
      we[i] = errs[i];
    }
    if (i - (uint64_t)s * k == 0) ws[s] = sizes[s];
  }
}

template <typename KT>
__global__ void narrow_kernel(const KT* wi, const uint64_t* wc, const uint64_t* we,
                              const uint32_t* wsz, uint32_t k, uint32_t count, KT* items,
                              uint32_t* counts, uint32_t* errs, uint32_t* sizes) {
  const uint64_t total = (uint64_t)count * k;
  for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < total;
       i += (uint64_t)gridDim.x * blockDim.x) {
    const uint32_t s = (uint32_t)(i / k);
    if (i - (uint64_t)s * k < wsz[s]) {
      items[i] = wi[i];
      counts[i] = (uint32_t)wc[i];  // the caller guarantees the counts fit (N + N/k < 2^32)
      errs[i] = (uint32_t)we[i];
    }
    if (i - (uint64_t)s * k == 0) sizes[s] = wsz[s];
  }
}

template <typename KT>
__global__ void __launch_bounds__(256) wide_prune_kernel(const KT* items, const uint64_t* counts,
                                                         const uint32_t* sizes, uint64_t thr,
                                                         KT* cand, uint32_t* n_cand) {
  __shared__ uint32_t red[8];
  const uint32_t size = sizes[0];
  uint32_t c = 0;
  for (uint32_t t = threadIdx.x; t < size; t += 256) {
    if (counts[t] >= thr) {  // canonical order: the candidates are a prefix
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

// ------------------------------------------------------------------------------ host side
struct WPlan {
  uint32_t NP, logH;
  WLayout L;
  bool g;
  size_t smem;
  int grid_cap;
};
static WPlan w_plan(int kb, uint32_t k, const DevInfo& d) {
  WPlan p;
  p.NP = 2;
  while (p.NP < 2 * k) p.NP <<= 1;
  p.logH = ceil_log2(2ull * k);
  if (p.logH < 5) p.logH = 5;
  p.L = w_layout(kb, p.NP, 1u << p.logH);
  p.g = p.L.total > (size_t)d.smem_optin - 4096;
  p.smem = p.g ? 0 : p.L.total;
  p.grid_cap = p.g ? 2 * d.sms : 1 << 30;
  return p;
}

size_t wide_combine_ws(int kb, uint32_t k, const DevInfo& d) {
  const WPlan p = w_plan(kb, k, d);
  return p.g ? p.L.total * (size_t)p.grid_cap : 0;
}

static cudaError_t wide_run(int kb, WArgs a, void* scratch, cudaStream_t s, const DevInfo& d) {
  const WPlan p = w_plan(kb, a.k, d);
  a.NP = p.NP;
  a.logH = p.logH;
  a.gscratch = p.g ? static_cast<unsigned char*>(scratch) : nullptr;
  a.gstride = p.L.total;
  if (a.nblocks == 0) return cudaSuccess;
  const int grid = (int)std::min<uint32_t>(a.nblocks, (uint32_t)p.grid_cap);
  if (kb == 4) {
    if (!p.g) allow_max_smem(wide_combine_kernel<uint32_t>, d);
    wide_combine_kernel<uint32_t><<<grid, W_NT, p.smem, s>>>(a);
  } else {
    if (!p.g) allow_max_smem(wide_combine_kernel<uint64_t>, d);
    wide_combine_kernel<uint64_t><<<grid, W_NT, p.smem, s>>>(a);
  }
  return cudaGetLastError();
}

cudaError_t wide_combine_launch(int kb, uint32_t k, uint32_t count, const void* ai,
                                const uint64_t* ac, const uint64_t* ae, const uint32_t* as,
                                const void* bi, const uint64_t* bc, const uint64_t* be,
                                const uint32_t* bs, void* oi, uint64_t* oc, uint64_t* oe,
                                uint32_t* os, void* scratch, cudaStream_t s, const DevInfo& d) {
  WArgs a{};
  a.a = WRef{ai, ac, ae, as};
  a.b = WRef{bi, bc, be, bs};
  a.o = WOut{oi, oc, oe, os};
  a.k = k;
  a.nblocks = count;
  a.nright = count;
  a.a_mul = a.b_mul = 1;
  a.canon_single = 1;
  return wide_run(kb, a, scratch, s, d);
}

// the fixed tree (R6) over `count` wide summaries: level buffers ping-pong in the workspace
struct WTreeWs {
  size_t lv[2][4], scratch, total;
};
static WTreeWs wtree_ws(int kb, uint32_t k, uint32_t count, const DevInfo& d) {
  WTreeWs w;
  Bump b;
  const uint32_t half = (count + 1) / 2;
  for (int i = 0; i < 2; ++i) {
    w.lv[i][0] = b.take<unsigned char>((size_t)half * k * kb);
    w.lv[i][1] = b.take<uint64_t>((size_t)half * k);
    w.lv[i][2] = b.take<uint64_t>((size_t)half * k);
    w.lv[i][3] = b.take<uint32_t>(half);
  }
  w.scratch = b.take<unsigned char>(wide_combine_ws(kb, k, d));
  w.total = b.bytes();
  return w;
}
size_t wide_merge_ws(int kb, uint32_t k, uint32_t count, const DevInfo& d) {
  return wtree_ws(kb, k, count, d).total;
}

cudaError_t wide_merge_launch(int kb, uint32_t k, uint32_t count, const void* items,
                              const uint64_t* counts, const uint64_t* errs, const uint32_t* sizes,
                              void* ri, uint64_t* rc, uint64_t* re, uint32_t* rs, void* ws,
                              cudaStream_t s, const DevInfo& d) {
  unsigned char* w = static_cast<unsigned char*>(ws);
  const WTreeWs L = wtree_ws(kb, k, count, d);
  WRef cur{items, counts, errs, sizes};
  uint32_t c = count;
  int pp = 0;
  while (true) {
    const uint32_t nxt = (c + 1) / 2;
    WArgs a{};
    a.a = cur;
    a.b = cur;
    a.k = k;
    a.a_mul = 2;
    a.b_mul = 2;
    a.b_add = 1;
    a.nblocks = nxt;
    a.nright = c / 2;
    a.canon_single = c == 1;  // a single summary: the root is its canonical order
    if (nxt == 1) {
      a.o = WOut{ri, rc, re, rs};
    } else {
      a.o = WOut{w + L.lv[pp][0], reinterpret_cast<uint64_t*>(w + L.lv[pp][1]),
                 reinterpret_cast<uint64_t*>(w + L.lv[pp][2]),
                 reinterpret_cast<uint32_t*>(w + L.lv[pp][3])};
    }
    const cudaError_t e = wide_run(kb, a, w + L.scratch, s, d);
    if (e != cudaSuccess || nxt == 1) return e;
    cur = WRef{a.o.items, a.o.counts, a.o.errs, a.o.sizes};
    c = nxt;
    pp ^= 1;
  }
}

cudaError_t widen_launch(int kb, uint32_t k, uint32_t count, const void* items,
                         const uint32_t* counts, const uint32_t* errs, const uint32_t* sizes,
                         void* wi, uint64_t* wc, uint64_t* we, uint32_t* wsz, cudaStream_t s) {
  const uint64_t total = (uint64_t)count * k;
  const int grid = (int)std::min<uint64_t>((total + 255) / 256, 4096);
  if (kb == 4)
    widen_kernel<uint32_t><<<std::max(grid, 1), 256, 0, s>>>(
        static_cast<const uint32_t*>(items), counts, errs, sizes, k, count,
        static_cast<uint32_t*>(wi), wc, we, wsz);
  else
    widen_kernel<uint64_t><<<std::max(grid, 1), 256, 0, s>>>(
        static_cast<const uint64_t*>(items), counts, errs, sizes, k, count,
        static_cast<uint64_t*>(wi), wc, we, wsz);
  return cudaGetLastError();
}

cudaError_t narrow_launch(int kb, uint32_t k, uint32_t count, const void* wi, const uint64_t* wc,
                          const uint64_t* we, const uint32_t* wsz, void* items, uint32_t* counts,
                          uint32_t* errs, uint32_t* sizes, cudaStream_t s) {
  const uint64_t total = (uint64_t)count * k;
  const int grid = std::max(1, (int)std::min<uint64_t>((total + 255) / 256, 4096));
  if (kb == 4)
    narrow_kernel<uint32_t><<<grid, 256, 0, s>>>(static_cast<const uint32_t*>(wi), wc, we, wsz, k,
                                                  count, static_cast<uint32_t*>(items), counts,
                                                  errs, sizes);
  else
    narrow_kernel<uint64_t><<<grid, 256, 0, s>>>(static_cast<const uint64_t*>(wi), wc, we, wsz, k,
                                                  count, static_cast<uint64_t*>(items), counts,
                                                  errs, sizes);
  return cudaGetLastError();
}

cudaError_t wide_prune_launch(int kb, const void* items, const uint64_t* counts,
                              const uint32_t* sizes, uint64_t n, uint32_t k, void* cand,
                              uint32_t* n_cand, cudaStream_t s) {
  const uint64_t thr = n / k + 1;  // floor(n/k) + 1
  if (kb == 4)
    wide_prune_kernel<uint32_t><<<1, 256, 0, s>>>(static_cast<const uint32_t*>(items), counts,
                                                   sizes, thr, static_cast<uint32_t*>(cand),
                                                   n_cand);
  else
    wide_prune_kernel<uint64_t><<<1, 256, 0, s>>>(static_cast<const uint64_t*>(items), counts,
                                                   sizes, thr, static_cast<uint64_t*>(cand),
                                                   n_cand);
  return cudaGetLastError();
}

}  // namespace pss
