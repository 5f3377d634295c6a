// accuracy.cu -- the paper's accuracy metrics:
// an exact k-majority set computed without Space Saving, and the report of precision, recall and
// average relative error of Algorithm 1's output against it.
//
// Exact k-majority (pss_exact_kmajority), "local heavy hitters": A is cut into sub-blocks of
// LHH_B items; if f(x) > n/k then f_r(x) > L_r/k in at least one sub-block r (otherwise
// f(x) = sum_r f_r(x) <= sum_r L_r/k = n/k). Pass 1 builds every sub-block's exact histogram in
// shared memory (a CTA-wide hash table, equal keys of a warp instruction aggregated with
// __match_any_sync) and inserts its locally heavy keys into a global hash set G. Pass 2 counts
// G's keys exactly, by the candidate count (decided on the device): up to K4_MAX_CAND, G is
// compacted into a candidate list and K4 (verify_kernel, the off-line counting scan) counts it;
// beyond (k >= 4096 makes every key of a sub-block locally heavy), the per-sub-block histograms are
// rebuilt and each local count is added to its key's entry of G. The candidates with count >=
// floor(n/k) + 1 are ranked by K5 (result_kernel).
// No step uses Space Saving, so the set is an independent truth for recall.
#include <algorithm>

#include "common.cuh"

namespace pss {

namespace {

constexpr uint32_t LHH_B = 4096;        // items per sub-block
constexpr uint32_t LHH_TS = 8192;       // shared hash-table entries (load <= 0.5)
constexpr uint32_t LHH_THREADS = 512;
constexpr uint32_t CLAIM = 0xffffffffu; // a shared entry being claimed (counts are <= LHH_B)
// K4 builds its candidate table serially: beyond this many candidates pass 2 is the histogram one
constexpr uint32_t K4_MAX_CAND = 32768;

__device__ __forceinline__ uint32_t mix_hash(uint32_t x) {
  x ^= x >> 16;
  x *= 0x7feb352du;
  x ^= x >> 15;
  x *= 0x846ca68bu;
  return x ^ (x >> 16);
}
__device__ __forceinline__ uint32_t mix_hash(uint64_t x) {
  return mix_hash((uint32_t)x ^ mix_hash((uint32_t)(x >> 32)));
}

template <typename KT>
struct GSet {  // global open-addressing set: state 0 empty, 1 being written, 2 ready
  KT* keys;
  uint32_t* state;
  unsigned long long* counts;  // pass 2 by histograms: exact counts
  uint32_t mask;
  uint32_t* overflow;
};

// a linear probe longer than this means the set is (nearly) full: the result is reported
// incomplete (overflow = 1) instead of scanning the whole table for every later key
constexpr uint32_t GSET_MAX_PROBE = 1024;

template <typename KT>
__device__ void gset_insert(const GSet<KT>& g, KT x) {
  if (__ldcg(g.overflow)) return;  // already incomplete
  uint32_t h = mix_hash(x) & g.mask;
  for (uint32_t probe = 0; probe <= min(g.mask, GSET_MAX_PROBE);) {
    const uint32_t s = ld_acquire(&g.state[h]);
    if (s == 0) {
      if (atomicCAS(&g.state[h], 0u, 1u) == 0u) {
        g.keys[h] = x;
        st_release(&g.state[h], 2u);
        return;
      }
      continue;  // lost the race: re-read the same entry
    }
    if (s == 1) continue;  // being written
    if (__ldcg(&g.keys[h]) == x) return;
    h = (h + 1) & g.mask;
    ++probe;
  }
  atomicExch(g.overflow, 1u);
}

// pass 2 by histograms: no writer is running, every entry is 0 or 2
template <typename KT>
__device__ __forceinline__ int64_t gset_find(const GSet<KT>& g, KT x) {
  uint32_t h = mix_hash(x) & g.mask;
  for (uint32_t probe = 0; probe <= min(g.mask, GSET_MAX_PROBE); ++probe) {
    if (g.state[h] == 0) return -1;
    if (g.keys[h] == x) return h;
    h = (h + 1) & g.mask;
  }
  return -1;
}

// PASS 1: locally heavy keys into G. PASS 2 (runs only if *run != 0): local counts into G.counts
template <typename KT, int PASS>
__global__ void __launch_bounds__(LHH_THREADS) lhh_kernel(const KT* __restrict__ A, uint64_t n,
                                                          uint32_t k, GSet<KT> g,
                                                          const uint32_t* run) {
  if (PASS == 2 && *run == 0) return;
  extern __shared__ __align__(16) unsigned char smem[];
  KT* keys = reinterpret_cast<KT*>(smem);
  uint32_t* cnt = reinterpret_cast<uint32_t*>(smem + LHH_TS * sizeof(KT));
  const uint64_t nsb = (n + LHH_B - 1) / LHH_B;
  const uint32_t lane = threadIdx.x & 31u;
  for (uint64_t sb = blockIdx.x; sb < nsb; sb += gridDim.x) {
    for (uint32_t e = threadIdx.x; e < LHH_TS; e += LHH_THREADS) cnt[e] = 0;
    __syncthreads();
    const uint64_t lo = sb * LHH_B;
    const uint32_t L = (uint32_t)(n - lo < LHH_B ? n - lo : LHH_B);
    for (uint32_t i = threadIdx.x; i < LHH_B; i += LHH_THREADS) {
      const bool valid = i < L;
      const uint32_t act = __ballot_sync(PSS_FULL, valid);
      if (!valid) continue;
      const KT x = A[lo + i];
      const uint32_t grp = __match_any_sync(act, x);
      if (lane != (uint32_t)(__ffs(grp) - 1)) continue;  // the group's leader adds its size
      const uint32_t mult = __popc(grp);
      uint32_t h = mix_hash(x) & (LHH_TS - 1);
      while (true) {
        const uint32_t c = *reinterpret_cast<volatile uint32_t*>(&cnt[h]);
        if (c == 0) {
          if (atomicCAS(&cnt[h], 0u, CLAIM) == 0u) {
            keys[h] = x;
            __threadfence_block();
            atomicExch(&cnt[h], mult);
            break;
          }
          continue;
        }
        if (c == CLAIM) continue;
        __threadfence_block();
        if (*reinterpret_cast<volatile KT*>(&keys[h]) == x) {
          atomicAdd(&cnt[h], mult);
          break;
        }
        h = (h + 1) & (LHH_TS - 1);
      }
    }
    __syncthreads();
    for (uint32_t e = threadIdx.x; e < LHH_TS; e += LHH_THREADS) {
      const uint32_t c = cnt[e];
      if (!c) continue;
      if (PASS == 1) {
        if ((uint64_t)c * k > L) gset_insert(g, keys[e]);  // f_r(x) > L_r / k
      } else {
        const int64_t j = gset_find(g, keys[e]);
        if (j >= 0) atomicAdd(&g.counts[j], (unsigned long long)c);
      }
    }
    __syncthreads();
  }
}

// the keys of G as a dense candidate list
template <typename KT>
__global__ void gset_compact_kernel(GSet<KT> g, KT* list, uint32_t* n_list) {
  for (uint32_t e = blockIdx.x * blockDim.x + threadIdx.x; e <= g.mask; e += gridDim.x * blockDim.x)
    if (g.state[e] == 2) list[atomicAdd(n_list, 1u)] = g.keys[e];
}

// which pass 2 runs: route[0] = the list length K4 counts (0: none), route[1] = 1 for histograms
__global__ void kmaj_route_kernel(const uint32_t* n_list, uint32_t* route) {
  const uint32_t nl = *n_list;
  route[0] = nl <= K4_MAX_CAND ? nl : 0u;
  route[1] = nl > K4_MAX_CAND ? 1u : 0u;
}

// histogram pass 2: the entries of G with count >= thr
template <typename KT>
__global__ void gset_collect_kernel(GSet<KT> g, const uint32_t* run, uint64_t thr, uint32_t cap,
                                    KT* cand, uint64_t* cexact, uint32_t* n_out) {
  if (*run == 0) return;
  for (uint32_t e = blockIdx.x * blockDim.x + threadIdx.x; e <= g.mask; e += gridDim.x * blockDim.x) {
    if (g.state[e] != 2 || g.counts[e] < thr) continue;
    const uint32_t p = atomicAdd(n_out, 1u);
    if (p < cap) {
      cand[p] = g.keys[e];
      cexact[p] = g.counts[e];
    }
  }
}

// the candidates with exact count >= thr (fewer than k: their counts sum to <= n)
template <typename KT>
__global__ void kmaj_filter_kernel(const KT* list, const uint64_t* exact, const uint32_t* n_list,
                                   uint64_t thr, uint32_t cap, KT* cand, uint64_t* cexact,
                                   uint32_t* n_out) {
  const uint32_t nl = *n_list;
  for (uint32_t j = blockIdx.x * blockDim.x + threadIdx.x; j < nl; j += gridDim.x * blockDim.x) {
    if (exact[j] < thr) continue;
    const uint32_t p = atomicAdd(n_out, 1u);
    if (p < cap) {
      cand[p] = list[j];
      cexact[p] = exact[j];
    }
  }
}

// precision, recall and ARE of the reported candidates: one CTA, fixed
// summation order (deterministic)
__global__ void __launch_bounds__(1024) accuracy_kernel(const uint32_t* fhat, uint32_t cap,
                                                        const uint32_t* d_n_cand,
                                                        const uint64_t* exact,
                                                        const uint32_t* d_n_true, uint64_t thr,
                                                        pss_accuracy_report* out) {
  __shared__ double s_all[32], s_true[32];
  __shared__ unsigned long long s_nt[32];
  const uint32_t nc = d_n_cand ? min(cap, *d_n_cand) : cap;
  double a = 0.0, t = 0.0;
  unsigned long long nt = 0;
  for (uint32_t j = threadIdx.x; j < nc; j += 1024) {
    const uint64_t f = exact[j];
    const double fh = (double)fhat[j];
    // a reported item was seen by some leaf, so f >= 1 (f = 0 would be a bug upstream: count 1)
    const double df = f ? fabs((double)f - fh) / (double)f : 1.0;
    a += df;
    if (f >= thr) {
      t += df;
      ++nt;
    }
  }
  for (int o = 16; o; o >>= 1) {
    a += __shfl_down_sync(PSS_FULL, a, o);
    t += __shfl_down_sync(PSS_FULL, t, o);
    nt += __shfl_down_sync(PSS_FULL, nt, o);
  }
  if ((threadIdx.x & 31) == 0) {
    s_all[threadIdx.x >> 5] = a;
    s_true[threadIdx.x >> 5] = t;
    s_nt[threadIdx.x >> 5] = nt;
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    double sa = 0.0, st = 0.0;
    unsigned long long snt = 0;
    for (int w = 0; w < 32; ++w) {
      sa += s_all[w];
      st += s_true[w];
      snt += s_nt[w];
    }
    const uint64_t ntrue = *d_n_true;
    pss_accuracy_report r;
    r.n_reported = nc;
    r.n_reported_true = snt;
    r.n_true = ntrue;
    r.precision = nc ? (double)snt / (double)nc : 1.0;
    r.recall = ntrue ? (double)snt / (double)ntrue : 1.0;
    r.are_reported = nc ? sa / (double)nc : 0.0;
    // a true k-majority item that was not reported has estimate 0: relative error 1
    r.are_true = ntrue ? (st + (double)(ntrue - snt)) / (double)ntrue : 0.0;
    *out = r;
  }
}

struct ExLayout {
  size_t keys, state, counts, nlist, ncand, overflow, route, list, lexact, cand, exact, vws, total;
  uint32_t cap;
};
ExLayout ex_layout(int kb, uint64_t n, uint32_t k, const DevInfo& d) {
  // G holds the locally heavy keys: at most n*k/LHH_B distinct ones (each has f > LHH_B/k);
  // capacity 2x that bound, between 2^12 and 2^24 entries (overflow is reported)
  const double bound = std::min<double>((double)n, (double)n * k / LHH_B);
  uint32_t cap = 1u << 12;
  while (cap < (1u << 24) && cap < 2.0 * bound) cap <<= 1;
  ExLayout L;
  L.cap = cap;
  Bump b;
  L.keys = b.take<unsigned char>((size_t)cap * kb);
  L.state = b.take<uint32_t>(cap);  // state .. route are cleared by one memset
  L.counts = b.take<unsigned long long>(cap);
  L.nlist = b.take<uint32_t>(1);
  L.ncand = b.take<uint32_t>(1);
  L.overflow = b.take<uint32_t>(1);
  L.route = b.take<uint32_t>(2);
  L.list = b.take<unsigned char>((size_t)cap * kb);
  L.lexact = b.take<uint64_t>(cap);
  L.cand = b.take<unsigned char>((size_t)k * kb);
  L.exact = b.take<uint64_t>(k);
  L.vws = b.take<unsigned char>(verify_ws(kb, std::min(cap, K4_MAX_CAND), d));
  L.total = b.bytes();
  return L;
}

template <typename KT>
cudaError_t exact_run(const KT* A, uint64_t n, uint32_t k, void* out_items, uint64_t* out_counts,
                      uint32_t* out_len, uint32_t* d_overflow, void* ws, cudaStream_t s,
                      const DevInfo& d) {
  unsigned char* w = static_cast<unsigned char*>(ws);
  const ExLayout L = ex_layout(sizeof(KT), n, k, d);
  GSet<KT> g{reinterpret_cast<KT*>(w + L.keys), reinterpret_cast<uint32_t*>(w + L.state),
             reinterpret_cast<unsigned long long*>(w + L.counts), L.cap - 1,
             d_overflow ? d_overflow : reinterpret_cast<uint32_t*>(w + L.overflow)};
  uint32_t* route = reinterpret_cast<uint32_t*>(w + L.route);
  uint32_t* nlist = reinterpret_cast<uint32_t*>(w + L.nlist);
  uint32_t* ncand = reinterpret_cast<uint32_t*>(w + L.ncand);
  KT* list = reinterpret_cast<KT*>(w + L.list);
  uint64_t* lexact = reinterpret_cast<uint64_t*>(w + L.lexact);
  // set states, list and candidate counts and the overflow flag start at zero
  cudaError_t e = cudaMemsetAsync(w + L.state, 0, L.list - L.state, s);
  if (e == cudaSuccess && d_overflow) e = cudaMemsetAsync(d_overflow, 0, sizeof(uint32_t), s);
  if (e != cudaSuccess) return e;
  const size_t smem = LHH_TS * (sizeof(KT) + sizeof(uint32_t));
  if (n) {
    auto k1 = lhh_kernel<KT, 1>;
    auto k2 = lhh_kernel<KT, 2>;
    allow_max_smem(k1, d);
    allow_max_smem(k2, d);
    int nb = 1;
    if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&nb, k1, LHH_THREADS, smem) != cudaSuccess ||
        nb < 1)
      nb = 1;
    const uint64_t nsb = (n + LHH_B - 1) / LHH_B;
    const int grid = (int)std::min<uint64_t>(nsb, (uint64_t)nb * d.sms);
    const int cgrid = std::max<int>(1, (int)std::min<uint32_t>(L.cap / 256, 4 * d.sms));
    k1<<<grid, LHH_THREADS, smem, s>>>(A, n, k, g, nullptr);
    gset_compact_kernel<KT><<<cgrid, 256, 0, s>>>(g, list, nlist);
    kmaj_route_kernel<<<1, 1, 0, s>>>(nlist, route);
    e = cudaGetLastError();
    // pass 2, one of two (the other's kernels return at once): K4, the off-line counting scan,
    // over the compacted list (route[0] candidates) ...
    const uint32_t kcap = std::min(L.cap, K4_MAX_CAND);
    if (e == cudaSuccess)
      e = verify_launch(A, n, sizeof(KT), list, kcap, route, lexact, w + L.vws, s, d);
    if (e != cudaSuccess) return e;
    kmaj_filter_kernel<KT><<<cgrid, 256, 0, s>>>(list, lexact, route, n / k + 1, k,
                                                 reinterpret_cast<KT*>(w + L.cand),
                                                 reinterpret_cast<uint64_t*>(w + L.exact), ncand);
    // ... or the histograms again, adding local counts to G (route[1])
    k2<<<grid, LHH_THREADS, smem, s>>>(A, n, k, g, route + 1);
    gset_collect_kernel<KT><<<cgrid, 256, 0, s>>>(g, route + 1, n / k + 1, k,
                                                  reinterpret_cast<KT*>(w + L.cand),
                                                  reinterpret_cast<uint64_t*>(w + L.exact), ncand);
    e = cudaGetLastError();
    if (e != cudaSuccess) return e;
  }
  return result_launch(sizeof(KT), k, w + L.cand, ncand, reinterpret_cast<uint64_t*>(w + L.exact),
                       n, k, out_items, out_counts, out_len, s);
}

}  // namespace

size_t exact_ws(int kb, uint64_t n, uint32_t k) { return ex_layout(kb, n, k, dev_info()).total; }

}  // namespace pss

using namespace pss;

extern "C" {

pss_status pss_exact_kmajority(const void* d_A, uint64_t n, pss_key_type kt, uint32_t k,
                               void* d_out_items, uint64_t* d_out_counts, uint32_t* d_out_len,
                               uint32_t* d_overflow, void* d_ws, size_t ws_bytes,
                               cudaStream_t stream) {
  const int kb = kt == PSS_KEY_U32 ? 4 : (kt == PSS_KEY_U64 ? 8 : 0);
  if (!kb || k < 2 || (n && !d_A) || !d_out_items || !d_out_counts || !d_out_len || !d_ws)
    return PSS_ERR_INVALID_ARG;
  if (n > PSS_MAX_N || k > PSS_MAX_K) return PSS_ERR_UNSUPPORTED;
  if (ws_bytes < exact_ws(kb, n, k)) return PSS_ERR_WORKSPACE_TOO_SMALL;
  const DevInfo d = dev_info();
  const cudaError_t e =
      kb == 4 ? exact_run(static_cast<const uint32_t*>(d_A), n, k, d_out_items, d_out_counts,
                          d_out_len, d_overflow, d_ws, stream, d)
              : exact_run(static_cast<const uint64_t*>(d_A), n, k, d_out_items, d_out_counts,
                          d_out_len, d_overflow, d_ws, stream, d);
  return e == cudaSuccess ? PSS_OK : PSS_ERR_CUDA;
}

pss_status pss_accuracy(const pss_summaries* root, uint64_t n, const uint32_t* d_n_cand,
                        const uint64_t* d_exact, const uint32_t* d_n_true,
                        pss_accuracy_report* d_report, cudaStream_t stream) {
  if (!root || !root->counts || root->count != 1 || root->k < 2 || !d_n_cand || !d_exact ||
      !d_n_true || !d_report)
    return PSS_ERR_INVALID_ARG;
  if (n > PSS_MAX_N) return PSS_ERR_UNSUPPORTED;
  accuracy_kernel<<<1, 1024, 0, stream>>>(root->counts, root->k, d_n_cand, d_exact, d_n_true,
                                          n / root->k + 1, d_report);
  return cudaGetLastError() == cudaSuccess ? PSS_OK : PSS_ERR_CUDA;
}

}  // extern "C"
