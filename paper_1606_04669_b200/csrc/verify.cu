// verify.cu -- K4/K5: the off-line verification scan ("a parallel scan of the input
// can be used to determine the actual frequent items") and the final k-majority report
// (PAPER.md:47, :80).
//
// K4 streams A once with 128-bit read-only loads. Every CTA indexes the candidate list in a
// shared-memory hash table (key -> candidate index, linear probing, load <= 1/2) and counts hits
// with shared-memory atomics; per-CTA counts are flushed into 64-bit global accumulators at the
// end. Candidate lists too large for shared memory use one global table built by the setup
// kernel. K5 keeps the candidates whose exact count reaches floor(n/k) + 1 and ranks them by
// (count desc, item asc).
#include "common.cuh"

namespace pss {

constexpr uint32_t VT_LOG_MAX = 11;  // shared-memory table: up to 2048 entries, n_cand <= 1024
constexpr int VTHREADS = 512;

struct VLayout {
  size_t acc, gkeys, gidx, total;
  uint32_t logT;
};

static VLayout v_layout(int kb, uint32_t cap) {
  VLayout L;
  L.logT = ceil_log2(2ull * (cap ? cap : 1));
  Bump b;
  L.acc = b.take<unsigned long long>(cap ? cap : 1);
  L.gkeys = b.take<unsigned char>(((size_t)1 << L.logT) * kb);
  L.gidx = b.take<uint32_t>((size_t)1 << L.logT);
  L.total = b.bytes();
  return L;
}

__device__ __forceinline__ uint32_t eff_count(uint32_t cap, const uint32_t* d_n) {
  return d_n ? min(cap, *d_n) : cap;
}

// insert candidate j into a table (duplicates may be inserted twice; lookups always see the
// first copy on the probe path, so counting stays consistent)
template <typename KT>
__device__ __forceinline__ void vt_insert(KT* tk, uint32_t* ti, uint32_t logT, KT x, uint32_t j) {
  const uint32_t mask = (1u << logT) - 1u;
  uint32_t h = hslot(x, logT);
  while (atomicCAS(&ti[h], 0xffffffffu, j) != 0xffffffffu) h = (h + 1u) & mask;
  tk[h] = x;
}

template <typename KT>
__device__ __forceinline__ int32_t vt_find(const KT* tk, const uint32_t* ti, uint32_t logT, KT x) {
  const uint32_t mask = (1u << logT) - 1u;
  uint32_t h = hslot(x, logT);
  while (true) {
    const uint32_t j = ti[h];
    if (j == 0xffffffffu) return -1;
    if (tk[h] == x) return (int32_t)h;
    h = (h + 1u) & mask;
  }
}

template <typename KT>
__global__ void verify_setup_kernel(const KT* cand, uint32_t cap, const uint32_t* d_n,
                                    unsigned long long* acc, KT* gk, uint32_t* gi,
                                    uint32_t logTcap) {
  const uint32_t nc = eff_count(cap, d_n);
  for (uint32_t j = threadIdx.x; j < nc; j += blockDim.x) acc[j] = 0;
  const uint32_t logT = ceil_log2(2ull * (nc ? nc : 1));
  if (logT <= VT_LOG_MAX) return;  // shared-memory tables are built per CTA
  const uint32_t T = 1u << logT;
  for (uint32_t h = threadIdx.x; h < T; h += blockDim.x) gi[h] = 0xffffffffu;
  __syncthreads();
  for (uint32_t j = threadIdx.x; j < nc; j += blockDim.x) vt_insert(gk, gi, logT, cand[j], j);
  (void)logTcap;
}

template <typename KT>
__device__ __forceinline__ void count_item(KT x, const KT* tk, const uint32_t* ti, uint32_t logT,
                                           uint32_t* scnt, unsigned long long* acc, bool gl) {
  const int32_t h = vt_find(tk, ti, logT, x);
  if (h >= 0) {
    if (gl)
      atomicAdd(&acc[ti[h]], 1ull);
    else
      atomicAdd(&scnt[h], 1u);
  }
}

template <typename KT>
__global__ void __launch_bounds__(VTHREADS) verify_kernel(const KT* __restrict__ A, uint64_t n,
                                                          const KT* cand, uint32_t cap,
                                                          const uint32_t* d_n,
                                                          unsigned long long* acc, const KT* gk,
                                                          const uint32_t* gi) {
  __shared__ KT tk_s[1u << VT_LOG_MAX];
  __shared__ uint32_t ti_s[1u << VT_LOG_MAX];
  __shared__ uint32_t scnt[1u << VT_LOG_MAX];
  const uint32_t nc = eff_count(cap, d_n);
  if (nc == 0) return;
  const uint32_t logT = ceil_log2(2ull * nc);
  const bool gl = logT > VT_LOG_MAX;
  const KT* tk = gl ? gk : tk_s;
  const uint32_t* ti = gl ? gi : ti_s;
  if (!gl) {
    const uint32_t T = 1u << logT;
    for (uint32_t h = threadIdx.x; h < T; h += VTHREADS) {
      ti_s[h] = 0xffffffffu;
      scnt[h] = 0;
    }
    __syncthreads();
    for (uint32_t j = threadIdx.x; j < nc; j += VTHREADS) vt_insert(tk_s, ti_s, logT, cand[j], j);
    __syncthreads();
  }
  // head items before the first 16-byte boundary, then 16-byte vectors, then the tail
  constexpr uint32_t E = 16 / sizeof(KT);
  const uintptr_t addr = reinterpret_cast<uintptr_t>(A);
  uint64_t head = ((16u - (addr & 15u)) & 15u) / sizeof(KT);
  if ((addr % sizeof(KT)) != 0) head = n;  // not naturally aligned: scalar path only
  if (head > n) head = n;
  const uint64_t nvec = (n - head) / E;
  const uint64_t tail0 = head + nvec * E;
  const uint64_t gtid = (uint64_t)blockIdx.x * VTHREADS + threadIdx.x;
  const uint64_t gstride = (uint64_t)gridDim.x * VTHREADS;
  for (uint64_t i = gtid; i < head; i += gstride) count_item(A[i], tk, ti, logT, scnt, acc, gl);
  const uint4* V = reinterpret_cast<const uint4*>(A + head);
  uint64_t v = gtid;
  for (; v + gstride < nvec; v += 2 * gstride) {  // two 16-byte loads in flight per thread
    const uint4 q0 = __ldg(V + v);
    const uint4 q1 = __ldg(V + v + gstride);
    const KT* x0 = reinterpret_cast<const KT*>(&q0);
    const KT* x1 = reinterpret_cast<const KT*>(&q1);
#pragma unroll
    for (uint32_t e = 0; e < E; ++e) count_item(x0[e], tk, ti, logT, scnt, acc, gl);
#pragma unroll
    for (uint32_t e = 0; e < E; ++e) count_item(x1[e], tk, ti, logT, scnt, acc, gl);
  }
  for (; v < nvec; v += gstride) {
    const uint4 q0 = __ldg(V + v);
    const KT* x0 = reinterpret_cast<const KT*>(&q0);
#pragma unroll
    for (uint32_t e = 0; e < E; ++e) count_item(x0[e], tk, ti, logT, scnt, acc, gl);
  }
  for (uint64_t i = tail0 + gtid; i < n; i += gstride) count_item(A[i], tk, ti, logT, scnt, acc, gl);
  if (!gl) {
    __syncthreads();
    const uint32_t T = 1u << logT;
    for (uint32_t h = threadIdx.x; h < T; h += VTHREADS)
      if (scnt[h]) atomicAdd(&acc[ti_s[h]], (unsigned long long)scnt[h]);
  }
}

// exact[j] = sum of acc over all candidate positions holding cand[j] (duplicates share counts)
template <typename KT>
__global__ void verify_finalize_kernel(const KT* cand, uint32_t cap, const uint32_t* d_n,
                                       const unsigned long long* acc, uint64_t* exact) {
  const uint32_t nc = eff_count(cap, d_n);
  const uint32_t j = blockIdx.x * blockDim.x + threadIdx.x;
  if (j >= nc) return;
  const KT x = cand[j];
  uint64_t t = 0;
  for (uint32_t i = 0; i < nc; ++i)
    if (cand[i] == x) t += acc[i];
  exact[j] = t;
}

size_t verify_ws(int kb, uint32_t cap, const DevInfo&) { return v_layout(kb, cap).total; }

template <typename KT>
static cudaError_t verify_run(const KT* A, uint64_t n, const KT* cand, uint32_t cap,
                              const uint32_t* d_n, uint64_t* exact, void* ws, cudaStream_t s,
                              const DevInfo& d) {
  VLayout L = v_layout(sizeof(KT), cap);
  unsigned char* w = static_cast<unsigned char*>(ws);
  auto* acc = reinterpret_cast<unsigned long long*>(w + L.acc);
  auto* gk = reinterpret_cast<KT*>(w + L.gkeys);
  auto* gi = reinterpret_cast<uint32_t*>(w + L.gidx);
  if (cap == 0) return cudaSuccess;
  verify_setup_kernel<KT><<<1, 1024, 0, s>>>(cand, cap, d_n, acc, gk, gi, L.logT);
  int nb = 0;
  cudaOccupancyMaxActiveBlocksPerMultiprocessor(&nb, verify_kernel<KT>, VTHREADS, 0);
  if (nb < 1) nb = 1;
  const uint64_t want = (n + (uint64_t)VTHREADS * 16 - 1) / ((uint64_t)VTHREADS * 16);
  const int grid = (int)std::max<uint64_t>(1, std::min<uint64_t>(want, (uint64_t)nb * d.sms));
  verify_kernel<KT><<<grid, VTHREADS, 0, s>>>(A, n, cand, cap, d_n, acc, gk, gi);
  verify_finalize_kernel<KT><<<(cap + 255) / 256, 256, 0, s>>>(cand, cap, d_n, acc, exact);
  return cudaGetLastError();
}

cudaError_t verify_launch(const void* A, uint64_t n, int kb, const void* cand, uint32_t cap,
                          const uint32_t* d_n_cand, uint64_t* exact, void* ws, cudaStream_t s,
                          const DevInfo& d) {
  if (kb == 4)
    return verify_run<uint32_t>(static_cast<const uint32_t*>(A), n,
                                static_cast<const uint32_t*>(cand), cap, d_n_cand, exact, ws, s, d);
  return verify_run<uint64_t>(static_cast<const uint64_t*>(A), n,
                              static_cast<const uint64_t*>(cand), cap, d_n_cand, exact, ws, s, d);
}

// ---- K5: {(x, f(x)) : f(x) >= floor(n/k) + 1}, ranked by (f desc, x asc). Internal: the
// candidates come from pss_prune, i.e. distinct root items.
template <typename KT>
__global__ void result_kernel(const KT* cand, uint32_t cap, const uint32_t* d_n,
                              const uint64_t* exact, uint64_t thr, KT* out_items,
                              uint64_t* out_counts, uint32_t* out_len) {
  const uint32_t nc = eff_count(cap, d_n);
  const uint32_t j = blockIdx.x * blockDim.x + threadIdx.x;
  if (j == 0) {
    uint32_t len = 0;
    for (uint32_t i = 0; i < nc; ++i) len += exact[i] >= thr;
    *out_len = len;
  }
  if (j >= nc || exact[j] < thr) return;
  const KT x = cand[j];
  const uint64_t f = exact[j];
  uint32_t rank = 0;
  for (uint32_t i = 0; i < nc; ++i)
    rank += exact[i] >= thr && (exact[i] > f || (exact[i] == f && cand[i] < x));
  out_items[rank] = x;
  out_counts[rank] = f;
}

cudaError_t result_launch(int kb, uint32_t cap, const void* cand, const uint32_t* d_n_cand,
                          const uint64_t* exact, uint64_t n, uint32_t k, void* out_items,
                          uint64_t* out_counts, uint32_t* out_len, cudaStream_t s) {
  const uint64_t thr = n / k + 1;
  const int grid = (int)((cap + 255) / 256 + (cap == 0));
  if (kb == 4)
    result_kernel<uint32_t><<<grid, 256, 0, s>>>(static_cast<const uint32_t*>(cand), cap,
                                                 d_n_cand, exact, thr,
                                                 static_cast<uint32_t*>(out_items), out_counts,
                                                 out_len);
  else
    result_kernel<uint64_t><<<grid, 256, 0, s>>>(static_cast<const uint64_t*>(cand), cap,
                                                 d_n_cand, exact, thr,
                                                 static_cast<uint64_t*>(out_items), out_counts,
                                                 out_len);
  return cudaGetLastError();
}

}  // namespace pss
