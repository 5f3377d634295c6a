// common.cuh -- device helpers shared by the libpss.so kernels (sm_100a only).
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

#include "pss.h"

#if defined(__CUDA_ARCH__) && (__CUDA_ARCH__ < 1000)
#error "libpss.so is written for sm_100a (B200) only"
#endif

#define PSS_FULL 0xffffffffu

namespace pss {

struct DevInfo {
  int sms = 148;
  int smem_optin = 227 * 1024;  // max dynamic smem per block (opt-in)
  int smem_per_sm = 228 * 1024;
};
DevInfo dev_info();

// ---- key traits: a multiplicative hash whose top bits index power-of-two tables
__device__ __forceinline__ uint32_t key_hash(uint32_t x) { return x * 0x9E3779B1u; }
__device__ __forceinline__ uint32_t key_hash(uint64_t x) {
  return (uint32_t)((x * 0x9E3779B97F4A7C15ull) >> 32);
}
template <typename KT>
__device__ __forceinline__ uint32_t hslot(KT x, uint32_t logH) {
  return logH ? key_hash(x) >> (32u - logH) : 0u;
}

__device__ __forceinline__ uint32_t lane_id() { return threadIdx.x & 31u; }
__device__ __forceinline__ uint32_t lanemask_lt() {
  uint32_t m;
  asm("mov.u32 %0, %%lanemask_lt;" : "=r"(m));
  return m;
}
// lane index of the n-th (0-based) set bit of `mask`, 32 if none; all lanes must be converged.
__device__ __forceinline__ uint32_t nth_set(uint32_t mask, uint32_t n) {
  const uint32_t lane = lane_id();
  bool me = ((mask >> lane) & 1u) && (uint32_t)__popc(mask & lanemask_lt()) == n;
  uint32_t b = __ballot_sync(PSS_FULL, me);
  return b ? (uint32_t)(__ffs(b) - 1) : 32u;
}

__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return (uint32_t)__cvta_generic_to_shared(p);
}

// ---- mbarrier + 1-D bulk async copy (TMA engine, cp.async.bulk) --------------------------
__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count)
               : "memory");
}
__device__ __forceinline__ void fence_mbar_init() {
  asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
}
__device__ __forceinline__ void fence_proxy_async() {
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
}
__device__ __forceinline__ void mbar_arrive_expect_tx(uint64_t* bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)),
               "r"(bytes)
               : "memory");
}
__device__ __forceinline__ void mbar_arrive(uint64_t* bar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(bar)) : "memory");
}
__device__ __forceinline__ bool mbar_try_wait(uint64_t* bar, uint32_t parity) {
  uint32_t ok;
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n\t"
      "selp.u32 %0, 1, 0, p;\n\t}"
      : "=r"(ok)
      : "r"(smem_u32(bar)), "r"(parity)
      : "memory");
  return ok != 0;
}
__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity) {
  while (!mbar_try_wait(bar, parity)) {
  }
}
// global -> shared bulk copy; dst/src 16-byte aligned, bytes a multiple of 16
__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, uint32_t bytes,
                                         uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::
          "r"(smem_u32(dst)),
      "l"(src), "r"(bytes), "r"(smem_u32(bar))
      : "memory");
}

__host__ __device__ __forceinline__ uint32_t ceil_log2(uint64_t x) {
  uint32_t l = 0;
  while ((1ull << l) < x) ++l;
  return l;
}
__host__ __device__ __forceinline__ size_t align_up(size_t x, size_t a) {
  return (x + a - 1) / a * a;
}

// gpu-scope acquire load / release store of a flag (producer-consumer across CTAs and kernels)
__device__ __forceinline__ uint32_t ld_acquire(const uint32_t* p) {
  uint32_t v;
  asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ void st_release(uint32_t* p, uint32_t v) {
  asm volatile("st.release.gpu.global.u32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}

// programmatic dependent launch: let the next kernel on the stream start (its CTAs are placed as
// this grid's CTAs exit); it synchronises through flags, then waits for this grid before exiting
__device__ __forceinline__ void pdl_launch_dependents() {
  asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
}
__device__ __forceinline__ void pdl_wait_prerequisites() {
  asm volatile("griddepcontrol.wait;" ::: "memory");
}

// canonical order (R5): count descending, then item ascending. true if (ca,ka) precedes (cb,kb).
template <typename KT>
__device__ __forceinline__ bool canon_before(uint32_t ca, KT ka, uint32_t cb, KT kb) {
  return ca > cb || (ca == cb && ka < kb);
}

// A kernel's dynamic shared-memory limit is a per-function, process-wide attribute: it is always
// raised to the device maximum (never to the size of one launch), so callers on concurrent
// streams with different sizes cannot race on it. Occupancy depends on each launch's own size.
template <typename Kern>
inline cudaError_t allow_max_smem(Kern kern, const DevInfo& d) {
  cudaFuncAttributes fa;
  cudaError_t e = cudaFuncGetAttributes(&fa, kern);
  if (e == cudaSuccess)
    e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize,
                             d.smem_optin - (int)fa.sharedSizeBytes);
  if (e != cudaSuccess) (void)cudaGetLastError();
  return e;
}

// ---- host-side bump allocator over a workspace
struct Bump {
  size_t off = 0;
  size_t al = 256;  // alignment of every region (16 is enough for shared-memory layouts)
  template <typename T>
  size_t take(size_t count) {
    size_t o = align_up(off, al);
    off = o + count * sizeof(T);
    return o;
  }
  size_t bytes() const { return align_up(off, al); }
};

// ---- internal launchers (csrc/*.cu) ----------------------------------------------------
size_t summarize_ws(uint64_t n, int kb, uint32_t k, uint32_t P, const DevInfo& d);
cudaError_t summarize_launch(const void* A, uint64_t n, int kb, uint32_t k, uint32_t P,
                             void* items, uint32_t* counts, uint32_t* errs, uint32_t* sizes,
                             void* ws, cudaStream_t s, const DevInfo& d, uint32_t r0 = 0,
                             uint32_t r1 = 0xffffffffu, uint32_t qi = 0, uint32_t T = 1,
                             uint32_t* leaf_flags = nullptr, bool pdl = false);
// K0 (hot.cu): the frequent keys of A[lo, hi) (u32) for K1's level-pinned bypass. `out`, HOT_WORDS
// words in the workspace: [0] number of keys (0: none), [1] the table's multiplier, [2] their
// occurrences in the sample, [3] sample size, [4..) the keys by rank, then a one-probe table of
// 2^HOT_LOG entries: with ha = key * multiplier and h = ha >> 21, entry h holds (rank ^ h) << 21 |
// ha's low 21 bits (rank HOT_NONE for an empty entry), so rotl(entry ^ ha, 11) is the key's rank
// if it is in the table and a value >= HOT_MAX otherwise.
constexpr uint32_t HOT_MAX = 64, HOT_LOG = 11, HOT_NONE = 127;
constexpr uint32_t HOT_TAG_MASK = (1u << (32 - HOT_LOG)) - 1u;
constexpr uint32_t HOT_WORDS = 4 + HOT_MAX + (1u << HOT_LOG);
cudaError_t hot_sample_launch(const void* A, uint64_t lo, uint64_t hi, uint32_t* out, bool force,
                              cudaStream_t s);
// K1h (hist.cu): leaves of blocks with at most k distinct keys as exact histograms; the other
// leaves are flagged (flagged[r] = 1) for K1
bool hist_used(uint64_t n, int kb, uint32_t k, uint32_t P, const DevInfo& d);
cudaError_t hist_launch(const void* A, uint64_t n, int kb, uint32_t k, uint32_t P, void* items,
                        uint32_t* counts, uint32_t* errs, uint32_t* sizes, uint32_t* queue,
                        unsigned char* flagged, cudaStream_t s, const DevInfo& d, uint32_t r0,
                        uint32_t r1, uint32_t T, uint32_t* leaf_flags);
// K1e (epoch.cu): the leaf summaries of u32 keys for 64 <= k <= 2048, one CTA per block, epoch by
// epoch; K1 takes the shapes it does not cover
bool epoch_used(uint64_t n, int kb, uint32_t k, uint32_t P, const DevInfo& d);
cudaError_t epoch_launch(const void* A, uint64_t n, uint32_t k, uint32_t P, void* items,
                         uint32_t* counts, uint32_t* errs, uint32_t* sizes, uint32_t* queue,
                         const unsigned char* skip, cudaStream_t s, const DevInfo& d, uint32_t r0,
                         uint32_t r1, uint32_t T, uint32_t* leaf_flags, bool pdl);
// wide.cu: summaries with 64-bit counts and errors (the tree above the leaves, > 2^31 items)
size_t wide_combine_ws(int kb, uint32_t k, const DevInfo& d);
size_t wide_merge_ws(int kb, uint32_t k, uint32_t count, const DevInfo& d);
cudaError_t wide_combine_launch(int kb, uint32_t k, uint32_t count, const void* ai,
                                const uint64_t* ac, const uint64_t* ae, const uint32_t* as,
                                const void* bi, const uint64_t* bc, const uint64_t* be,
                                const uint32_t* bs, void* oi, uint64_t* oc, uint64_t* oe,
                                uint32_t* os, void* scratch, cudaStream_t s, const DevInfo& d);
cudaError_t wide_merge_launch(int kb, uint32_t k, uint32_t count, const void* items,
                              const uint64_t* counts, const uint64_t* errs, const uint32_t* sizes,
                              void* ri, uint64_t* rc, uint64_t* re, uint32_t* rs, void* ws,
                              cudaStream_t s, const DevInfo& d);
cudaError_t widen_launch(int kb, uint32_t k, uint32_t count, const void* items,
                         const uint32_t* counts, const uint32_t* errs, const uint32_t* sizes,
                         void* wi, uint64_t* wc, uint64_t* we, uint32_t* wsz, cudaStream_t s);
cudaError_t narrow_launch(int kb, uint32_t k, uint32_t count, const void* wi, const uint64_t* wc,
                          const uint64_t* we, const uint32_t* wsz, void* items, uint32_t* counts,
                          uint32_t* errs, uint32_t* sizes, cudaStream_t s);
cudaError_t wide_prune_launch(int kb, const void* items, const uint64_t* counts,
                              const uint32_t* sizes, uint64_t n, uint32_t k, void* cand,
                              uint32_t* n_cand, cudaStream_t s);
// partition queues in the summarize workspace: launches over disjoint ranges [r0, r1) that may be
// in flight together use distinct qi < SS_MAX_RANGES
constexpr uint32_t SS_MAX_RANGES = 64;

size_t merge_ws(int kb, uint32_t k, uint32_t P, const DevInfo& d);
// fixed binary tree over P leaves -> root (canonical). With leaf_flags, the leaves may still be
// in production (K1 sets leaf_flags[r] once leaf r is written): the tree kernel is launched as a
// programmatic dependent of K1 and waits per leaf; merge_tree_reset must have run before K1.
cudaError_t merge_tree_launch(int kb, uint32_t k, uint32_t P, const void* items,
                              const uint32_t* counts, const uint32_t* errs, const uint32_t* sizes,
                              void* r_items, uint32_t* r_counts, uint32_t* r_errs,
                              uint32_t* r_sizes, void* ws, cudaStream_t s, const DevInfo& d,
                              const uint32_t* leaf_flags = nullptr);
// true if merge_tree_launch(..., leaf_flags) overlaps K1 for this shape (persistent tree kernel)
bool merge_tree_overlaps(int kb, uint32_t k, uint32_t P, const DevInfo& d);
// clears the tree's node flags and task queue (before K1 when the tree overlaps it)
cudaError_t merge_tree_reset(int kb, uint32_t k, uint32_t P, void* ws, cudaStream_t s,
                             const DevInfo& d);
size_t combine_ws(int kb, uint32_t k, uint32_t count, const DevInfo& d);
cudaError_t combine_launch(int kb, uint32_t k, uint32_t count, const void* a_items,
                           const uint32_t* a_counts, const uint32_t* a_errs,
                           const uint32_t* a_sizes, const void* b_items, const uint32_t* b_counts,
                           const uint32_t* b_errs, const uint32_t* b_sizes, void* o_items,
                           uint32_t* o_counts, uint32_t* o_errs, uint32_t* o_sizes, void* ws,
                           cudaStream_t s, const DevInfo& d);

cudaError_t prune_launch(int kb, uint32_t k, const void* items, const uint32_t* counts,
                         const uint32_t* sizes, uint64_t n, void* cand, uint32_t* n_cand,
                         cudaStream_t s);

size_t verify_ws(int kb, uint32_t cap, const DevInfo& d);
cudaError_t verify_launch(const void* A, uint64_t n, int kb, const void* cand, uint32_t cap,
                          const uint32_t* d_n_cand, uint64_t* exact, void* ws, cudaStream_t s,
                          const DevInfo& d);
size_t exact_ws(int kb, uint64_t n, uint32_t k);
cudaError_t result_launch(int kb, uint32_t cap, const void* cand, const uint32_t* d_n_cand,
                          const uint64_t* exact, uint64_t n, uint32_t k, void* out_items,
                          uint64_t* out_counts, uint32_t* out_len, cudaStream_t s);

}  // namespace pss
