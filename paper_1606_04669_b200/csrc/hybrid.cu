// hybrid.cu -- the paper's hybrid MPI/OpenMP decomposition as an alternative tree shape (SURVEY.md
// section 8(f) row f4): "the input array is initially partitioned among the
// MPI processes, and then each MPI process sub-array is partitioned again among the available
// OpenMP threads". Leaves come from K1 with two-level bounds; each
// process reduces its T leaves with the fixed tree (R6), then the Pp process roots are reduced with
// the same tree. With T a power of two this is exactly pss_merge's tree over the Pp*T leaves (the
// first log2(T) levels pair complete groups), so one tree launch does it; otherwise one tree per
// process, then one over the roots. Host code only (kernels: K1, K2).
#include <algorithm>

#include "common.cuh"

namespace pss {
namespace {

int kbytes(int kt) { return kt == PSS_KEY_U32 ? 4 : (kt == PSS_KEY_U64 ? 8 : 0); }

struct HLayout {
  size_t items, counts, errs, sizes, scratch, total;
};
HLayout h_layout(int kb, uint32_t k, uint32_t Pp, uint32_t T, const DevInfo& d) {
  HLayout L;
  Bump b;
  L.items = b.take<unsigned char>((size_t)Pp * k * kb);
  L.counts = b.take<uint32_t>((size_t)Pp * k);
  L.errs = b.take<uint32_t>((size_t)Pp * k);
  L.sizes = b.take<uint32_t>(Pp);
  L.scratch = b.take<unsigned char>(
      std::max(merge_ws(kb, k, (uint32_t)std::max<uint64_t>((uint64_t)Pp * T, 1), d),
               merge_ws(kb, k, std::max(T, Pp), d)));
  L.total = b.bytes();
  return L;
}

bool pow2(uint32_t x) { return x && !(x & (x - 1)); }

}  // namespace
}  // namespace pss

using namespace pss;

extern "C" {

size_t pss_hybrid_workspace_bytes(uint64_t n, uint32_t k, uint32_t Pp, uint32_t T,
                                  pss_key_type kt) {
  const int kb = kbytes(kt);
  if (!kb || k < 2 || !Pp || !T || (uint64_t)Pp * T > 0xffffffffull) return 0;
  const DevInfo d = dev_info();
  return std::max(summarize_ws(n, kb, k, Pp * T, d), h_layout(kb, k, Pp, T, d).total);
}

pss_status pss_summarize_hybrid(const void* d_A, uint64_t n, pss_key_type kt, uint32_t k,
                                uint32_t Pp, uint32_t T, pss_summaries* leaves, void* d_ws,
                                size_t ws_bytes, cudaStream_t stream) {
  const int kb = kbytes(kt);
  if (!kb || k < 2 || !Pp || !T || !leaves || (n && !d_A) || !d_ws) return PSS_ERR_INVALID_ARG;
  if (n > PSS_MAX_N || k > PSS_MAX_K || (uint64_t)Pp * T > 0xffffffffull)
    return PSS_ERR_UNSUPPORTED;
  if (!leaves->items || !leaves->counts || !leaves->errs || !leaves->sizes)
    return PSS_ERR_INVALID_ARG;
  if (leaves->k != k || leaves->key_type != (int32_t)kt || leaves->count != Pp * T)
    return PSS_ERR_CAPACITY_MISMATCH;
  if (ws_bytes < pss_hybrid_workspace_bytes(n, k, Pp, T, kt)) return PSS_ERR_WORKSPACE_TOO_SMALL;
  const DevInfo d = dev_info();
  const cudaError_t e = summarize_launch(d_A, n, kb, k, Pp * T, leaves->items, leaves->counts,
                                         leaves->errs, leaves->sizes, d_ws, stream, d, 0,
                                         0xffffffffu, 0, T);
  return e == cudaSuccess ? PSS_OK : PSS_ERR_CUDA;
}

pss_status pss_merge_hybrid(const pss_summaries* leaves, uint32_t T, pss_summaries* root,
                            void* d_ws, size_t ws_bytes, cudaStream_t stream) {
  if (!leaves || !root || !d_ws || !T || !leaves->items || !leaves->counts || !leaves->errs ||
      !leaves->sizes || !root->items || !root->counts || !root->errs || !root->sizes)
    return PSS_ERR_INVALID_ARG;
  const int kb = kbytes(leaves->key_type);
  if (!kb || leaves->k < 2 || leaves->count == 0 || leaves->count % T) return PSS_ERR_INVALID_ARG;
  if (leaves->k > PSS_MAX_K) return PSS_ERR_UNSUPPORTED;
  if (root->k != leaves->k || root->key_type != leaves->key_type || root->count != 1)
    return PSS_ERR_CAPACITY_MISMATCH;
  const uint32_t k = leaves->k, Pp = leaves->count / T;
  if (ws_bytes < pss_hybrid_workspace_bytes(0, k, Pp, T, (pss_key_type)leaves->key_type))
    return PSS_ERR_WORKSPACE_TOO_SMALL;
  const DevInfo d = dev_info();
  unsigned char* w = static_cast<unsigned char*>(d_ws);
  const HLayout L = h_layout(kb, k, Pp, T, d);
  cudaError_t e;
  if (pow2(T) || Pp == 1 || T == 1) {
    e = merge_tree_launch(kb, k, leaves->count, leaves->items, leaves->counts, leaves->errs,
                          leaves->sizes, root->items, root->counts, root->errs, root->sizes,
                          w + L.scratch, stream, d);
  } else {
    e = cudaSuccess;
    const unsigned char* li = static_cast<const unsigned char*>(leaves->items);
    for (uint32_t p = 0; p < Pp && e == cudaSuccess; ++p) {
      const size_t o = (size_t)p * T * k;
      e = merge_tree_launch(kb, k, T, li + o * kb, leaves->counts + o, leaves->errs + o,
                            leaves->sizes + (size_t)p * T, w + L.items + (size_t)p * k * kb,
                            reinterpret_cast<uint32_t*>(w + L.counts) + (size_t)p * k,
                            reinterpret_cast<uint32_t*>(w + L.errs) + (size_t)p * k,
                            reinterpret_cast<uint32_t*>(w + L.sizes) + p, w + L.scratch, stream,
                            d);
    }
    if (e == cudaSuccess)
      e = merge_tree_launch(kb, k, Pp, w + L.items, reinterpret_cast<uint32_t*>(w + L.counts),
                            reinterpret_cast<uint32_t*>(w + L.errs),
                            reinterpret_cast<uint32_t*>(w + L.sizes), root->items, root->counts,
                            root->errs, root->sizes, w + L.scratch, stream, d);
  }
  return e == cudaSuccess ? PSS_OK : PSS_ERR_CUDA;
}

}  // extern "C"
