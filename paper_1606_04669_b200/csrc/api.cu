// api.cu -- the C-ABI of libpss.so (include/pss.h): argument validation, workspace layout and
// launch order. No torch types, no allocation, no global mutable state.
#include <algorithm>
#include <cstdlib>

#include "common.cuh"

namespace pss {

DevInfo dev_info() {
  DevInfo d;
  int dev = 0;
  if (cudaGetDevice(&dev) != cudaSuccess) return d;
  int v = 0;
  if (cudaDeviceGetAttribute(&v, cudaDevAttrMultiProcessorCount, dev) == cudaSuccess) d.sms = v;
  if (cudaDeviceGetAttribute(&v, cudaDevAttrMaxSharedMemoryPerBlockOptin, dev) == cudaSuccess)
    d.smem_optin = v;
  if (cudaDeviceGetAttribute(&v, cudaDevAttrMaxSharedMemoryPerMultiprocessor, dev) ==
      cudaSuccess)
    d.smem_per_sm = v;
  return d;
}

static int key_bytes(int kt) { return kt == PSS_KEY_U32 ? 4 : (kt == PSS_KEY_U64 ? 8 : 0); }

static bool summaries_ok(const pss_summaries* s) {
  return s && key_bytes(s->key_type) && s->items && s->counts && s->errs && s->sizes &&
         s->k >= 2 && s->count >= 1;
}

static pss_status cuda_status(cudaError_t e) { return e == cudaSuccess ? PSS_OK : PSS_ERR_CUDA; }

// workspace of the fused summarize + merge: K1's, the tree's (disjoint: the two kernels overlap)
// and one ready flag per leaf
struct SMLayout {
  size_t sum, merge, flags, total;
};
static SMLayout sm_layout(uint64_t n, int kb, uint32_t k, uint32_t P, const DevInfo& d) {
  SMLayout L;
  Bump b;
  L.sum = b.take<unsigned char>(summarize_ws(n, kb, k, P, d));
  L.merge = b.take<unsigned char>(merge_ws(kb, k, P, d));
  L.flags = b.take<uint32_t>(P);
  L.total = b.bytes();
  return L;
}

// a2 + a4: K1, then the tree kernel launched as its programmatic dependent so that the tree's
// CTAs take the SMs K1's persistent CTAs leave in its last wave and combine leaves as soon as
// they are written (per-leaf flags); shapes the persistent tree does not cover run in order
static cudaError_t summarize_merge_launch(const void* A, uint64_t n, int kb, uint32_t k,
                                          uint32_t P, void* li, uint32_t* lc, uint32_t* le,
                                          uint32_t* ls, void* ri, uint32_t* rc, uint32_t* re,
                                          uint32_t* rs, void* ws, cudaStream_t s,
                                          const DevInfo& d) {
  unsigned char* w = static_cast<unsigned char*>(ws);
  const SMLayout L = sm_layout(n, kb, k, P, d);
  uint32_t* flags = reinterpret_cast<uint32_t*>(w + L.flags);
  const bool ovl = merge_tree_overlaps(kb, k, P, d) && !std::getenv("PSS_NO_OVERLAP");
  cudaError_t e = cudaSuccess;
  if (ovl) {
    e = cudaMemsetAsync(flags, 0, (size_t)P * sizeof(uint32_t), s);
    if (e == cudaSuccess) e = merge_tree_reset(kb, k, P, w + L.merge, s, d);
  }
  if (e == cudaSuccess)
    e = summarize_launch(A, n, kb, k, P, li, lc, le, ls, w + L.sum, s, d, 0, 0xffffffffu, 0, 1,
                         ovl ? flags : nullptr, ovl);
  if (e == cudaSuccess)
    e = merge_tree_launch(kb, k, P, li, lc, le, ls, ri, rc, re, rs, w + L.merge, s, d,
                          ovl ? flags : nullptr);
  return e;
}

// workspace plan of pss_query: leaves, root, candidates, exact counts, output staging, scratch
struct QLayout {
  size_t l_items, l_counts, l_errs, l_sizes, r_items, r_counts, r_errs, r_sizes, cand, ncand,
      exact, o_items, o_counts, o_len, scratch, total;
};
static QLayout q_layout(uint64_t n, int kb, uint32_t k, uint32_t P, const DevInfo& d) {
  QLayout L;
  Bump b;
  L.l_items = b.take<unsigned char>((size_t)P * k * kb);
  L.l_counts = b.take<uint32_t>((size_t)P * k);
  L.l_errs = b.take<uint32_t>((size_t)P * k);
  L.l_sizes = b.take<uint32_t>(P);
  L.r_items = b.take<unsigned char>((size_t)k * kb);
  L.r_counts = b.take<uint32_t>(k);
  L.r_errs = b.take<uint32_t>(k);
  L.r_sizes = b.take<uint32_t>(1);
  L.cand = b.take<unsigned char>((size_t)k * kb);
  L.ncand = b.take<uint32_t>(1);
  L.exact = b.take<uint64_t>(k);
  L.o_items = b.take<unsigned char>((size_t)k * kb);
  L.o_counts = b.take<uint64_t>(k);
  L.o_len = b.take<uint32_t>(1);
  const size_t sc = std::max({sm_layout(n, kb, k, P, d).total, verify_ws(kb, k, d)});
  L.scratch = b.take<unsigned char>(sc);
  L.total = b.bytes();
  return L;
}

}  // namespace pss

using namespace pss;

extern "C" {

const char* pss_status_string(pss_status s) {
  switch (s) {
    case PSS_OK: return "PSS_OK";
    case PSS_ERR_INVALID_ARG: return "PSS_ERR_INVALID_ARG";
    case PSS_ERR_UNSUPPORTED: return "PSS_ERR_UNSUPPORTED";
    case PSS_ERR_CAPACITY_MISMATCH: return "PSS_ERR_CAPACITY_MISMATCH";
    case PSS_ERR_WORKSPACE_TOO_SMALL: return "PSS_ERR_WORKSPACE_TOO_SMALL";
    case PSS_ERR_CUDA: return "PSS_ERR_CUDA";
  }
  return "PSS_UNKNOWN_STATUS";
}

static bool wsummaries_ok(const pss_wsummaries* s) {
  return s && key_bytes(s->key_type) && s->items && s->counts && s->errs && s->sizes &&
         s->k >= 2 && s->count >= 1;
}

pss_status pss_widen(const pss_summaries* in, pss_wsummaries* out, cudaStream_t stream) {
  if (!summaries_ok(in) || !wsummaries_ok(out)) return PSS_ERR_INVALID_ARG;
  if (in->k != out->k || in->key_type != out->key_type || in->count != out->count)
    return PSS_ERR_CAPACITY_MISMATCH;
  return cuda_status(widen_launch(key_bytes(in->key_type), in->k, in->count, in->items,
                                  in->counts, in->errs, in->sizes, out->items, out->counts,
                                  out->errs, out->sizes, stream));
}

pss_status pss_combine_wide(const pss_wsummaries* a, const pss_wsummaries* b,
                            pss_wsummaries* out, void* d_ws, size_t ws_bytes,
                            cudaStream_t stream) {
  if (!wsummaries_ok(a) || !wsummaries_ok(b) || !wsummaries_ok(out) || !d_ws)
    return PSS_ERR_INVALID_ARG;
  if (a->k > PSS_MAX_K) return PSS_ERR_UNSUPPORTED;
  if (a->k != b->k || a->k != out->k || a->key_type != b->key_type ||
      a->key_type != out->key_type || a->count != b->count || a->count != out->count)
    return PSS_ERR_CAPACITY_MISMATCH;
  const int kb = key_bytes(a->key_type);
  const DevInfo d = dev_info();
  if (ws_bytes < wide_combine_ws(kb, a->k, d) + 256) return PSS_ERR_WORKSPACE_TOO_SMALL;
  return cuda_status(wide_combine_launch(kb, a->k, a->count, a->items, a->counts, a->errs,
                                         a->sizes, b->items, b->counts, b->errs, b->sizes,
                                         out->items, out->counts, out->errs, out->sizes, d_ws,
                                         stream, d));
}

pss_status pss_merge_wide(const pss_wsummaries* nodes, pss_wsummaries* root, void* d_ws,
                          size_t ws_bytes, cudaStream_t stream) {
  if (!wsummaries_ok(nodes) || !wsummaries_ok(root) || !d_ws) return PSS_ERR_INVALID_ARG;
  if (nodes->k > PSS_MAX_K) return PSS_ERR_UNSUPPORTED;
  if (root->k != nodes->k || root->key_type != nodes->key_type || root->count != 1)
    return PSS_ERR_CAPACITY_MISMATCH;
  const int kb = key_bytes(nodes->key_type);
  const DevInfo d = dev_info();
  if (ws_bytes < wide_merge_ws(kb, nodes->k, nodes->count, d) + 256)
    return PSS_ERR_WORKSPACE_TOO_SMALL;
  return cuda_status(wide_merge_launch(kb, nodes->k, nodes->count, nodes->items, nodes->counts,
                                       nodes->errs, nodes->sizes, root->items, root->counts,
                                       root->errs, root->sizes, d_ws, stream, d));
}

pss_status pss_prune_wide(const pss_wsummaries* root, uint64_t n, void* d_cand,
                          uint32_t* d_n_cand, cudaStream_t stream) {
  if (!wsummaries_ok(root) || !d_cand || !d_n_cand || root->count != 1)
    return PSS_ERR_INVALID_ARG;
  if (n >> 63) return PSS_ERR_UNSUPPORTED;
  return cuda_status(wide_prune_launch(key_bytes(root->key_type), root->items, root->counts,
                                       root->sizes, n, root->k, d_cand, d_n_cand, stream));
}

const char* pss_version(void) { return "pss-b200 0.2 (sm_100a)"; }

int pss_leaf_kernels(uint64_t n, uint32_t k, uint32_t P, pss_key_type kt) {
  const int kb = key_bytes(kt);
  if (!kb || k < 2 || P == 0) return 0;
  const DevInfo d = dev_info();
  return (epoch_used(n, kb, k, P, d) ? PSS_LEAF_K1E : PSS_LEAF_K1) |
         (hist_used(n, kb, k, P, d) ? PSS_LEAF_K1H : 0);
}

size_t pss_workspace_bytes(int op, uint64_t n, uint32_t k, uint32_t P, pss_key_type kt) {
  const int kb = key_bytes(kt);
  if (!kb) return 0;
  const DevInfo d = dev_info();
  switch (op) {
    case PSS_OP_SUMMARIZE: return summarize_ws(n, kb, k, P, d);
    case PSS_OP_MERGE: return merge_ws(kb, k, P ? P : 1, d);
    case PSS_OP_COMBINE: return combine_ws(kb, k, P, d);
    case PSS_OP_VERIFY: return verify_ws(kb, k, d);
    case PSS_OP_QUERY: return q_layout(n, kb, k, P ? P : 1, d).total;
    case PSS_OP_EXACT: return exact_ws(kb, n, k);
    case PSS_OP_SUMMARIZE_MERGE: return sm_layout(n, kb, k, P ? P : 1, d).total;
    case PSS_OP_COMBINE_WIDE: return wide_combine_ws(kb, k, d) + 256;
    case PSS_OP_MERGE_WIDE: return wide_merge_ws(kb, k, P ? P : 1, d) + 256;
  }
  return 0;
}

pss_status pss_summarize(const void* d_A, uint64_t n, pss_key_type kt, uint32_t k, uint32_t P,
                         pss_summaries* leaves, void* d_ws, size_t ws_bytes,
                         cudaStream_t stream) {
  const int kb = key_bytes(kt);
  if (!kb || k < 2 || P == 0 || !leaves || (n && !d_A) || !d_ws) return PSS_ERR_INVALID_ARG;
  if (n > PSS_MAX_N || k > PSS_MAX_K) return PSS_ERR_UNSUPPORTED;
  if (!summaries_ok(leaves)) return PSS_ERR_INVALID_ARG;
  if (leaves->k != k || leaves->key_type != (int32_t)kt || leaves->count != P)
    return PSS_ERR_CAPACITY_MISMATCH;
  const DevInfo d = dev_info();
  if (ws_bytes < summarize_ws(n, kb, k, P, d)) return PSS_ERR_WORKSPACE_TOO_SMALL;
  return cuda_status(summarize_launch(d_A, n, kb, k, P, leaves->items, leaves->counts,
                                      leaves->errs, leaves->sizes, d_ws, stream, d));
}

pss_status pss_summarize_merge(const void* d_A, uint64_t n, pss_key_type kt, uint32_t k,
                               uint32_t P, pss_summaries* leaves, pss_summaries* root, void* d_ws,
                               size_t ws_bytes, cudaStream_t stream) {
  const int kb = key_bytes(kt);
  if (!kb || k < 2 || P == 0 || !leaves || !root || (n && !d_A) || !d_ws)
    return PSS_ERR_INVALID_ARG;
  if (n > PSS_MAX_N || k > PSS_MAX_K) return PSS_ERR_UNSUPPORTED;
  if (!summaries_ok(leaves) || !summaries_ok(root)) return PSS_ERR_INVALID_ARG;
  if (leaves->k != k || leaves->key_type != (int32_t)kt || leaves->count != P ||
      root->k != k || root->key_type != (int32_t)kt || root->count != 1)
    return PSS_ERR_CAPACITY_MISMATCH;
  const DevInfo d = dev_info();
  if (ws_bytes < sm_layout(n, kb, k, P, d).total) return PSS_ERR_WORKSPACE_TOO_SMALL;
  return cuda_status(summarize_merge_launch(d_A, n, kb, k, P, leaves->items, leaves->counts,
                                            leaves->errs, leaves->sizes, root->items,
                                            root->counts, root->errs, root->sizes, d_ws, stream,
                                            d));
}

pss_status pss_merge(const pss_summaries* leaves, pss_summaries* root, void* d_ws,
                     size_t ws_bytes, cudaStream_t stream) {
  if (!summaries_ok(leaves) || !summaries_ok(root) || !d_ws) return PSS_ERR_INVALID_ARG;
  if (leaves->k > PSS_MAX_K) return PSS_ERR_UNSUPPORTED;
  if (root->k != leaves->k || root->key_type != leaves->key_type || root->count != 1)
    return PSS_ERR_CAPACITY_MISMATCH;
  const int kb = key_bytes(leaves->key_type);
  const DevInfo d = dev_info();
  if (ws_bytes < merge_ws(kb, leaves->k, leaves->count, d)) return PSS_ERR_WORKSPACE_TOO_SMALL;
  return cuda_status(merge_tree_launch(kb, leaves->k, leaves->count, leaves->items,
                                       leaves->counts, leaves->errs, leaves->sizes, root->items,
                                       root->counts, root->errs, root->sizes, d_ws, stream, d));
}

pss_status pss_combine(const pss_summaries* a, const pss_summaries* b, pss_summaries* out,
                       void* d_ws, size_t ws_bytes, cudaStream_t stream) {
  if (!summaries_ok(a) || !summaries_ok(b) || !summaries_ok(out) || !d_ws)
    return PSS_ERR_INVALID_ARG;
  if (a->k > PSS_MAX_K) return PSS_ERR_UNSUPPORTED;
  if (a->k != b->k || a->k != out->k || a->key_type != b->key_type ||
      a->key_type != out->key_type || a->count != b->count || a->count != out->count)
    return PSS_ERR_CAPACITY_MISMATCH;
  const int kb = key_bytes(a->key_type);
  const DevInfo d = dev_info();
  if (ws_bytes < combine_ws(kb, a->k, a->count, d)) return PSS_ERR_WORKSPACE_TOO_SMALL;
  return cuda_status(combine_launch(kb, a->k, a->count, a->items, a->counts, a->errs, a->sizes,
                                    b->items, b->counts, b->errs, b->sizes, out->items,
                                    out->counts, out->errs, out->sizes, d_ws, stream, d));
}

pss_status pss_prune(const pss_summaries* root, uint64_t n, void* d_cand, uint32_t* d_n_cand,
                     cudaStream_t stream) {
  if (!summaries_ok(root) || !d_cand || !d_n_cand || root->count != 1) return PSS_ERR_INVALID_ARG;
  if (n >> 63) return PSS_ERR_UNSUPPORTED;  // the threshold is 64-bit arithmetic
  return cuda_status(prune_launch(key_bytes(root->key_type), root->k, root->items, root->counts,
                                  root->sizes, n, d_cand, d_n_cand, stream));
}

pss_status pss_verify(const void* d_A, uint64_t n, pss_key_type kt, const void* d_cand,
                      uint32_t n_cand, const uint32_t* d_n_cand, uint64_t* d_exact, void* d_ws,
                      size_t ws_bytes, cudaStream_t stream) {
  const int kb = key_bytes(kt);
  if (!kb || (n && !d_A) || (n_cand && (!d_cand || !d_exact)) || !d_ws) return PSS_ERR_INVALID_ARG;
  if (n > PSS_MAX_N) return PSS_ERR_UNSUPPORTED;
  const DevInfo d = dev_info();
  if (ws_bytes < verify_ws(kb, n_cand, d)) return PSS_ERR_WORKSPACE_TOO_SMALL;
  return cuda_status(verify_launch(d_A, n, kb, d_cand, n_cand, d_n_cand, d_exact, d_ws, stream, d));
}

pss_status pss_report(const void* d_cand, uint32_t n_cand, const uint32_t* d_n_cand,
                      const uint64_t* d_exact, pss_key_type kt, uint64_t n, uint32_t k,
                      void* d_out_items, uint64_t* d_out_counts, uint32_t* d_out_len,
                      cudaStream_t stream) {
  const int kb = key_bytes(kt);
  if (!kb || k < 2 || !d_out_len || (n_cand && (!d_cand || !d_exact || !d_out_items || !d_out_counts)))
    return PSS_ERR_INVALID_ARG;
  if (n >> 63) return PSS_ERR_UNSUPPORTED;  // 64-bit threshold and exact counts
  return cuda_status(result_launch(kb, n_cand, d_cand, d_n_cand, d_exact, n, k, d_out_items,
                                   d_out_counts, d_out_len, stream));
}

// a5..a7 after the root: prune, verify, report
static pss_status prune_verify(const void* d_A, uint64_t n, int kb, uint32_t k,
                               void* d_out_items, uint64_t* d_out_counts, uint32_t* d_out_len,
                               unsigned char* w, const QLayout& L, cudaStream_t s,
                               const DevInfo& d) {
  void* ri = w + L.r_items;
  uint32_t* rc = reinterpret_cast<uint32_t*>(w + L.r_counts);
  uint32_t* rs = reinterpret_cast<uint32_t*>(w + L.r_sizes);
  void* cand = w + L.cand;
  uint32_t* nc = reinterpret_cast<uint32_t*>(w + L.ncand);
  uint64_t* exact = reinterpret_cast<uint64_t*>(w + L.exact);
  cudaError_t e = prune_launch(kb, k, ri, rc, rs, n, cand, nc, s);
  if (e == cudaSuccess) e = verify_launch(d_A, n, kb, cand, k, nc, exact, w + L.scratch, s, d);
  if (e == cudaSuccess)
    e = result_launch(kb, k, cand, nc, exact, n, k, d_out_items, d_out_counts, d_out_len, s);
  return cuda_status(e);
}

// a4..a7 over leaves already in the workspace
static pss_status tree_and_verify(const void* d_A, uint64_t n, int kb, uint32_t k, uint32_t P,
                                  void* d_out_items, uint64_t* d_out_counts, uint32_t* d_out_len,
                                  unsigned char* w, const QLayout& L, cudaStream_t s,
                                  const DevInfo& d) {
  const cudaError_t e = merge_tree_launch(
      kb, k, P, w + L.l_items, reinterpret_cast<uint32_t*>(w + L.l_counts),
      reinterpret_cast<uint32_t*>(w + L.l_errs), reinterpret_cast<uint32_t*>(w + L.l_sizes),
      w + L.r_items, reinterpret_cast<uint32_t*>(w + L.r_counts),
      reinterpret_cast<uint32_t*>(w + L.r_errs), reinterpret_cast<uint32_t*>(w + L.r_sizes),
      w + L.scratch, s, d);
  if (e != cudaSuccess) return PSS_ERR_CUDA;
  return prune_verify(d_A, n, kb, k, d_out_items, d_out_counts, d_out_len, w, L, s, d);
}

// a2 + a4 (overlapped) then a5..a7
static pss_status query_impl(const void* d_A, uint64_t n, int kb, uint32_t k, uint32_t P,
                             void* d_out_items, uint64_t* d_out_counts, uint32_t* d_out_len,
                             unsigned char* w, const QLayout& L, cudaStream_t s,
                             const DevInfo& d) {
  const cudaError_t e = summarize_merge_launch(
      d_A, n, kb, k, P, w + L.l_items, reinterpret_cast<uint32_t*>(w + L.l_counts),
      reinterpret_cast<uint32_t*>(w + L.l_errs), reinterpret_cast<uint32_t*>(w + L.l_sizes),
      w + L.r_items, reinterpret_cast<uint32_t*>(w + L.r_counts),
      reinterpret_cast<uint32_t*>(w + L.r_errs), reinterpret_cast<uint32_t*>(w + L.r_sizes),
      w + L.scratch, s, d);
  if (e != cudaSuccess) return PSS_ERR_CUDA;
  return prune_verify(d_A, n, kb, k, d_out_items, d_out_counts, d_out_len, w, L, s, d);
}

// chunks of the pipelined host->device copy in pss_query_host (1 = copy, then compute)
static uint32_t h2d_chunks(uint64_t n, int kb, uint32_t P) {
  uint64_t G = n * kb >= (64ull << 20) ? 16 : 1;
  if (const char* v = std::getenv("PSS_DEBUG_H2D_CHUNKS")) G = (uint64_t)std::atoll(v);
  G = std::min<uint64_t>({G, (uint64_t)P, (uint64_t)SS_MAX_RANGES});
  return G ? (uint32_t)G : 1u;
}

pss_status pss_query(const void* d_A, uint64_t n, pss_key_type kt, uint32_t k, uint32_t P,
                     void* d_out_items, uint64_t* d_out_counts, uint32_t* d_out_len, void* d_ws,
                     size_t ws_bytes, cudaStream_t stream) {
  const int kb = key_bytes(kt);
  if (!kb || k < 2 || P == 0 || (n && !d_A) || !d_out_items || !d_out_counts || !d_out_len ||
      !d_ws)
    return PSS_ERR_INVALID_ARG;
  if (n > PSS_MAX_N || k > PSS_MAX_K) return PSS_ERR_UNSUPPORTED;
  const DevInfo d = dev_info();
  const QLayout L = q_layout(n, kb, k, P, d);
  if (ws_bytes < L.total) return PSS_ERR_WORKSPACE_TOO_SMALL;
  return query_impl(d_A, n, kb, k, P, d_out_items, d_out_counts, d_out_len,
                    static_cast<unsigned char*>(d_ws), L, stream, d);
}

pss_status pss_query_host(const void* h_A, void* d_A, uint64_t n, pss_key_type kt, uint32_t k,
                          uint32_t P, void* h_out_items, uint64_t* h_out_counts,
                          uint32_t* h_out_len, void* d_ws, size_t ws_bytes,
                          cudaStream_t stream) {
  const int kb = key_bytes(kt);
  if (!kb || k < 2 || P == 0 || (n && (!d_A || !h_A)) || !h_out_items || !h_out_counts ||
      !h_out_len || !d_ws)
    return PSS_ERR_INVALID_ARG;
  if (n > PSS_MAX_N || k > PSS_MAX_K) return PSS_ERR_UNSUPPORTED;
  const DevInfo d = dev_info();
  const QLayout L = q_layout(n, kb, k, P, d);
  if (ws_bytes < L.total) return PSS_ERR_WORKSPACE_TOO_SMALL;
  unsigned char* w = static_cast<unsigned char*>(d_ws);
  cudaError_t e = cudaSuccess;
  // The copy of A is cut at partition boundaries into G chunks on a private copy stream; the
  // leaves of chunk g are summarized on `stream` as soon as its bytes have landed, so the
  // summaries overlap the host->device transfer and only the last chunk's leaves, the merge
  // tree and the verification pass (which needs all of A) run after it.
  const uint32_t G = h2d_chunks(n, kb, P);
  if (G <= 1) {
    if (n) e = cudaMemcpyAsync(d_A, h_A, n * kb, cudaMemcpyHostToDevice, stream);
    if (e != cudaSuccess) return PSS_ERR_CUDA;
    pss_status st = query_impl(d_A, n, kb, k, P, w + L.o_items,
                               reinterpret_cast<uint64_t*>(w + L.o_counts),
                               reinterpret_cast<uint32_t*>(w + L.o_len), w, L, stream, d);
    if (st != PSS_OK) return st;
  } else {
    cudaStream_t cs = nullptr;
    cudaEvent_t ev[SS_MAX_RANGES + 1] = {};
    e = cudaStreamCreateWithFlags(&cs, cudaStreamNonBlocking);
    for (uint32_t g = 0; g <= G && e == cudaSuccess; ++g)
      e = cudaEventCreateWithFlags(&ev[g], cudaEventDisableTiming);
    // the copies must not overwrite d_A before earlier work on `stream` is done with it
    if (e == cudaSuccess) e = cudaEventRecord(ev[G], stream);
    if (e == cudaSuccess) e = cudaStreamWaitEvent(cs, ev[G], 0);
    const char* hA = static_cast<const char*>(h_A);
    char* dA = static_cast<char*>(d_A);
    for (uint32_t g = 0; g < G && e == cudaSuccess; ++g) {
      const uint32_t r0 = (uint32_t)((uint64_t)g * P / G), r1 = (uint32_t)((uint64_t)(g + 1) * P / G);
      const uint64_t lo = (uint64_t)r0 * n / P, hi = (uint64_t)r1 * n / P;  // a1 bounds
      e = cudaMemcpyAsync(dA + lo * kb, hA + lo * kb, (hi - lo) * kb, cudaMemcpyHostToDevice, cs);
      if (e == cudaSuccess) e = cudaEventRecord(ev[g], cs);
      if (e == cudaSuccess) e = cudaStreamWaitEvent(stream, ev[g], 0);
      if (e == cudaSuccess)
        e = summarize_launch(d_A, n, kb, k, P, w + L.l_items,
                             reinterpret_cast<uint32_t*>(w + L.l_counts),
                             reinterpret_cast<uint32_t*>(w + L.l_errs),
                             reinterpret_cast<uint32_t*>(w + L.l_sizes), w + L.scratch, stream, d,
                             r0, r1, g);
    }
    // stream-ordered release: destruction waits for the enqueued work
    for (uint32_t g = 0; g <= G; ++g)
      if (ev[g]) cudaEventDestroy(ev[g]);
    if (cs) cudaStreamDestroy(cs);
    if (e != cudaSuccess) return PSS_ERR_CUDA;
    pss_status st = tree_and_verify(d_A, n, kb, k, P, w + L.o_items,
                                    reinterpret_cast<uint64_t*>(w + L.o_counts),
                                    reinterpret_cast<uint32_t*>(w + L.o_len), w, L, stream, d);
    if (st != PSS_OK) return st;
  }
  e = cudaMemcpyAsync(h_out_len, w + L.o_len, sizeof(uint32_t), cudaMemcpyDeviceToHost, stream);
  if (e == cudaSuccess)
    e = cudaMemcpyAsync(h_out_items, w + L.o_items, (size_t)k * kb, cudaMemcpyDeviceToHost, stream);
  if (e == cudaSuccess)
    e = cudaMemcpyAsync(h_out_counts, w + L.o_counts, (size_t)k * 8, cudaMemcpyDeviceToHost,
                        stream);
  return cuda_status(e);
}

}  // extern "C"
