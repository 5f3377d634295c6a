// stream.cu -- on-line ingestion: the
// stream is cut into consecutive leaves of `leaf_len` items (the last one possibly shorter) and
// its summary at any point is the fixed binary COMBINE tree (reading R6) over the
// leaves so far. Nothing is re-read: this is the on-line setting of PAPER.md:42 (no verification
// pass; candidates come from pss_prune on the root).
//
// The tree is built incrementally as a binary counter. With c complete leaves, stack level j holds
// the root of the complete subtree over leaves [p, p + 2^j) for every set bit j of c (p = the
// higher set bits of c) -- exactly a node of the R6 tree. A feed summarizes its whole leaves with
// K1 in batches, cuts each batch into maximal aligned power-of-two blocks, reduces every block
// with the tree kernel (the R6 tree of 2^j leaves is the complete tree), and pushes the block
// root with carries: a pushed node at level j whose sibling is on the stack is combined with it
// (COMBINE, Alg. 2) into level j + 1. The summary of the stream is the right fold
// COMBINE(S_1, COMBINE(S_2, ... COMBINE(S_t, partial))) over the stack from the highest level
// down, then the summary of the partial leaf: this is the R6 tree over all the leaves (R6's root
// splits off its largest complete left subtree, recursively).
//
// Counts: a block holds at most batch_leaves * leaf_len <= 2^31 items, so leaves and block roots
// keep u32 counts (R9); the stack and the fold above the blocks use 64-bit counts (wide.cu), so a
// stream may reach 2^63 items -- beyond one GPU's HBM when fed from the host (P:195's 29 10^9).
//
// Host code only: the kernels are K1 (summarize.cu, hist.cu), K2 (merge.cu) and wide.cu.
#include <algorithm>

#include "common.cuh"

namespace pss {

namespace {

struct StreamLayout {
  size_t stk_items, stk_counts, stk_errs, stk_sizes;  // STACK_LEVELS wide summaries
  size_t wt_items, wt_counts, wt_errs, wt_sizes;      // 4 wide: block root, fold ping-pong, leaf
  size_t nt_items, nt_counts, nt_errs, nt_sizes;      // 1 narrow: a block's root from the tree
  size_t b_items, b_counts, b_errs, b_sizes;          // batch_leaves leaf summaries
  size_t staging;                                     // leaf_len keys: the partial leaf
  size_t hostbuf;                                     // 2 x batch_leaves * leaf_len keys (feed_host)
  size_t flags;                                       // batch_leaves ready flags (K1 -> tree)
  size_t sumscratch, scratch, wscratch, total;        // K1's, the tree's, the wide COMBINE's
};
constexpr uint32_t STACK_LEVELS = 64;

StreamLayout stream_layout(int kb, uint32_t k, uint32_t leaf_len, uint32_t batch,
                           const DevInfo& d) {
  StreamLayout L;
  Bump b;
  L.stk_items = b.take<unsigned char>((size_t)STACK_LEVELS * k * kb);
  L.stk_counts = b.take<uint64_t>((size_t)STACK_LEVELS * k);
  L.stk_errs = b.take<uint64_t>((size_t)STACK_LEVELS * k);
  L.stk_sizes = b.take<uint32_t>(STACK_LEVELS);
  L.wt_items = b.take<unsigned char>((size_t)4 * k * kb);
  L.wt_counts = b.take<uint64_t>((size_t)4 * k);
  L.wt_errs = b.take<uint64_t>((size_t)4 * k);
  L.wt_sizes = b.take<uint32_t>(4);
  L.nt_items = b.take<unsigned char>((size_t)k * kb);
  L.nt_counts = b.take<uint32_t>(k);
  L.nt_errs = b.take<uint32_t>(k);
  L.nt_sizes = b.take<uint32_t>(1);
  L.b_items = b.take<unsigned char>((size_t)batch * k * kb);
  L.b_counts = b.take<uint32_t>((size_t)batch * k);
  L.b_errs = b.take<uint32_t>((size_t)batch * k);
  L.b_sizes = b.take<uint32_t>(batch);
  L.staging = b.take<unsigned char>((size_t)leaf_len * kb);
  L.hostbuf = b.take<unsigned char>((size_t)2 * batch * leaf_len * kb);
  L.flags = b.take<uint32_t>(batch);
  const uint64_t nb = (uint64_t)batch * leaf_len;
  L.sumscratch = b.take<unsigned char>(
      std::max(summarize_ws(nb, kb, k, batch, d), summarize_ws(leaf_len, kb, k, 1, d)));
  L.scratch = b.take<unsigned char>(merge_ws(kb, k, batch, d));
  L.wscratch = b.take<unsigned char>(
      std::max(wide_combine_ws(kb, k, d), wide_merge_ws(kb, k, 1, d)));
  L.total = b.bytes();
  return L;
}

// a view of one summary inside a workspace region (narrow: u32 counts, wide: u64 counts)
struct One {
  void* items;
  uint32_t* counts;
  uint32_t* errs;
  uint32_t* sizes;
};
struct WOne {
  void* items;
  uint64_t* counts;
  uint64_t* errs;
  uint32_t* sizes;
};

struct StreamCtx {
  int kb;
  uint32_t k, leaf_len, batch;
  unsigned char* w;
  StreamLayout L;
  DevInfo d;

  One region(size_t oi, size_t oc, size_t oe, size_t os, uint32_t i) const {
    return One{w + oi + (size_t)i * k * kb, reinterpret_cast<uint32_t*>(w + oc) + (size_t)i * k,
               reinterpret_cast<uint32_t*>(w + oe) + (size_t)i * k,
               reinterpret_cast<uint32_t*>(w + os) + i};
  }
  WOne wregion(size_t oi, size_t oc, size_t oe, size_t os, uint32_t i) const {
    return WOne{w + oi + (size_t)i * k * kb, reinterpret_cast<uint64_t*>(w + oc) + (size_t)i * k,
                reinterpret_cast<uint64_t*>(w + oe) + (size_t)i * k,
                reinterpret_cast<uint32_t*>(w + os) + i};
  }
  WOne stack(uint32_t j) const {
    return wregion(L.stk_items, L.stk_counts, L.stk_errs, L.stk_sizes, j);
  }
  WOne wtmp(uint32_t i) const { return wregion(L.wt_items, L.wt_counts, L.wt_errs, L.wt_sizes, i); }
  One ntmp() const { return region(L.nt_items, L.nt_counts, L.nt_errs, L.nt_sizes, 0); }
  One leaf(uint32_t i) const { return region(L.b_items, L.b_counts, L.b_errs, L.b_sizes, i); }
  void* scratch() const { return w + L.scratch; }

  // the R6 root of `cnt` consecutive leaf summaries starting at `first` (narrow: a block holds at
  // most batch_leaves * leaf_len <= 2^31 items); with leaf_flags, a tree kernel overlapping the
  // K1 launch that produces the leaves
  cudaError_t tree(const One& first, uint32_t cnt, const One& out, cudaStream_t s,
                   const uint32_t* leaf_flags = nullptr) const {
    return merge_tree_launch(kb, k, cnt, first.items, first.counts, first.errs, first.sizes,
                             out.items, out.counts, out.errs, out.sizes, scratch(), s, d,
                             leaf_flags);
  }
  cudaError_t widen(const One& in, const WOne& out, cudaStream_t s) const {
    return widen_launch(kb, k, 1, in.items, in.counts, in.errs, in.sizes, out.items, out.counts,
                        out.errs, out.sizes, s);
  }
  // above the blocks the stream may exceed 2^31 items: COMBINE with 64-bit counts (wide.cu)
  cudaError_t combine(const WOne& a, const WOne& b, const WOne& out, cudaStream_t s) const {
    return wide_combine_launch(kb, k, 1, a.items, a.counts, a.errs, a.sizes, b.items, b.counts,
                               b.errs, b.sizes, out.items, out.counts, out.errs, out.sizes,
                               w + L.wscratch, s, d);
  }
  cudaError_t canonical(const WOne& in, const WOne& out, cudaStream_t s) const {
    return wide_merge_launch(kb, k, 1, in.items, in.counts, in.errs, in.sizes, out.items,
                             out.counts, out.errs, out.sizes, w + L.wscratch, s, d);
  }
  cudaError_t summarize(const void* A, uint64_t n, uint32_t P, const One& out, cudaStream_t s,
                        uint32_t* leaf_flags = nullptr) const {
    return summarize_launch(A, n, kb, k, P, out.items, out.counts, out.errs, out.sizes,
                            w + L.sumscratch, s, d, 0, 0xffffffffu, 0, 1, leaf_flags,
                            leaf_flags != nullptr);
  }

  // push the root of the aligned block [p, p + 2^j) of complete leaves, whose 2^j leaf summaries
  // start at `first`; c = p is the number of complete leaves before the block
  cudaError_t push_block(uint64_t p, uint32_t j, const One& first, cudaStream_t s,
                         const uint32_t* leaf_flags = nullptr) const {
    uint32_t top = j;  // carries run while the sibling (bit `top` of p) is on the stack
    while (top < STACK_LEVELS && ((p >> top) & 1u)) ++top;
    if (top >= STACK_LEVELS) return cudaErrorInvalidValue;
    cudaError_t e = tree(first, 1u << j, ntmp(), s, leaf_flags);
    if (e != cudaSuccess) return e;
    if (top == j) return widen(ntmp(), stack(j), s);
    e = widen(ntmp(), wtmp(0), s);
    uint32_t cur = 0;
    for (uint32_t t = j; t < top && e == cudaSuccess; ++t) {
      const WOne out = (t + 1 == top) ? stack(top) : wtmp(cur == 1 ? 2 : 1);
      e = combine(stack(t), wtmp(cur), out, s);
      cur = cur == 1 ? 2 : 1;
    }
    return e;
  }

  // largest aligned power-of-two block of leaves starting at leaf p that fits in `room`
  static uint32_t block_log(uint64_t p, uint32_t room) {
    uint32_t j = 0;
    while (j < 31 && ((p >> j) & 1u) == 0 && (2u << j) <= room) ++j;
    return j;
  }

  // summarize and push `nl` complete leaves read from A (nl <= batch), the first being leaf c.
  // The first block's tree overlaps K1 (pss_summarize_merge's scheme) when it runs persistently.
  cudaError_t push_leaves(const void* A, uint64_t c, uint32_t nl, cudaStream_t s) const {
    if (!nl) return cudaSuccess;
    const uint32_t j0 = block_log(c, nl);
    uint32_t* flags = reinterpret_cast<uint32_t*>(w + L.flags);
    const bool ovl = merge_tree_overlaps(kb, k, 1u << j0, d);
    cudaError_t e = cudaSuccess;
    if (ovl) {
      e = cudaMemsetAsync(flags, 0, (size_t)nl * sizeof(uint32_t), s);
      if (e == cudaSuccess) e = merge_tree_reset(kb, k, 1u << j0, scratch(), s, d);
    }
    if (e == cudaSuccess)
      e = summarize(A, (uint64_t)nl * leaf_len, nl, leaf(0), s, ovl ? flags : nullptr);
    uint32_t i = 0;
    while (i < nl && e == cudaSuccess) {
      const uint32_t j = i == 0 ? j0 : block_log(c + i, nl - i);
      e = push_block(c + i, j, leaf(i), s, i == 0 && ovl ? flags : nullptr);
      i += 1u << j;
    }
    return e;
  }

  // the summary of the stream so far (R6 tree over its leaves) into the wide summary `out`
  cudaError_t root(uint64_t n_seen, const WOne& out, cudaStream_t s) const {
    const uint64_t complete = n_seen / leaf_len, have = n_seen % leaf_len;
    // the fold's operands from the right: the partial leaf, then stack levels upwards
    WOne ops[STACK_LEVELS + 1];
    uint32_t nops = 0;
    cudaError_t e = cudaSuccess;
    if (have) {
      e = summarize(w + L.staging, have, 1, leaf(0), s);
      if (e == cudaSuccess) e = widen(leaf(0), wtmp(3), s);
      ops[nops++] = wtmp(3);
    }
    for (uint32_t j = 0; j < STACK_LEVELS; ++j)
      if ((complete >> j) & 1u) ops[nops++] = stack(j);
    if (e != cudaSuccess) return e;
    if (nops == 0) return cudaMemsetAsync(out.sizes, 0, sizeof(uint32_t), s);
    if (nops == 1) return canonical(ops[0], out, s);
    // acc = ops[0]; acc = COMBINE(ops[i], acc) for i = 1..nops-1, the last one into `out`
    WOne acc = ops[0];
    uint32_t cur = 1;
    for (uint32_t i = 1; i < nops && e == cudaSuccess; ++i) {
      const WOne dst = (i + 1 == nops) ? out : wtmp(cur);
      e = combine(ops[i], acc, dst, s);
      acc = dst;
      cur = cur == 1 ? 2 : 1;
    }
    return e;
  }
};

bool ctx_of(const pss_stream* st, StreamCtx& c) {
  c.kb = st->key_type == PSS_KEY_U32 ? 4 : (st->key_type == PSS_KEY_U64 ? 8 : 0);
  if (!c.kb || st->k < 2 || st->k > PSS_MAX_K || st->leaf_len == 0 || st->batch_leaves == 0 ||
      !st->d_ws)
    return false;
  c.k = st->k;
  c.leaf_len = st->leaf_len;
  c.batch = st->batch_leaves;
  c.w = static_cast<unsigned char*>(st->d_ws);
  c.d = dev_info();
  c.L = stream_layout(c.kb, c.k, c.leaf_len, c.batch, c.d);
  return st->ws_bytes >= c.L.total;
}

// a narrow (u32) root needs f_hat <= N + floor(N/k) <= 2^32 - 1 (R9, invariant I of SURVEY.md
// 8(c)); the stream itself keeps 64-bit counts above its blocks and may grow to 2^63 items
uint64_t stream_narrow_max_n(uint32_t k) {
  const uint64_t lim = 0xffffffffull;
  return lim * k / (k + 1);
}
constexpr uint64_t STREAM_MAX_N = 1ull << 63;

// ingest len keys at d_chunk (device) into the stream described by c and st->n_seen
cudaError_t feed_device(const StreamCtx& c, pss_stream* st, const void* d_chunk, uint64_t len,
                        cudaStream_t s) {
  const unsigned char* A = static_cast<const unsigned char*>(d_chunk);
  const uint64_t LL = c.leaf_len;
  uint64_t n0 = st->n_seen;
  cudaError_t e = cudaSuccess;
  // 1. complete the partial leaf in the staging buffer
  const uint64_t have = n0 % LL;
  if (have && len) {
    const uint64_t t = std::min(len, LL - have);
    e = cudaMemcpyAsync(c.w + c.L.staging + have * c.kb, A, t * c.kb, cudaMemcpyDeviceToDevice, s);
    if (e == cudaSuccess && have + t == LL) e = c.push_leaves(c.w + c.L.staging, n0 / LL, 1, s);
    if (e != cudaSuccess) return e;
    A += t * c.kb;
    len -= t;
    n0 += t;
  }
  // 2. whole leaves straight from the chunk, in batches of the leaf buffer's capacity
  uint64_t whole = len / LL;
  while (whole && e == cudaSuccess) {
    const uint32_t nl = (uint32_t)std::min<uint64_t>(whole, c.batch);
    e = c.push_leaves(A, n0 / LL, nl, s);
    A += (uint64_t)nl * LL * c.kb;
    len -= (uint64_t)nl * LL;
    n0 += (uint64_t)nl * LL;
    whole -= nl;
  }
  // 3. the rest starts a new partial leaf
  if (len && e == cudaSuccess)
    e = cudaMemcpyAsync(c.w + c.L.staging, A, len * c.kb, cudaMemcpyDeviceToDevice, s);
  if (e == cudaSuccess) st->n_seen = n0 + len;
  return e;
}

}  // namespace
}  // namespace pss

using namespace pss;

extern "C" {

size_t pss_stream_workspace_bytes(pss_key_type kt, uint32_t k, uint32_t leaf_len,
                                  uint32_t batch_leaves) {
  const int kb = kt == PSS_KEY_U32 ? 4 : (kt == PSS_KEY_U64 ? 8 : 0);
  if (!kb || k < 2 || leaf_len == 0 || batch_leaves == 0) return 0;
  return stream_layout(kb, k, leaf_len, batch_leaves, dev_info()).total;
}

pss_status pss_stream_init(pss_stream* st, pss_key_type kt, uint32_t k, uint32_t leaf_len,
                           uint32_t batch_leaves, void* d_ws, size_t ws_bytes) {
  if (!st || !d_ws || k < 2 || leaf_len == 0 || batch_leaves == 0 ||
      (kt != PSS_KEY_U32 && kt != PSS_KEY_U64))
    return PSS_ERR_INVALID_ARG;
  if (k > PSS_MAX_K || leaf_len > PSS_MAX_N || (uint64_t)batch_leaves * leaf_len > PSS_MAX_N)
    return PSS_ERR_UNSUPPORTED;
  pss_stream s0;
  s0.key_type = kt;
  s0.k = k;
  s0.leaf_len = leaf_len;
  s0.batch_leaves = batch_leaves;
  s0.n_seen = 0;
  s0.d_ws = d_ws;
  s0.ws_bytes = ws_bytes;
  StreamCtx c;
  if (!ctx_of(&s0, c)) return PSS_ERR_WORKSPACE_TOO_SMALL;
  *st = s0;
  return PSS_OK;
}

pss_status pss_stream_feed(pss_stream* st, const void* d_chunk, uint64_t len,
                           cudaStream_t stream) {
  if (!st || (len && !d_chunk)) return PSS_ERR_INVALID_ARG;
  StreamCtx c;
  if (!ctx_of(st, c)) return PSS_ERR_INVALID_ARG;
  if (st->n_seen + len > STREAM_MAX_N || st->n_seen + len < st->n_seen)
    return PSS_ERR_UNSUPPORTED;
  return feed_device(c, st, d_chunk, len, stream) == cudaSuccess ? PSS_OK : PSS_ERR_CUDA;
}

pss_status pss_stream_feed_host(pss_stream* st, const void* h_chunk, uint64_t len,
                                cudaStream_t stream) {
  if (!st || (len && !h_chunk)) return PSS_ERR_INVALID_ARG;
  StreamCtx c;
  if (!ctx_of(st, c)) return PSS_ERR_INVALID_ARG;
  if (st->n_seen + len > STREAM_MAX_N || st->n_seen + len < st->n_seen)
    return PSS_ERR_UNSUPPORTED;
  if (!len) return PSS_OK;
  // pieces of one batch of leaves, copied on a private stream into two alternating device
  // buffers; piece g is ingested on `stream` as soon as it has landed, and buffer g % 2 is
  // refilled only after the ingestion of piece g - 2 is done with it
  const uint64_t piece = (uint64_t)c.batch * c.leaf_len;
  unsigned char* buf[2] = {c.w + c.L.hostbuf, c.w + c.L.hostbuf + piece * c.kb};
  cudaStream_t cs = nullptr;
  cudaEvent_t landed[2] = {}, used[2] = {};
  cudaError_t e = cudaStreamCreateWithFlags(&cs, cudaStreamNonBlocking);
  for (int i = 0; i < 2 && e == cudaSuccess; ++i) {
    e = cudaEventCreateWithFlags(&landed[i], cudaEventDisableTiming);
    if (e == cudaSuccess) e = cudaEventCreateWithFlags(&used[i], cudaEventDisableTiming);
    // the buffers are free once the work already enqueued on `stream` is done
    if (e == cudaSuccess) e = cudaEventRecord(used[i], stream);
  }
  const unsigned char* h = static_cast<const unsigned char*>(h_chunk);
  for (uint64_t off = 0, g = 0; off < len && e == cudaSuccess; off += piece, ++g) {
    const uint64_t m = std::min(piece, len - off);
    const int b = (int)(g & 1);
    e = cudaStreamWaitEvent(cs, used[b], 0);
    if (e == cudaSuccess)
      e = cudaMemcpyAsync(buf[b], h + off * c.kb, m * c.kb, cudaMemcpyHostToDevice, cs);
    if (e == cudaSuccess) e = cudaEventRecord(landed[b], cs);
    if (e == cudaSuccess) e = cudaStreamWaitEvent(stream, landed[b], 0);
    if (e == cudaSuccess) e = feed_device(c, st, buf[b], m, stream);
    if (e == cudaSuccess) e = cudaEventRecord(used[b], stream);
  }
  // the copy stream's last copy precedes work on `stream` (waited above); release is
  // stream-ordered
  for (int i = 0; i < 2; ++i) {
    if (landed[i]) cudaEventDestroy(landed[i]);
    if (used[i]) cudaEventDestroy(used[i]);
  }
  if (cs) cudaStreamDestroy(cs);
  return e == cudaSuccess ? PSS_OK : PSS_ERR_CUDA;
}

pss_status pss_stream_root_wide(const pss_stream* st, pss_wsummaries* root,
                                cudaStream_t stream) {
  if (!st || !root || !root->items || !root->counts || !root->errs || !root->sizes)
    return PSS_ERR_INVALID_ARG;
  StreamCtx c;
  if (!ctx_of(st, c)) return PSS_ERR_INVALID_ARG;
  if (root->k != st->k || root->key_type != st->key_type || root->count != 1)
    return PSS_ERR_CAPACITY_MISMATCH;
  const WOne out{root->items, root->counts, root->errs, root->sizes};
  return c.root(st->n_seen, out, stream) == cudaSuccess ? PSS_OK : PSS_ERR_CUDA;
}

pss_status pss_stream_root(const pss_stream* st, pss_summaries* root, cudaStream_t stream) {
  if (!st || !root || !root->items || !root->counts || !root->errs || !root->sizes)
    return PSS_ERR_INVALID_ARG;
  StreamCtx c;
  if (!ctx_of(st, c)) return PSS_ERR_INVALID_ARG;
  if (root->k != st->k || root->key_type != st->key_type || root->count != 1)
    return PSS_ERR_CAPACITY_MISMATCH;
  if (st->n_seen > stream_narrow_max_n(st->k)) return PSS_ERR_UNSUPPORTED;
  // the wide root, then its counts in 32 bits (they fit: N + floor(N/k) < 2^32)
  cudaError_t e = c.root(st->n_seen, c.wtmp(0), stream);
  const WOne r = c.wtmp(0);
  if (e == cudaSuccess)
    e = narrow_launch(c.kb, c.k, 1, r.items, r.counts, r.errs, r.sizes, root->items, root->counts,
                      root->errs, root->sizes, stream);
  return e == cudaSuccess ? PSS_OK : PSS_ERR_CUDA;
}

}  // extern "C"
