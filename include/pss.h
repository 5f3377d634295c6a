/*
 * pss.h -- C-ABI of libpss.so: the data-parallel hot path of Parallel Space Saving
 * (Cafaro, Pulimeno, Epicoco, Aloisio, "Parallel Space Saving on Multi and Many-Core Processors",
 * arXiv 1606.04669) on one NVIDIA B200 (sm_100a).
 *
 * Citations "P:line" are lines of the paper's text; readings R1..R12 of points the paper
 * leaves open are listed in DESIGN.md section 3 and apply to every call below.
 *
 * Conventions shared by every call
 *  - Memory: every pointer named d_* and every pointer inside pss_summaries is DEVICE memory owned
 *    by the caller (e.g. torch tensors); h_* pointers are HOST memory (pinned recommended). The
 *    library never allocates or frees memory and keeps no global mutable state.
 *  - Asynchrony: every call enqueues work on `stream` and returns; outputs are valid after the
 *    stream is synchronised. Calls on distinct streams may run concurrently if their buffers and
 *    workspaces are disjoint.
 *  - Errors: arguments are validated before anything is launched; a failed validation returns a
 *    status != PSS_OK and launches nothing. A launch failure returns PSS_ERR_CUDA (the CUDA error is
 *    read with cudaGetLastError). No exception crosses the ABI.
 *  - Keys: uint32 or uint64 item ids (pss_key_type). Every value, including 0 and all-ones, is a
 *    valid id (R12). Counts and errors are uint32 (R9: n <= 2^31 so f_hat <= n + n/k < 2^32);
 *    exact counts are uint64.
 *  - Workspace: scratch device memory of at least pss_workspace_bytes(op, ...) bytes, 256-byte
 *    aligned, passed as d_ws/ws_bytes; its contents need not be initialised and are clobbered.
 */
#ifndef PSS_H_
#define PSS_H_

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#ifndef __CUDA_RUNTIME_API_H__
typedef struct CUstream_st* cudaStream_t;
#endif

typedef enum {
  PSS_OK = 0,
  PSS_ERR_INVALID_ARG = 1,         /* null pointer, k < 2, P == 0, bad key type, ... */
  PSS_ERR_UNSUPPORTED = 2,         /* n > 2^31 (u32 counters, R9), k > PSS_MAX_K */
  PSS_ERR_CAPACITY_MISMATCH = 3,   /* summaries with different k or key type */
  PSS_ERR_WORKSPACE_TOO_SMALL = 4, /* ws_bytes < pss_workspace_bytes(...) */
  PSS_ERR_CUDA = 5                 /* a CUDA launch or runtime call failed */
} pss_status;

typedef enum { PSS_KEY_U32 = 0, PSS_KEY_U64 = 1 } pss_key_type;

/* ops for pss_workspace_bytes */
typedef enum {
  PSS_OP_SUMMARIZE = 0,
  PSS_OP_MERGE = 1,
  PSS_OP_COMBINE = 2,
  PSS_OP_VERIFY = 3,
  PSS_OP_QUERY = 4,
  PSS_OP_EXACT = 5, /* pss_exact_kmajority; P is ignored */
  PSS_OP_SUMMARIZE_MERGE = 6,
  PSS_OP_COMBINE_WIDE = 7, /* pss_combine_wide; P = count */
  PSS_OP_MERGE_WIDE = 8    /* pss_merge_wide; P = count; n is ignored */
} pss_op;

#define PSS_MAX_K 65000u
#define PSS_MAX_N (1ull << 31)

/*
 * A batch of `count` stream summaries of capacity k, structure of arrays, in device memory.
 * Summary i occupies entries [i*k, i*k + sizes[i]) of items/counts/errs; entries past sizes[i] are
 * unspecified. A counter is (item e, estimated frequency f_hat, error eps) (eps is reading
 * R3 -- the paper's summaries store (e, f_hat) only). Leaves are in slot order (R2); merged
 * summaries and roots are in canonical order: count descending, then item ascending (R5).
 */
typedef struct {
  int32_t key_type;  /* pss_key_type */
  uint32_t k;        /* counters per summary, 2 <= k <= PSS_MAX_K */
  uint32_t count;    /* number of summaries */
  void* items;       /* [count][k] uint32_t or uint64_t */
  uint32_t* counts;  /* [count][k] f_hat */
  uint32_t* errs;    /* [count][k] eps */
  uint32_t* sizes;   /* [count] occupied counters, <= k */
} pss_summaries;

/* Bytes of workspace an op needs. For PSS_OP_VERIFY, k is the candidate capacity (max n_cand);
 * for PSS_OP_MERGE, P is the number of leaves; n is ignored except by SUMMARIZE and QUERY. */
size_t pss_workspace_bytes(int op, uint64_t n, uint32_t k, uint32_t P, pss_key_type kt);

/*
 * pss_summarize -- the per-block local step of Algorithm 1: block decomposition
 * left = floor(r n / P), right = floor((r+1) n / P) - 1 for r = 0..P-1 (Alg. 1 l.3-4, P:92-95;
 * P:84), then SpaceSaving(A, left, right, k) on every block (Alg. 1 l.5; update
 * rules P:82 with R1: ties evict the lowest slot index; R2: free counters fill in slot order).
 *   d_A     : n keys of type kt, read-only, naturally aligned.
 *   n       : 0 <= n <= 2^31.
 *   k, P    : k >= 2 ("2 <= k"; k > n is allowed and gives exact summaries); P >= 1
 *             (P > n gives empty leaves, R10).
 *   leaves  : caller-owned, leaves->count == P, leaves->k == k, leaves->key_type == kt. Written:
 *             sizes[r] and entries [r*k, r*k + sizes[r]) in slot order.
 */
pss_status pss_summarize(const void* d_A, uint64_t n, pss_key_type kt, uint32_t k, uint32_t P,
                         pss_summaries* leaves, void* d_ws, size_t ws_bytes, cudaStream_t stream);

/*
 * pss_merge -- ParallelReduction(local, k, COMBINE) (Alg. 1 l.7) over a fixed balanced
 * binary tree (R6): level by level, nodes (2i, 2i+1) are combined with COMBINE (Alg. 2,
 * P:122-157) and an odd last node is carried up unchanged. COMBINE is commutative but not
 * associative, so the tree shape is part of the result.
 *   leaves : P = leaves->count >= 1 summaries (any order within a summary).
 *   root   : root->count == 1, same k and key type. Written in canonical order (R5).
 */
pss_status pss_merge(const pss_summaries* leaves, pss_summaries* root, void* d_ws,
                     size_t ws_bytes, cudaStream_t stream);

/*
 * pss_summarize_merge -- pss_summarize then pss_merge (Alg. 1 l.3-7) in one call, with
 * the same results bit for bit. The tree kernel is launched as a programmatic dependent of the
 * leaf kernel: its CTAs take the SMs the leaf kernel's persistent CTAs leave during its last wave
 * and combine leaves as soon as they are written (one ready flag per leaf, release/acquire), so
 * the merge overlaps the end of the summaries instead of following them.
 *   leaves : as for pss_summarize (count P; written, slot order).
 *   root   : as for pss_merge (count 1; canonical order).
 *   workspace : pss_workspace_bytes(PSS_OP_SUMMARIZE_MERGE, n, k, P, kt).
 */
pss_status pss_summarize_merge(const void* d_A, uint64_t n, pss_key_type kt, uint32_t k,
                               uint32_t P, pss_summaries* leaves, pss_summaries* root, void* d_ws,
                               size_t ws_bytes, cudaStream_t stream);

/*
 * pss_combine -- one COMBINE(S1, S2, k) (Alg. 2; prose P:112-115) for every i:
 * out[i] = COMBINE(a[i], b[i]). m1, m2 are the minima of S1, S2 (0 for a summary with fewer than
 * k occupied counters, R4); matched items get f1 + f2 (eps1 + eps2), items of S1 only f1 + m2
 * (eps1 + m2), items of S2 only f2 + m1 (eps2 + m1); Prune(k) keeps the k greatest (R5 ties).
 *   a, b, out : same k and key type; a->count == b->count == out->count.
 */
pss_status pss_combine(const pss_summaries* a, const pss_summaries* b, pss_summaries* out,
                       void* d_ws, size_t ws_bytes, cudaStream_t stream);

/*
 * pss_prune -- Pruned(global, n, k) (Alg. 1 l.8-9): keep the root counters with
 * f_hat >= floor(n/k) + 1 (the k-majority threshold; R7), in root order.
 *   root     : one summary in canonical order (as written by pss_merge).
 *   d_cand   : capacity root->k keys of the root's type; d_n_cand : one uint32.
 */
pss_status pss_prune(const pss_summaries* root, uint64_t n, void* d_cand, uint32_t* d_n_cand,
                     cudaStream_t stream);

/*
 * Wide summaries: the same counters with uint64 f_hat and eps, for the tree above the leaves when
 * the summarized stream may exceed 2^31 items -- the top levels over several ranks' subtree roots
 * (the paper's MPI reduction) and the on-line stream's upper tree (P:195
 * streams of 29 10^9 items; R14). Reading R9 bounds a u32 count by n + n/k < 2^32 only for
 * n <= 2^31; with 64-bit counters the bound is n <= 2^63. Layout and order as pss_summaries.
 */
typedef struct {
  int32_t key_type;  /* pss_key_type */
  uint32_t k;        /* counters per summary, 2 <= k <= PSS_MAX_K */
  uint32_t count;    /* number of summaries */
  void* items;       /* [count][k] uint32_t or uint64_t */
  uint64_t* counts;  /* [count][k] f_hat */
  uint64_t* errs;    /* [count][k] eps */
  uint32_t* sizes;   /* [count] occupied counters, <= k */
} pss_wsummaries;

/* pss_widen -- out[i] = in[i] with 64-bit counts and errors (same k, key type and count; same
 * order). No workspace. */
pss_status pss_widen(const pss_summaries* in, pss_wsummaries* out, cudaStream_t stream);

/* pss_combine_wide -- out[i] = COMBINE(a[i], b[i]) (Alg. 2; R3-R5) with 64-bit
 * arithmetic, canonical order. workspace: pss_workspace_bytes(PSS_OP_COMBINE_WIDE, 0, k, count,
 * kt). */
pss_status pss_combine_wide(const pss_wsummaries* a, const pss_wsummaries* b,
                            pss_wsummaries* out, void* d_ws, size_t ws_bytes,
                            cudaStream_t stream);

/* pss_merge_wide -- the fixed binary tree (R6, Alg. 1 l.7) over nodes->count wide summaries (e.g.
 * the ranks' subtree roots in rank order): the root in canonical order (a single summary is put in
 * canonical order). workspace: pss_workspace_bytes(PSS_OP_MERGE_WIDE, 0, k, count, kt). */
pss_status pss_merge_wide(const pss_wsummaries* nodes, pss_wsummaries* root, void* d_ws,
                          size_t ws_bytes, cudaStream_t stream);

/* pss_prune_wide -- pss_prune on a wide root: counters with f_hat >= floor(n/k) + 1 (R7),
 * root order, for any n < 2^63. */
pss_status pss_prune_wide(const pss_wsummaries* root, uint64_t n, void* d_cand,
                          uint32_t* d_n_cand, cudaStream_t stream);

/*
 * pss_verify -- the off-line verification scan ("a parallel scan of the input can be used to
 * determine the actual frequent items"): d_exact[j] = #{i < n : A[i] == cand[j]} (R8).
 *   d_cand   : n_cand keys (duplicates allowed).
 *   d_n_cand : optional (may be NULL) device uint32 holding the actual number of candidates; the
 *              kernels use min(*d_n_cand, n_cand), so the call can follow pss_prune without a host
 *              round trip. Entries of d_exact past that count are left untouched.
 *   d_exact  : n_cand uint64 outputs, candidate order.
 */
pss_status pss_verify(const void* d_A, uint64_t n, pss_key_type kt, const void* d_cand,
                      uint32_t n_cand, const uint32_t* d_n_cand, uint64_t* d_exact, void* d_ws,
                      size_t ws_bytes, cudaStream_t stream);

/*
 * pss_report -- the k-majority answer after verification: the candidates whose exact
 * count reaches floor(n/k) + 1, ordered by (exact count desc, item asc). The candidates must be
 * distinct (as written by pss_prune).
 *   d_cand, n_cand, d_n_cand : as for pss_verify; d_exact : their exact counts.
 *   d_out_items : capacity n_cand keys; d_out_counts : capacity n_cand uint64; d_out_len : uint32.
 */
pss_status pss_report(const void* d_cand, uint32_t n_cand, const uint32_t* d_n_cand,
                      const uint64_t* d_exact, pss_key_type kt, uint64_t n, uint32_t k,
                      void* d_out_items, uint64_t* d_out_counts, uint32_t* d_out_len,
                      cudaStream_t stream);

/*
 * pss_query -- the whole off-line pipeline: summarize, merge, prune, verify, then report the
 * k-majority set {(x, f(x)) : f(x) >= floor(n/k) + 1} ordered by (f desc, x asc).
 * Exact by the no-false-negative guarantee plus verification.
 *   d_out_items  : capacity k keys; d_out_counts : capacity k uint64; d_out_len : one uint32.
 */
pss_status pss_query(const void* d_A, uint64_t n, pss_key_type kt, uint32_t k, uint32_t P,
                     void* d_out_items, uint64_t* d_out_counts, uint32_t* d_out_len, void* d_ws,
                     size_t ws_bytes, cudaStream_t stream);

/*
 * pss_query_host -- pss_query from HOST buffers (the end-to-end call): copies h_A (n keys,
 * host, pinned recommended) to d_A (device, capacity n keys), runs pss_query, and copies the
 * result back to h_out_items (capacity k), h_out_counts (capacity k) and h_out_len (one uint32).
 * The d->h copies are enqueued on `stream`; the host buffers are valid after it is synchronised.
 * Inputs of 64 MiB or more are copied in 16 chunks cut at partition boundaries (Alg. 1 l.3-4) on
 * a private stream created and released inside the call; the leaves of each chunk are summarized
 * on `stream` as soon as the chunk has landed, so only the last chunk's leaves, the merge tree
 * and the verification pass follow the transfer. The copies start after the work already
 * enqueued on `stream`. Result identical to the unpipelined call.
 */
pss_status pss_query_host(const void* h_A, void* d_A, uint64_t n, pss_key_type kt, uint32_t k,
                          uint32_t P, void* h_out_items, uint64_t* h_out_counts,
                          uint32_t* h_out_len, void* d_ws, size_t ws_bytes, cudaStream_t stream);

/*
 * ---- On-line ingestion -------------------------------------
 * The stream is cut into consecutive leaves of leaf_len items (Alg. 1's blocks, with a
 * fixed length instead of floor(r n / P) bounds; the last leaf may be shorter), each summarized by
 * sequential Space Saving (R1, R2), and its summary at any point is the fixed balanced
 * binary COMBINE tree (R6; Alg. 2) over the leaves so far. When the number of items is
 * a multiple of leaf_len, that is bit for bit the root pss_summarize + pss_merge compute with
 * P = n / leaf_len. The tree is maintained incrementally (a binary counter of complete subtrees)
 * and nothing is re-read: this is the on-line setting of P:42, so candidates come from pss_prune
 * on the root (no verification pass; no false negatives).
 *
 * State: a pss_stream (host struct, caller-owned; written by pss_stream_init and every feed) plus
 * a device workspace of pss_stream_workspace_bytes(...) bytes that holds the subtree stack, the
 * partial leaf, a batch of leaf summaries and the host-feed buffers. A stream is used by one host
 * thread and one CUDA stream at a time. Counts: a leaf and a block of batch_leaves leaves hold at
 * most 2^31 items (u32 counters, R9); the subtree stack and the fold above the blocks keep 64-bit
 * counts (pss_wsummaries), so a stream may reach N = 2^63 items (P:195's streams of 29 10^9 items,
 * beyond one GPU's HBM when fed from the host); a feed past it returns PSS_ERR_UNSUPPORTED and
 * changes nothing.
 */
typedef struct {
  int32_t key_type;      /* pss_key_type */
  uint32_t k;            /* counters per summary */
  uint32_t leaf_len;     /* items per leaf, >= 1 */
  uint32_t batch_leaves; /* leaves summarized per K1 launch (workspace capacity), >= 1 */
  uint64_t n_seen;       /* items ingested so far */
  void* d_ws;            /* device workspace (caller-owned) */
  size_t ws_bytes;
} pss_stream;

/* Bytes of device workspace a stream needs (0 for invalid arguments). Dominated by
 * 2 * batch_leaves * leaf_len keys of host-feed buffers and batch_leaves leaf summaries. */
size_t pss_stream_workspace_bytes(pss_key_type kt, uint32_t k, uint32_t leaf_len,
                                  uint32_t batch_leaves);

/* Initialise *st as an empty stream (host only, launches nothing; the workspace need not be
 * cleared). INVALID_ARG for null pointers, k < 2, leaf_len == 0, batch_leaves == 0 or a bad key
 * type; UNSUPPORTED for k > PSS_MAX_K or batch_leaves * leaf_len > 2^31; WORKSPACE_TOO_SMALL. */
pss_status pss_stream_init(pss_stream* st, pss_key_type kt, uint32_t k, uint32_t leaf_len,
                           uint32_t batch_leaves, void* d_ws, size_t ws_bytes);

/* Append len keys from DEVICE memory (read-only; may be reused once the work enqueued on `stream`
 * is done). Any len, including 0 and pieces that split a leaf. Updates st->n_seen. */
pss_status pss_stream_feed(pss_stream* st, const void* d_chunk, uint64_t len, cudaStream_t stream);

/* Append len keys from HOST memory (pinned recommended): copied in pieces of batch_leaves *
 * leaf_len keys on a private copy stream into two alternating device buffers, each piece ingested
 * on `stream` as soon as it has landed (the copy of piece g + 1 overlaps the kernels of piece g).
 * h_chunk must stay valid and unmodified until `stream` is synchronised. */
pss_status pss_stream_feed_host(pss_stream* st, const void* h_chunk, uint64_t len,
                                cudaStream_t stream);

/* The summary of the stream so far (the R6 tree over its leaves, the partial leaf included), in
 * canonical order (R5) into root (count 1, same k and key type), with 64-bit counts. Does not
 * change the stream. */
pss_status pss_stream_root_wide(const pss_stream* st, pss_wsummaries* root, cudaStream_t stream);

/* The same root with u32 counts: only while N + floor(N/k) < 2^32 (N <= floor((2^32 - 1) k /
 * (k + 1)), R9), else PSS_ERR_UNSUPPORTED. */
pss_status pss_stream_root(const pss_stream* st, pss_summaries* root, cudaStream_t stream);

/*
 * ---- Accuracy ---------------------------------------------
 * pss_exact_kmajority -- the k-majority set {(x, f(x)) : f(x) >= floor(n/k) + 1}
 * computed WITHOUT Space Saving, as the truth for recall and precision: A is cut into
 * sub-blocks of 4096 keys; an item with f(x) > n/k has f_r(x) > L_r/k in some sub-block r, so the
 * locally heavy keys of every sub-block (exact per-sub-block histograms) form a candidate set that
 * a second pass counts exactly. Output ordered by (f desc, x asc), like pss_query.
 *   d_out_items : capacity k keys; d_out_counts : capacity k uint64; d_out_len : one uint32.
 *   d_overflow  : optional (may be NULL) uint32 set to 1 if the candidate set outgrew its table
 *                 (2^12..2^24 entries sized from n*k/4096; then the output is incomplete), else 0.
 *   workspace   : pss_workspace_bytes(PSS_OP_EXACT, n, k, 0, kt).
 */
pss_status pss_exact_kmajority(const void* d_A, uint64_t n, pss_key_type kt, uint32_t k,
                               void* d_out_items, uint64_t* d_out_counts, uint32_t* d_out_len,
                               uint32_t* d_overflow, void* d_ws, size_t ws_bytes,
                               cudaStream_t stream);

/* The paper's accuracy metrics of Algorithm 1's output (two ARE populations). */
typedef struct {
  uint64_t n_reported;      /* candidates reported by Algorithm 1 (pss_prune of the root) */
  uint64_t n_reported_true; /* of which true k-majority items (exact count >= floor(n/k) + 1) */
  uint64_t n_true;          /* true k-majority items (pss_exact_kmajority) */
  double precision;         /* n_reported_true / n_reported (1 if nothing is reported) */
  double recall;            /* n_reported_true / n_true (1 if there is no k-majority item) */
  double are_reported;      /* mean |f - f_hat| / f over the reported items (0 if none) */
  double are_true;          /* mean over the true k-majority items; an unreported one counts 1 */
} pss_accuracy_report;

/*
 * pss_accuracy -- writes *d_report (device memory) for the candidates of `root`:
 *   root     : the root summary (canonical order, as written by pss_merge / pss_stream_root); the
 *              reported items are its first *d_n_cand counters, their estimates f_hat its counts.
 *   n        : the stream length the root summarizes.
 *   d_n_cand : device uint32 written by pss_prune(root, n, ...).
 *   d_exact  : device uint64[*d_n_cand]: pss_verify of those candidates (exact f).
 *   d_n_true : device uint32, the length written by pss_exact_kmajority (or any exact count of
 *              the items with f >= floor(n/k) + 1).
 * ARE sums are fp64 in a fixed order (deterministic).
 */
pss_status pss_accuracy(const pss_summaries* root, uint64_t n, const uint32_t* d_n_cand,
                        const uint64_t* d_exact, const uint32_t* d_n_true,
                        pss_accuracy_report* d_report, cudaStream_t stream);

/*
 * ---- Hybrid decomposition ---------------------------------
 * The paper's hybrid MPI/OpenMP design as an alternative tree shape: Pp
 * processes take the blocks floor(p n / Pp) .. floor((p+1) n / Pp) - 1 (Alg. 1 l.3-4 at the
 * process level) and each splits its block again among T threads with the same formulas; leaf
 * r = p*T + t. Each process reduces its T leaves with the fixed binary tree (R6), then the Pp
 * process roots are reduced with the same tree. Pp = 1 or T = 1 is Algorithm 1 with T or Pp
 * blocks; with T a power of two and Pp*T dividing n it is bit for bit pss_summarize + pss_merge
 * with P = Pp*T. COMBINE is not associative, so other shapes give other (equally guaranteed)
 * roots.
 */
size_t pss_hybrid_workspace_bytes(uint64_t n, uint32_t k, uint32_t Pp, uint32_t T,
                                  pss_key_type kt);
/* leaves: count == Pp*T, slot order, leaf p*T + t = thread t of process p. */
pss_status pss_summarize_hybrid(const void* d_A, uint64_t n, pss_key_type kt, uint32_t k,
                                uint32_t Pp, uint32_t T, pss_summaries* leaves, void* d_ws,
                                size_t ws_bytes, cudaStream_t stream);
/* leaves->count must be a multiple of T (Pp = count / T); root canonical (R5). Workspace:
 * pss_hybrid_workspace_bytes(0, k, Pp, T, kt). Non-power-of-two T runs one tree launch per
 * process. */
pss_status pss_merge_hybrid(const pss_summaries* leaves, uint32_t T, pss_summaries* root,
                            void* d_ws, size_t ws_bytes, cudaStream_t stream);

/*
 * pss_read_probe -- K6, the read-bandwidth probe: reads the n keys of d_A
 * once with 128-bit loads and writes their bitwise fold to *d_out (one uint32, device). Its time
 * over the hot path's own input is the attainable HBM read bandwidth the path is compared with.
 *   d_A : 16-byte aligned (INVALID_ARG otherwise), read-only.
 */
pss_status pss_read_probe(const void* d_A, uint64_t n, pss_key_type kt, uint32_t* d_out,
                          cudaStream_t stream);

/*
 * pss_leaf_kernels -- which kernels pss_summarize (and every call that summarizes leaves) runs for
 * this shape, as bit flags: PSS_LEAF_K1 (the per-warp batched rule, csrc/summarize.cu),
 * PSS_LEAF_K1E (the per-CTA epoch formulation, csrc/epoch.cu; u32 keys, 64 <= k <= 2048),
 * PSS_LEAF_K1H (the histogram kernel in front, for blocks with at most k distinct keys; blocks it
 * gives up on go to K1E or K1). All of them produce the leaves of Alg. 1 l.5 bit for
 * bit; this query only reports the routing (tests and tools). 0 for an invalid shape. Host only.
 */
#define PSS_LEAF_K1 1
#define PSS_LEAF_K1E 2
#define PSS_LEAF_K1H 4
int pss_leaf_kernels(uint64_t n, uint32_t k, uint32_t P, pss_key_type kt);

/* Human-readable name of a status. */
const char* pss_status_string(pss_status s);

/* Library version, e.g. "pss-b200 0.1". */
const char* pss_version(void);

#ifdef __cplusplus
}
#endif
#endif /* PSS_H_ */
