"""GPU parity: the CUDA path (through the C-ABI) against the CPU oracle, element by element.

All arithmetic is integer, so the bar is bit-exact: leaves in slot order, merged summaries and
the root in canonical order, candidates in root order, exact counts, and the final answer.
Small cases and the full BASELINE sizes (in bench.py's launch configuration) compare every
output: every leaf, the root, candidates, exact counts and the answer (the last also against a
brute-force histogram).
"""
import numpy as np
import pytest
import torch

import inputs
import oracle

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def pss():
    if not torch.cuda.is_available():
        pytest.skip("needs a GPU")
    from conftest import build_lib
    build_lib()
    import paper_1606_04669_b200 as p
    return p


def to_dev(A):
    return torch.from_numpy(np.ascontiguousarray(A)).cuda()


def host_summary(S, i=0):
    return S.host(i)


def run_path(pss, A, k, P):
    dA = to_dev(A)
    leaves = pss.pss_summarize(dA, k, P)
    root = pss.pss_merge(leaves)
    cand, n_cand = pss.pss_prune(root, A.size)
    exact = pss.pss_verify(dA, cand, n_cand)
    items, counts, length = pss.pss_query(dA, k, P)
    # the fused call (the tree kernel overlapping the leaf kernel through per-leaf flags)
    f_leaves, f_root = pss.pss_summarize_merge(dA, k, P)
    # the same answer without Space Saving (f3's truth: local heavy hitters + exact counts)
    x_items, x_counts, x_len, x_over = pss.pss_exact_kmajority(dA, k)
    torch.cuda.synchronize()
    nc = int(n_cand.item())
    ln = int(length.item())
    xl = int(x_len.item())
    assert int(x_over.item()) == 0
    return dict(leaves=leaves, root=root, f_leaves=f_leaves, f_root=f_root,
                cand=cand[:nc].cpu().numpy().astype(np.uint64).tolist(),
                exact=exact[:nc].cpu().numpy().astype(np.uint64).tolist(),
                result=(items[:ln].cpu().numpy().astype(np.uint64).tolist(),
                        counts[:ln].cpu().numpy().astype(np.uint64).tolist()),
                exact_km=(x_items[:xl].cpu().numpy().astype(np.uint64).tolist(),
                          x_counts[:xl].cpu().numpy().astype(np.uint64).tolist()))


def assert_full_parity(pss, A, k, P, threads=8):
    got = run_path(pss, A, k, P)
    ref = oracle.pipeline(A, k, P, threads=threads)
    for r in range(P):
        assert got["leaves"].host(r) == ref.leaves[r].as_tuples(), f"leaf {r}"
    assert got["root"].host(0) == ref.root.as_tuples(), "root"
    assert got["f_root"].host(0) == ref.root.as_tuples(), "root (pss_summarize_merge)"
    assert torch.equal(got["f_leaves"].sizes, got["leaves"].sizes)
    assert got["cand"] == ref.cand.tolist()
    assert got["exact"] == ref.exact.tolist()
    assert got["result"][0] == ref.result[0].tolist()
    assert got["result"][1] == ref.result[1].tolist()
    assert got["exact_km"] == got["result"]  # == the oracle's answer, checked just above
    return got, ref


# ---------------------------------------------------------------- small cases, every output
def test_worked_example_E6(pss, golden):
    from conftest import letters
    case = golden["pipeline"][0]
    A = letters(case["stream"]).astype(np.uint32)
    got, _ = assert_full_parity(pss, A, case["k"], case["P"])
    assert got["root"].host(0) == [tuple(x) for x in case["root"]]
    assert got["result"][0] == case["result"]


def test_C1_full(pss):
    w = inputs.WORKLOADS["C1"]
    assert_full_parity(pss, w.generate(), w.k, w.P)


@pytest.mark.parametrize("n,k,P,s,U", [
    (1000, 2, 1, 1.1, 50), (1000, 3, 7, 0.8, 20), (4097, 5, 3, 1.3, 1000), (777, 31, 5, 1.1, 100),
    (5000, 33, 9, 1.1, 400), (12345, 64, 13, 1.05, 5000), (3, 10, 5, 1.1, 10),     # P > n
    (50, 100, 3, 1.1, 1000),                                                           # k > n
    (100_000, 8, 3, 1.5, 30), (65_536, 1000, 1, 1.1, 1e6), (200_000, 2, 16, 0.6, 1e5),
    (131_072, 257, 2, 1.1, 1e8), (0, 10, 4, 1.1, 10), (1, 2, 1, 1.1, 10)])
def test_random_small(pss, n, k, P, s, U):
    A = inputs.zipf(n, s, U, seed=n * 7 + k)
    assert_full_parity(pss, A, k, P)


@pytest.mark.parametrize("seed", range(12))
def test_tiny_universe_hazards(pss, seed):
    """Tiny universes and tiny k force fill->evict inside a 32-item window, exhausted minimum
    levels and victim-hit hazards in almost every window."""
    rng = np.random.default_rng(seed)
    n = int(rng.integers(1, 20000))
    U = int(rng.integers(2, 12))
    k = int(rng.integers(2, 9))
    P = int(rng.integers(1, 9))
    A = rng.integers(0, U, size=n).astype(np.uint32) * np.uint32(2654435761 & 0xFFFFFFFF)
    assert_full_parity(pss, A.astype(np.uint32), k, P)


def test_all_equal_and_all_distinct(pss):
    assert_full_parity(pss, np.full(70_000, 42, np.uint32), 10, 3)
    A = np.random.default_rng(1).permutation(np.arange(100_000, dtype=np.uint32)) * 7
    assert_full_parity(pss, A.astype(np.uint32), 50, 4)
    assert_full_parity(pss, A.astype(np.uint32), 1000, 2)


def test_extreme_keys(pss):
    """0 and all-ones are ordinary ids (R12): nothing may use a key as a sentinel."""
    rng = np.random.default_rng(5)
    A = rng.choice(np.array([0, 0xFFFFFFFF, 0xFFFFFFFE, 1, 7], np.uint32), size=30_000,
                   p=[0.3, 0.3, 0.2, 0.1, 0.1])
    assert_full_parity(pss, A, 3, 5)
    B = rng.choice(np.array([0, 2**64 - 1, 2**64 - 2, 1 << 63, 5], np.uint64), size=30_000)
    assert_full_parity(pss, B, 2, 3)


@pytest.mark.parametrize("n,k,P", [(300_000, 100, 7), (1 << 20, 2000, 16), (100_001, 3, 5)])
def test_u64_keys_with_tail(pss, n, k, P):
    A = inputs.zipf(n, 1.8, float(1 << 40), seed=5, key_bytes=8, tail_frac=0.01)
    assert_full_parity(pss, A, k, P)


@pytest.mark.parametrize("k", [5000, 20000])
def test_large_k_global_state(pss, k):
    """Summaries too large for shared memory (C4's k >= 5000) take the global-memory path."""
    A = inputs.zipf(1 << 19, 1.5, float(1 << 32), seed=4)
    assert_full_parity(pss, A, k, 8)


def test_several_tiles_and_ragged_tail(pss):
    """n = 2^22 + 12345 with 65 536-item-ish blocks, k = 1000, Zipf(1.1): many TMA stages per
    block, unaligned block starts, and a ragged array end."""
    A = inputs.zipf((1 << 22) + 12345, 1.1, 1e8, seed=2)
    assert_full_parity(pss, A, 1000, 64, threads=16)


def test_unaligned_device_pointer(pss):
    A = inputs.zipf(100_003, 1.1, 1e5, seed=11)
    big = torch.from_numpy(np.concatenate([np.zeros(1, np.uint32), A])).cuda()
    dA = big[1:]  # 4-byte aligned, not 16-byte aligned
    k, P = 50, 6
    leaves = pss.pss_summarize(dA, k, P)
    root = pss.pss_merge(leaves)
    cand, n_cand = pss.pss_prune(root, A.size)
    exact = pss.pss_verify(dA, cand, n_cand)
    torch.cuda.synchronize()
    ref = oracle.pipeline(A, k, P)
    for r in range(P):
        assert leaves.host(r) == ref.leaves[r].as_tuples()
    assert root.host(0) == ref.root.as_tuples()
    nc = int(n_cand.item())
    assert exact[:nc].cpu().numpy().tolist() == ref.exact.tolist()


# ---------------------------------------------------------------- COMBINE and verify directly
def random_summary(rng, k, full, key_bytes=4, pool=None):
    size = k if full else int(rng.integers(0, k))
    pool = pool if pool is not None else rng.integers(0, 1 << 31, size=4 * k + 8)
    items = rng.choice(pool, size=size, replace=False).astype(np.uint64)
    counts = rng.integers(1, 50, size=size).astype(np.uint64)
    errs = np.minimum(counts - 1, rng.integers(0, 10, size=size)).astype(np.uint64)
    return oracle.Summary(items, counts, errs)


@pytest.mark.parametrize("k", [2, 3, 17, 100, 1000])
def test_combine_direct(pss, k):
    rng = np.random.default_rng(k)
    count = 24
    pool = rng.integers(0, 1 << 31, size=3 * k + 4)  # overlapping item sets
    pairs = [(random_summary(rng, k, i % 3 != 0, pool=pool), random_summary(rng, k, i % 4 != 0, pool=pool))
             for i in range(count)]
    def pack(ss):
        S = pss.Summaries.empty(count, k, pss.KEY_U32)
        it = np.zeros((count, k), np.uint32)
        c = np.zeros((count, k), np.uint32)
        e = np.zeros((count, k), np.uint32)
        sz = np.zeros(count, np.uint32)
        for i, s in enumerate(ss):
            it[i, :len(s)], c[i, :len(s)], e[i, :len(s)] = s.items, s.counts, s.errs
            sz[i] = len(s)
        S.items.copy_(torch.from_numpy(it)); S.counts.copy_(torch.from_numpy(c))
        S.errs.copy_(torch.from_numpy(e)); S.sizes.copy_(torch.from_numpy(sz))
        return S
    a, b = pack([p[0] for p in pairs]), pack([p[1] for p in pairs])
    out = pss.pss_combine(a, b)
    torch.cuda.synchronize()
    for i, (s1, s2) in enumerate(pairs):
        assert out.host(i) == oracle.combine(s1, s2, k).as_tuples(), i


def test_verify_duplicates_absent_and_device_count(pss):
    A = inputs.zipf(500_000, 1.2, 1e4, seed=3)
    cand = np.array([inputs.mix32(0), 12345, inputs.mix32(0), inputs.mix32(5), 0, 0xFFFFFFFF],
                    np.uint32)
    dA = to_dev(A)
    ex = pss.pss_verify(dA, to_dev(cand))
    ex2 = pss.pss_verify(dA, to_dev(cand), torch.tensor([3], dtype=torch.uint32).cuda())
    torch.cuda.synchronize()
    want = oracle.verify(A, cand).tolist()
    assert ex.cpu().numpy().tolist() == want
    assert ex2[:3].cpu().numpy().tolist() == want[:3]
    many = np.unique(A)[:3000]  # a candidate list too large for the shared-memory table
    ex3 = pss.pss_verify(dA, to_dev(many))
    torch.cuda.synchronize()
    assert ex3.cpu().numpy().tolist() == oracle.verify(A, many).tolist()
    # the three counting modes: per-lane counters, per-warp grouped counters, global atomics
    for nc in (1, 80, 81, 127, 128, 129, 500, 2048, 2049):
        c = np.unique(A)[:nc]
        ex4 = pss.pss_verify(dA, to_dev(c))
        torch.cuda.synchronize()
        assert ex4.cpu().numpy().tolist() == oracle.verify(A, c).tolist(), nc


@pytest.mark.parametrize("kb", [4, 8])
def test_verify_keys_equal_to_table_fillers(pss, kb):
    """Empty table entries hold a filler key (all-ones for u32 tables, 0 for u64) with no
    candidate index: stream items equal to the filler that are not candidates count nowhere."""
    rng = np.random.default_rng(kb)
    dt = np.uint32 if kb == 4 else np.uint64
    filler = dt(0xFFFFFFFF) if kb == 4 else dt(0)
    A = rng.integers(1, 50, size=300_007).astype(dt)
    A[rng.random(A.size) < 0.3] = filler
    for cand in (np.array([3, 7, 11], dt), np.arange(1, 100, dtype=dt), np.arange(1, 300, dtype=dt)):
        ex = pss.pss_verify(to_dev(A), to_dev(cand))
        torch.cuda.synchronize()
        assert ex.cpu().numpy().tolist() == oracle.verify(A, cand).tolist(), cand.size


def test_query_host_end_to_end(pss):
    A = inputs.zipf(1 << 20, 1.1, 1e6, seed=9)
    k, P = 200, 16
    items, counts = pss.pss_query_host(torch.from_numpy(A).pin_memory(), k, P)
    ref = oracle.pipeline(A, k, P, threads=8)
    assert items.numpy().astype(np.uint64).tolist() == ref.result[0].tolist()
    assert counts.numpy().tolist() == ref.result[1].tolist()


@pytest.mark.parametrize("chunks,kb,k,P", [(3, 4, 200, 16), (16, 4, 100, 37), (7, 8, 64, 29),
                                           (5, 4, 4500, 11), (64, 4, 50, 64)])
def test_query_host_pipelined_copy(pss, monkeypatch, chunks, kb, k, P):
    """pss_query_host cut into copy chunks at partition boundaries (each chunk's leaves are
    summarized while later chunks are in flight): same answer as the oracle, ragged n and P."""
    monkeypatch.setenv("PSS_DEBUG_H2D_CHUNKS", str(chunks))
    A = inputs.zipf((1 << 19) + 12345, 1.2, 1e6, seed=31 + chunks, key_bytes=kb)
    items, counts = pss.pss_query_host(torch.from_numpy(A).pin_memory(), k, P)
    ref = oracle.pipeline(A, k, P, threads=8)
    assert items.numpy().astype(np.uint64).tolist() == ref.result[0].tolist()
    assert counts.numpy().tolist() == ref.result[1].tolist()


# ---------------------------------------------------------------- full BASELINE sizes
def bruteforce_kmajority(A, k):
    u, c = np.unique(A, return_counts=True)
    sel = c * k > A.size
    order = np.lexsort((u[sel], -c[sel].astype(np.int64)))
    return u[sel][order].astype(np.uint64).tolist(), c[sel][order].astype(np.uint64).tolist()


FULL = ["C1", "C2", "H", "C3-s0.5", "C3-s1.0", "C3-s1.5", "C3-s2.0", "C3-s3.0", "C4-k200",
        "C4-k1000", "C4-k5000", "C4-k20000", "C5"]


def padded_host(S):
    """Device summaries -> numpy (sizes, items, counts, errs) with zeros beyond each size."""
    sz = S.sizes.cpu().numpy().astype(np.int64)
    mask = np.arange(S.k)[None, :] < sz[:, None]
    out = [sz]
    for t in (S.items, S.counts, S.errs):
        out.append(np.where(mask, t.cpu().numpy().astype(np.uint64), np.uint64(0)))
    return out


@pytest.mark.parametrize("name", FULL)
def test_full_size(pss, name):
    """BASELINE.json configs at full size, bench.py's launch configuration (k, P): EVERY leaf
    (slot order) and the root (canonical order) bit-exact against the oracle (Space Saving per
    block; the fixed COMBINE tree), both from
    the separate calls and from the fused pss_summarize_merge; candidates, exact counts and the
    answer exact; the answer equals the brute-force k-majority set (recall 1)."""
    w = inputs.WORKLOADS[name]
    need = w.n * w.key_bytes * 4 + w.P * w.k * 8 * 6
    try:
        import psutil
        if psutil.virtual_memory().available < need + (8 << 30):
            pytest.skip(f"{name} needs ~{need >> 30} GiB of host memory")
    except ImportError:
        pass
    A = w.generate()
    n, k, P = A.size, w.k, w.P
    got = run_path(pss, A, k, P)
    th = inputs.host_threads()
    it, c, e, sz = oracle.leaves_padded(A, k, P, threads=th)
    for which in ("leaves", "f_leaves"):
        gsz, git, gc, ge = padded_host(got[which])
        bad = np.flatnonzero((gsz != sz) | (git != it).any(1) | (gc != c).any(1) | (ge != e).any(1))
        assert bad.size == 0, f"{name}: {bad.size} of {P} leaves differ ({which}), first {bad[:5]}"
    root = oracle.tree_padded(it, c, e, sz, k, threads=th)
    del it, c, e
    assert got["root"].host(0) == root.as_tuples(), f"{name} root"
    assert got["f_root"].host(0) == root.as_tuples(), f"{name} root (pss_summarize_merge)"
    thr = oracle.threshold(n, k)
    assert got["cand"] == oracle.prune(root, n, k).tolist()
    assert got["cand"] == [int(x) for x, cc in zip(root.items, root.counts) if cc >= thr]
    assert got["exact"] == oracle.verify(A, np.array(got["cand"], np.uint64)).tolist()
    want = bruteforce_kmajority(A, k)
    assert got["result"] == want
    assert got["exact_km"] == want
    assert set(want[0]) <= set(root.items.tolist())  # recall 1


@pytest.mark.parametrize("load", [0.75, 0.85])
def test_crowded_index_kick_and_rehash_paths(pss, load, monkeypatch):
    """Force the summary index to 75-85% occupancy (test hook PSS_DEBUG_INDEX_LOAD) so that
    inserts collide, take the serial cuckoo-kick path and sometimes rebuild the index."""
    monkeypatch.setenv("PSS_DEBUG_INDEX_LOAD", str(load))
    for n, k, P, s, U in [(300_000, 100, 5, 1.1, 1e6), (200_000, 37, 3, 0.8, 5e4),
                          (100_000, 1000, 2, 1.1, 1e8)]:
        A = inputs.zipf(n, s, U, seed=n + k)
        assert_full_parity(pss, A, k, P)


def test_read_probe(pss):
    """K6 reads every byte of A: its fold is the XOR of A's 32-bit words (ragged 16-byte tails)."""
    for n, kb in [(0, 4), (1, 4), (7, 4), (1 << 20, 4), (12345, 8), (3, 8)]:
        A = np.random.default_rng(n).integers(0, 2**32, size=n * kb // 4, dtype=np.uint64)
        words = A.astype(np.uint32)
        keys = words if kb == 4 else words.view(np.uint64)
        got = int(pss.pss_read_probe(torch.from_numpy(keys).cuda()).item())
        want = int(np.bitwise_xor.reduce(words)) if words.size else 0
        assert got == want, (n, kb)


def test_summarize_merge_repeatable(pss):
    """The overlapped call releases leaves to the tree kernel through flags cleared before every
    launch: back-to-back calls on one stream (no host sync) give the same leaves and root."""
    for n, k, P in [(1 << 20, 100, 64), (300_000, 1000, 17), (2_000_000, 50, 256)]:
        A = torch.from_numpy(inputs.zipf(n, 1.1, 1e6, seed=n + P)).cuda()
        ref_l, ref_r = pss.pss_summarize_merge(A, k, P)
        ref = (ref_r.host(0), ref_l.sizes.clone(), ref_l.counts.clone())
        outs = [pss.pss_summarize_merge(A, k, P) for _ in range(8)]
        torch.cuda.synchronize()
        for l2, r2 in outs:
            assert r2.host(0) == ref[0]
            assert torch.equal(l2.sizes, ref[1]) and torch.equal(l2.counts, ref[2])
        assert ref[0] == pss.pss_merge(pss.pss_summarize(A, k, P)).host(0)


@pytest.mark.parametrize("n,k,P,s,U,kb", [
    (3 * 65536, 600, 3, 1.1, 1e5, 4), (2 * 65536 + 17, 1023, 2, 0.9, 5e4, 4),
    (65536, 1024, 1, 1.3, 3e4, 4), (4 * 65536, 2047, 4, 1.1, 1e6, 4),
    (2 * 65536, 1500, 2, 1.1, 2e4, 8), (131_071 * 2, 700, 2, 1.0, 1e4, 8)])
def test_specialized_layout_shapes(pss, n, k, P, s, U, kb):
    """Blocks of 2^16 .. 2^17 - 1 keys with k in [512, 1023] run K1 compiled with its layout
    constants (slot bits 10, count bits 17): every output against the oracle, both key types, at
    the edges of the range and just outside it (k = 1024, 1500, 2047: the runtime-layout kernel)."""
    A = inputs.zipf(n, s, U, seed=n + k, key_bytes=kb)
    assert_full_parity(pss, A, k, P)


@pytest.mark.parametrize("load", [0.8])
def test_specialized_layout_crowded_index(pss, load, monkeypatch):
    """The kick and rehash paths of the specialized K1 (crowded index, PSS_DEBUG_INDEX_LOAD)."""
    monkeypatch.setenv("PSS_DEBUG_INDEX_LOAD", str(load))
    A = inputs.zipf(2 * 65536, 0.9, 2e4, seed=31)
    assert_full_parity(pss, A, 900, 2)
