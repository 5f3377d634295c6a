"""GPU parity of the on-line stream (include/pss.h pss_stream_*): the root after
every feed equals the oracle's R6 tree over fixed-length leaves of the prefix fed so far, bit for
bit (all integer work). Chunks are ragged: empty, inside one leaf, completing a partial leaf,
spanning several batches of leaves, from device and from pinned host memory."""
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


def feed_and_check(pss, A, k, leaf_len, batch, cuts, host=False, check_every=True):
    kt = pss.KEY_U32 if A.dtype == np.uint32 else pss.KEY_U64
    st = pss.Stream(k, leaf_len, kt, batch_leaves=batch)
    tA = torch.from_numpy(A)
    dA = tA.cuda() if not host else None
    src = tA.pin_memory() if host else dA
    pos = 0
    for i, c in enumerate(list(cuts) + [A.size]):
        c = min(c, A.size)
        if c < pos:
            continue
        st.feed(src[pos:c])
        pos = c
        assert st.n_seen == pos
        if check_every or pos == A.size:
            got = st.root().host(0)
            want = oracle.stream_root(A[:pos], k, leaf_len).as_tuples()
            assert got == want, f"prefix {pos} (feed {i})"
    return st


def test_worked_examples(pss, golden):
    from conftest import letters
    for case in golden["stream"]:
        A = letters(case["stream"]).astype(np.uint32)
        st = pss.Stream(case["k"], case["leaf_len"], pss.KEY_U32, batch_leaves=2)
        st.feed(torch.from_numpy(A).cuda())
        assert st.root().host(0) == [tuple(x) for x in case["root"]], case["name"]


def test_empty_stream(pss):
    st = pss.Stream(10, 100)
    assert st.root().host(0) == []
    st.feed(torch.zeros(0, dtype=torch.uint32, device="cuda"))
    assert st.root().host(0) == [] and st.n_seen == 0


@pytest.mark.parametrize("seed", range(6))
def test_ragged_device_feeds(pss, seed):
    rng = np.random.default_rng(seed)
    n = int(rng.integers(2000, 40000))
    leaf_len = int(rng.integers(37, 3000))
    k = int(rng.integers(2, 64))
    batch = int(rng.integers(1, 9))          # small batches: many K1 launches and carries
    A = inputs.zipf(n, float(rng.uniform(0.8, 1.6)), 5000.0, seed=seed + 100)
    cuts = np.sort(rng.integers(0, n, size=int(rng.integers(1, 12))))
    cuts = np.concatenate([cuts, cuts[:1]])  # a repeated cut feeds an empty chunk
    feed_and_check(pss, A, k, leaf_len, batch, sorted(cuts.tolist()))


def test_aligned_big_blocks(pss):
    """Feeds of exact multiples of the leaf length: whole aligned power-of-two blocks reduced by
    the tree kernel, carries across feeds, a count of leaves with many set bits (2^6 - 1)."""
    A = inputs.zipf(63 * 512, 1.1, 1e6, seed=9)
    cuts = [512 * x for x in (1, 3, 7, 8, 24, 40, 41, 62)]
    feed_and_check(pss, A, 40, 512, 16, cuts)


def test_host_feeds(pss):
    rng = np.random.default_rng(4)
    A = inputs.zipf(60000, 1.2, 1e4, seed=4)
    cuts = sorted(rng.integers(0, A.size, size=6).tolist())
    feed_and_check(pss, A, 30, 1000, 3, cuts, host=True)


def test_u64_keys(pss):
    A = inputs.zipf(50000, 1.8, float(1 << 40), seed=5, key_bytes=8, tail_frac=0.01)
    feed_and_check(pss, A, 64, 4096, 4, [1, 4095, 4097, 20000, 33333])


def test_equals_one_shot_path(pss):
    """n = P * leaf_len: the stream's root is the root of pss_summarize + pss_merge with P blocks
    (Alg. 1's bounds are r * leaf_len), whatever the feeds."""
    n, k, P = 1 << 20, 500, 64
    A = inputs.zipf(n, 1.1, 1e8, seed=12)
    dA = torch.from_numpy(A).cuda()
    one = pss.pss_merge(pss.pss_summarize(dA, k, P)).host(0)
    st = pss.Stream(k, n // P, pss.KEY_U32, batch_leaves=16)
    for lo, hi in [(0, 1000), (1000, 300_000), (300_000, 300_001), (300_001, n)]:
        st.feed(dA[lo:hi])
    assert st.root().host(0) == one
    assert one == oracle.tree(oracle.leaves(A, k, P, threads=8), k).as_tuples()


def test_full_size_host_stream(pss):
    """C2's 2^28 keys fed from pinned host memory in 8 pieces through 2 x 256 MiB device buffers:
    the root equals the one-shot GPU root with P = 4096 (checked against the oracle on sampled
    leaves in test_gpu_parity), and every true k-majority item is a candidate."""
    w = inputs.WORKLOADS["C2"]
    A = w.generate()
    hA = torch.from_numpy(A).pin_memory()
    dA = hA.cuda()
    one = pss.pss_merge(pss.pss_summarize(dA, w.k, w.P)).host(0)
    st = pss.Stream(w.k, A.size // w.P, pss.KEY_U32, batch_leaves=1024)
    step = A.size // 8
    for g in range(8):
        st.feed(hA[g * step:(g + 1) * step])
    root = st.root()
    assert root.host(0) == one
    cand, n_cand = pss.pss_prune(root, A.size)
    cset = set(cand[:int(n_cand.item())].cpu().numpy().astype(np.uint64).tolist())
    u, c = torch.unique(dA.view(torch.int32), return_counts=True)  # brute-force histogram
    true = u[c * w.k > A.size].cpu().numpy().view(np.uint32).astype(np.uint64).tolist()
    assert set(true) <= cset and len(true) > 0


def test_large_k_stream(pss):
    """k = 5000 (global-memory K1 state, level-by-level merges) with ragged feeds."""
    A = inputs.zipf(300_000, 1.1, 1e6, seed=78)
    feed_and_check(pss, A, 5000, 40_000, 3, [1, 39_999, 40_001, 150_000], check_every=False)


def test_summarize_merge_large_k(pss):
    """The fused call falls back to the ordered path when the tree cannot run persistently."""
    A = inputs.zipf(500_000, 1.1, 1e6, seed=79)
    dA = torch.from_numpy(A).cuda()
    leaves, root = pss.pss_summarize_merge(dA, 5000, 6)
    assert root.host(0) == oracle.tree(oracle.leaves(A, 5000, 6, threads=6), 5000).as_tuples()


def test_stream_beyond_2_32_items(pss):
    """A stream of the paper's scale (29 10^9 items; the on-line setting of P:42): H's
    2^29 keys fed 9 times, 4.83 10^9 items > 2^32, k = 100, leaves of 2^16. Above its blocks the
    stream keeps 64-bit counts; its root equals the oracle's fixed tree over the 9 x 8192 leaves."""
    w = inputs.WORKLOADS["H"]
    A = w.generate()
    k, LL, reps = 100, 1 << 16, 9
    dA = torch.from_numpy(A).cuda()
    st = pss.Stream(k, LL, pss.KEY_U32, batch_leaves=1024)
    for _ in range(reps):
        st.feed(dA)
    root = st.root(wide=True)
    torch.cuda.synchronize()
    assert st.n_seen == reps * A.size > 1 << 32
    with pytest.raises(pss.PssError):
        st.root()  # u32 counts are refused past R9's bound
    it, c, e, sz = oracle.leaves_padded(A, k, A.size // LL, threads=inputs.host_threads())
    ref = oracle.tree_padded(*(np.concatenate([x] * reps) for x in (it, c, e, sz)), k,
                             threads=inputs.host_threads())
    assert root.host(0) == ref.as_tuples()


def test_stream_count_beyond_2_32(pss):
    """Closed form: one key repeated 9 x 2^29 times is the whole summary, with count 9 x 2^29
    (> 2^32: a u32 counter would wrap) and error 0."""
    x = 0xDEADBEEF
    dA = torch.full((1 << 29,), x, dtype=torch.uint32, device="cuda")
    st = pss.Stream(10, 1 << 16, pss.KEY_U32, batch_leaves=4096)
    for _ in range(9):
        st.feed(dA)
    assert st.root(wide=True).host(0) == [(x, 9 << 29, 0)]
