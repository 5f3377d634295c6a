"""Wide summaries (64-bit counts and errors) for the tree above the leaves when a stream exceeds
2^31 items (several ranks' roots, the on-line stream): every call against the oracle, whose
COMBINE, tree, prune and report are 64-bit (oracle/pss_oracle.c), with counts beyond 2^32."""
import numpy as np
import pytest
import torch

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


def big_summary(rng, k, full, pool, scale):
    """A summary in canonical order with counts around `scale` (beyond 2^32 when scale is)."""
    size = k if full else int(rng.integers(0, k + 1))
    items = rng.choice(pool, size=size, replace=False).astype(np.uint64)
    counts = (scale + rng.integers(1, 1 << 20, size=size)).astype(np.uint64)
    errs = (counts // np.uint64(3)).astype(np.uint64)
    return oracle.canonical(oracle.Summary(items, counts, errs))


def pack(pss, ss, k, kt):
    S = pss.Summaries.empty(len(ss), k, kt, "cuda", wide=True)
    dt = np.uint32 if kt == pss.KEY_U32 else np.uint64
    it = np.zeros((len(ss), k), dt)
    c = np.zeros((len(ss), k), np.uint64)
    e = np.zeros((len(ss), k), np.uint64)
    sz = np.zeros(len(ss), np.uint32)
    for i, s in enumerate(ss):
        it[i, :len(s)], c[i, :len(s)], e[i, :len(s)] = s.items.astype(dt), s.counts, s.errs
        sz[i] = len(s)
    S.items.copy_(torch.from_numpy(it))
    S.counts.copy_(torch.from_numpy(c))
    S.errs.copy_(torch.from_numpy(e))
    S.sizes.copy_(torch.from_numpy(sz))
    return S


@pytest.mark.parametrize("k,kb", [(2, 4), (17, 8), (100, 4), (1000, 4), (2500, 8)])
def test_combine_wide_equals_oracle(pss, k, kb):
    rng = np.random.default_rng(k + kb)
    kt = pss.KEY_U32 if kb == 4 else pss.KEY_U64
    pool = rng.integers(0, 1 << 31, size=3 * k + 4)
    pairs = [(big_summary(rng, k, i % 3 != 0, pool, 1 << 33),
              big_summary(rng, k, i % 4 != 0, pool, 1 << 34)) for i in range(12)]
    a = pack(pss, [p[0] for p in pairs], k, kt)
    b = pack(pss, [p[1] for p in pairs], k, kt)
    out = pss.pss_combine_wide(a, b)
    torch.cuda.synchronize()
    for i, (s1, s2) in enumerate(pairs):
        assert out.host(i) == oracle.combine(s1, s2, k).as_tuples(), i


@pytest.mark.parametrize("count", [1, 2, 3, 5, 8, 13])
def test_merge_wide_equals_oracle_tree(pss, count):
    rng = np.random.default_rng(count)
    k = 300
    pool = rng.integers(0, 1 << 31, size=4 * k)
    ss = [big_summary(rng, k, i % 2 == 0, pool, 1 << 35) for i in range(count)]
    root = pss.pss_merge_wide(pack(pss, ss, k, pss.KEY_U32))
    torch.cuda.synchronize()
    assert root.host(0) == oracle.tree(ss, k).as_tuples()


def test_widen_then_merge_equals_narrow_merge(pss):
    """Below 2^31 items the wide tree is the narrow one: widening the leaves of a real input and
    merging them wide gives pss_merge's root."""
    import inputs
    A = torch.from_numpy(inputs.zipf(1 << 20, 1.1, 1e6, seed=5)).cuda()
    leaves = pss.pss_summarize(A, 200, 16)
    narrow = pss.pss_merge(leaves)
    wide = pss.pss_merge_wide(pss.pss_widen(leaves))
    torch.cuda.synchronize()
    assert wide.host(0) == narrow.host(0)


@pytest.mark.parametrize("n", [(1 << 31) + 7, 1 << 36, (1 << 40) + 12345])
def test_prune_and_report_beyond_2_31(pss, n):
    """pss_prune_wide and pss_report with n > 2^31 (the threshold floor(n/k) + 1, in 64
    bits) against the oracle's prune and result."""
    rng = np.random.default_rng(n % 1000)
    k = 64
    thr = oracle.threshold(n, k)
    pool = rng.integers(0, 1 << 31, size=4 * k)
    items = rng.choice(pool, size=k, replace=False).astype(np.uint64)
    counts = (thr - (1 << 20) + rng.integers(0, 1 << 21, size=k)).astype(np.uint64)
    root = oracle.canonical(oracle.Summary(items, counts, counts // np.uint64(7)))
    W = pack(pss, [root], k, pss.KEY_U32)
    cand, n_cand = pss.pss_prune_wide(W, n)
    torch.cuda.synchronize()
    nc = int(n_cand.item())
    want = oracle.prune(root, n, k)
    assert 0 < nc < k and cand[:nc].cpu().numpy().astype(np.uint64).tolist() == want.tolist()
    exact = (thr - 5 + rng.integers(0, 10, size=nc)).astype(np.uint64)
    oi, oc, ol = pss.pss_report(cand, torch.from_numpy(exact).cuda(), n, k, n_cand=n_cand)
    torch.cuda.synchronize()
    ln = int(ol.item())
    ri, rc = oracle.result(want, exact, n, k)
    assert oi[:ln].cpu().numpy().astype(np.uint64).tolist() == ri.tolist()
    assert oc[:ln].cpu().numpy().tolist() == rc.tolist()
