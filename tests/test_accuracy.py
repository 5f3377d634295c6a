"""GPU parity of the accuracy row: pss_exact_kmajority (local heavy hitters, no
Space Saving) against the k-majority definition from a sort-based histogram (oracle.kmajority),
bit for bit; pss_accuracy's precision/recall (exact rationals) and ARE (fp64, summation order
differs: relative tolerance 1e-12) against oracle.accuracy on the same root and exact counts."""
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


def exact_gpu(pss, dA, k):
    items, counts, length, overflow = pss.pss_exact_kmajority(dA, k)
    ln = int(length.item())
    assert int(overflow.item()) == 0
    return (items[:ln].cpu().numpy().astype(np.uint64).tolist(),
            counts[:ln].cpu().numpy().astype(np.uint64).tolist())


def check_exact(pss, A, k):
    got = exact_gpu(pss, torch.from_numpy(A).cuda(), k)
    u, c = oracle.kmajority(A, k)
    assert got == (u.tolist(), c.tolist())


@pytest.mark.parametrize("n,k,s,U", [
    (0, 10, 1.1, 10), (1, 2, 1.1, 10), (4095, 3, 1.1, 50), (4097, 7, 0.9, 1000),
    (100_000, 100, 1.1, 1e6), (250_000, 1000, 1.1, 1e8), (123_457, 20000, 1.5, 2**32 - 1),
    (300_000, 2, 0.5, 1e5), (77_777, 64, 2.0, 1e3)])
def test_exact_kmajority_small(pss, n, k, s, U):
    check_exact(pss, inputs.zipf(n, s, U, seed=n + k), k)


def test_exact_kmajority_edges(pss):
    check_exact(pss, np.full(10_000, 0xFFFFFFFF, np.uint32), 2)        # one key, all-ones id
    check_exact(pss, np.arange(50_000, dtype=np.uint32), 10)            # nothing is frequent
    A = np.repeat(np.array([0, 5, 9], np.uint32), [5001, 5000, 4999])   # exact-threshold ties
    check_exact(pss, np.random.default_rng(1).permutation(A), 3)
    B = inputs.zipf(200_000, 1.8, float(1 << 40), seed=5, key_bytes=8, tail_frac=0.01)
    check_exact(pss, B, 500)


# full BASELINE sizes: test_gpu_parity.py::test_full_size compares pss_exact_kmajority with a
# brute-force histogram on every config


def run_accuracy(pss, A, k, P):
    dA = torch.from_numpy(A).cuda()
    root = pss.pss_merge(pss.pss_summarize(dA, k, P))
    cand, n_cand = pss.pss_prune(root, A.size)
    exact = pss.pss_verify(dA, cand, n_cand)
    _, _, n_true, _ = pss.pss_exact_kmajority(dA, k)
    rep = pss.pss_accuracy(root, A.size, n_cand, exact, n_true).as_dict()
    nc = int(n_cand.item())
    ref_root = oracle.tree(oracle.leaves(A, k, P, threads=8), k)
    assert root.host(0) == ref_root.as_tuples()
    rc = oracle.prune(ref_root, A.size, k)
    u, c = np.unique(A, return_counts=True)
    want = oracle.accuracy(rc, ref_root.counts[:rc.size], dict(zip(u.tolist(), c.tolist())), A.size, k)
    assert nc == want["n_reported"]
    for f in ("n_reported", "n_reported_true", "n_true", "precision", "recall"):
        assert rep[f] == want[f], f
    for f in ("are_reported", "are_true"):
        assert abs(rep[f] - want[f]) <= 1e-12 * max(1.0, abs(want[f])), f
    return rep


@pytest.mark.parametrize("n,k,P,s,U", [(200_000, 100, 16, 1.1, 1e6), (1 << 20, 1000, 64, 1.1, 1e8),
                                       (500_000, 50, 7, 0.8, 1e4), (300_000, 20, 3, 2.0, 1e3)])
def test_accuracy_report(pss, n, k, P, s, U):
    rep = run_accuracy(pss, inputs.zipf(n, s, U, seed=n + P), k, P)
    assert rep["recall"] == 1.0  # no false negatives


def test_accuracy_no_candidates(pss):
    rep = run_accuracy(pss, np.arange(20_000, dtype=np.uint32), 10, 4)
    assert rep["n_reported"] == 0 and rep["precision"] == 1.0 and rep["recall"] == 1.0
