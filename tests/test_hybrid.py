"""GPU parity of the hybrid decomposition (include/pss.h pss_*_hybrid): leaves of
the two-level decomposition and the per-process-then-cross-process tree against oracle.hybrid, bit
for bit, including non-power-of-two thread counts (a different tree shape from pss_merge)."""
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


@pytest.mark.parametrize("n,k,Pp,T,s,U", [
    (50_000, 30, 2, 3, 1.1, 1e4), (77_777, 100, 5, 7, 1.1, 1e6), (10_007, 8, 3, 1, 0.9, 500),
    (10_007, 8, 1, 5, 0.9, 500), (200_000, 1000, 4, 6, 1.1, 1e8), (3, 5, 2, 3, 1.1, 10),
    (120_000, 64, 3, 8, 1.5, 1e5)])
def test_hybrid_parity(pss, n, k, Pp, T, s, U):
    A = inputs.zipf(n, s, U, seed=n + Pp * 10 + T)
    dA = torch.from_numpy(A).cuda()
    leaves = pss.pss_summarize_hybrid(dA, k, Pp, T)
    root = pss.pss_merge_hybrid(leaves, T)
    ref_leaves, ref_root = oracle.hybrid(A, k, Pp, T)
    for r in range(Pp * T):
        assert leaves.host(r) == ref_leaves[r].as_tuples(), f"leaf {r}"
    assert root.host(0) == ref_root.as_tuples()


def test_hybrid_power_of_two_equals_flat(pss):
    """T a power of two and Pp*T | n: the hybrid root is pss_summarize + pss_merge's root."""
    n, k, Pp, T = 1 << 20, 500, 16, 4
    A = inputs.zipf(n, 1.1, 1e8, seed=33)
    dA = torch.from_numpy(A).cuda()
    flat = pss.pss_merge(pss.pss_summarize(dA, k, Pp * T)).host(0)
    assert pss.pss_merge_hybrid(pss.pss_summarize_hybrid(dA, k, Pp, T), T).host(0) == flat


def test_hybrid_u64(pss):
    A = inputs.zipf(100_000, 1.8, float(1 << 40), seed=5, key_bytes=8, tail_frac=0.01)
    dA = torch.from_numpy(A).cuda()
    root = pss.pss_merge_hybrid(pss.pss_summarize_hybrid(dA, 200, 3, 5), 5)
    assert root.host(0) == oracle.hybrid(A, 200, 3, 5)[1].as_tuples()


def test_hybrid_large_k(pss):
    """k = 5000: K1 keeps its state in global memory and every tree level is its own launch."""
    A = inputs.zipf(400_000, 1.1, 1e6, seed=77)
    dA = torch.from_numpy(A).cuda()
    root = pss.pss_merge_hybrid(pss.pss_summarize_hybrid(dA, 5000, 2, 3), 3)
    assert root.host(0) == oracle.hybrid(A, 5000, 2, 3)[1].as_tuples()
