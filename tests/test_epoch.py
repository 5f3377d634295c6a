"""K1e (csrc/epoch.cu): leaves of u32 keys with 64 <= k <= 2048, epoch by epoch, one CTA per block.

Every leaf is compared bit for bit with the oracle's sequential Space Saving (R1/R2),
and with K1 (the per-warp batched rule, forced by PSS_EPOCH=0) on the same input. The inputs are
chosen to exercise what is specific to the epoch formulation: many V events (universes just above
k, where nearly every key is a member when it recurs), epochs that end inside a window and exactly
at window ends, ragged block tails, single-event epochs (a uniform stream over k + 1 keys), the
fill epoch ending mid-window or never (k >= distinct keys), extreme key values, and k at both ends
of K1e's range.
"""
import os

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
    old = os.environ.get("PSS_EPOCH")
    os.environ["PSS_EPOCH"] = "1"  # K1e on for this module (K1 is forced per call below)
    from conftest import build_lib
    build_lib()
    import paper_1606_04669_b200 as p
    yield p
    if old is None:
        os.environ.pop("PSS_EPOCH", None)
    else:
        os.environ["PSS_EPOCH"] = old


def leaves_of(pss, A, k, P):
    dA = torch.from_numpy(np.ascontiguousarray(A)).cuda()
    S = pss.pss_summarize(dA, k, P)
    torch.cuda.synchronize()
    return [S.host(r) for r in range(P)]


def check(pss, A, k, P, monkeypatch, against_k1=True):
    assert pss.epoch_used(A.size, k, P, 4), "K1e should take this shape"
    got = leaves_of(pss, A, k, P)
    ref = oracle.leaves(A, k, P, threads=8)
    for r in range(P):
        assert got[r] == ref[r].as_tuples(), f"leaf {r} (n={A.size}, k={k}, P={P})"
    if against_k1:
        with monkeypatch.context() as m:
            m.setenv("PSS_EPOCH", "0")
            assert not pss.epoch_used(A.size, k, P, 4)
            assert leaves_of(pss, A, k, P) == got


@pytest.mark.parametrize("k", [64, 100, 257, 1000, 2047, 2048])
@pytest.mark.parametrize("extra", [1, 7, 64])
def test_universe_just_above_k(pss, monkeypatch, k, extra):
    """U = k + extra keys: almost every recurring key is a member (V events in every epoch)."""
    rng = np.random.default_rng(k * 131 + extra)
    n = int(rng.integers(3 * k, 40 * k))
    A = (rng.integers(0, k + extra, size=n).astype(np.uint64) * 2654435761 % (1 << 32))
    check(pss, A.astype(np.uint32), k, int(rng.integers(1, 4)), monkeypatch)


@pytest.mark.parametrize("k", [64, 1000, 2048])
def test_round_robin_k_plus_one(pss, monkeypatch, k):
    """k + 1 keys in round robin: every item evicts, every epoch has a handful of events."""
    A = (np.arange(20 * (k + 1), dtype=np.uint64) % (k + 1) * 40503 + 11).astype(np.uint32)
    check(pss, A, k, 1, monkeypatch)
    check(pss, A[::-1].copy(), k, 3, monkeypatch)


@pytest.mark.parametrize("n,k,P,s,U", [
    (1 << 17, 1000, 2, 1.1, 1e8), (1 << 17, 1000, 2, 0.5, 1e8), (300_001, 500, 5, 1.3, 5e4),
    (65_536 * 3 + 17, 1000, 3, 1.1, 1e6), (200_000, 64, 7, 0.9, 1e4), (100_000, 2000, 2, 1.5, 1e8),
    (1_000_000, 1000, 16, 1.1, 1e8), (150_000, 300, 1, 2.0, 1e8), (123_457, 777, 4, 1.0, 3000)])
def test_zipf(pss, monkeypatch, n, k, P, s, U):
    A = inputs.zipf(n, s, U, seed=n + k)
    check(pss, A, k, P, monkeypatch)


@pytest.mark.parametrize("n", [1, 2, 63, 511, 512, 513, 1023, 1024, 1025, 4096, 70_000])
def test_window_edges(pss, monkeypatch, n):
    """Block lengths around the 512-item window; k > distinct (fill epoch never ends) and not."""
    rng = np.random.default_rng(n)
    for U in (50, 3000):
        A = (rng.integers(0, U, size=n).astype(np.uint64) * 97 + 5).astype(np.uint32)
        check(pss, A, 100, 1, monkeypatch)


def test_extreme_keys(pss, monkeypatch):
    """0 and all-ones are ordinary ids (R12): empty table / U-table entries are not keys."""
    rng = np.random.default_rng(9)
    base = rng.integers(0, 1 << 32, size=300, dtype=np.uint64).astype(np.uint32)
    base[:4] = [0, 0xFFFFFFFF, 0xFFFFFFFE, 0x7FFFFFFF]
    A = rng.choice(base, size=80_000)
    check(pss, A, 128, 3, monkeypatch)
    A[::3] = 0xFFFFFFFF
    check(pss, A, 64, 2, monkeypatch)


def test_all_distinct_and_all_equal(pss, monkeypatch):
    A = (np.random.default_rng(3).permutation(np.arange(150_000, dtype=np.uint64)) * 7 + 1)
    check(pss, A.astype(np.uint32), 1000, 2, monkeypatch)
    check(pss, np.full(90_000, 0xFFFFFFFF, np.uint32), 64, 3, monkeypatch)


def test_hybrid_bounds(pss):
    """The two-level decomposition (f4) through K1e."""
    A = inputs.zipf(400_003, 1.1, 1e6, seed=17)
    dA = torch.from_numpy(A).cuda()
    S = pss.pss_summarize_hybrid(dA, 500, 3, 5)
    torch.cuda.synchronize()
    ref, _ = oracle.hybrid(A, 500, 3, 5)
    for r in range(15):
        assert S.host(r) == ref[r].as_tuples()
