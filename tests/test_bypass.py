"""GPU parity of K1's level-pinned bypass (summarize.cu, hot.cu): with PSS_BYPASS=2 the bypass
runs on every shape the kernel supports (u32 keys, packed counters) and keeps any table of
frequent keys, so small blocks, tiny k and keys that hover at the minimum level (pinned, unpinned,
evicted, re-inserted) are exercised. Every leaf and the root are compared with the oracle's
sequential Space Saving bit for bit; PSS_BYPASS=0 must give the same bits.
"""
import numpy as np
import pytest
import torch

import inputs
import oracle
from test_gpu_parity import assert_full_parity, pss, to_dev  # noqa: F401  (pss is a fixture)

pytestmark = pytest.mark.gpu


@pytest.fixture(autouse=True)
def force_bypass(monkeypatch):
    monkeypatch.setenv("PSS_BYPASS", "2")


def leaves_equal(pss, A, k, P):
    ref = oracle.leaves(A, k, P, threads=8)
    got = pss.pss_summarize(to_dev(A), k, P)
    torch.cuda.synchronize()
    for r in range(P):
        assert got.host(r) == ref[r].as_tuples(), f"leaf {r}"
    return got


@pytest.mark.parametrize("n,k,P,s,U", [
    (200_000, 64, 3, 1.3, 5000), (1 << 20, 1000, 16, 1.1, 1e8), (300_000, 257, 2, 1.1, 1e8),
    (100_000, 8, 3, 1.5, 30), (65_536, 1000, 1, 1.1, 1e6), (200_000, 2, 16, 0.6, 1e5),
    (250_000, 100, 5, 3.0, 1e6), (131_071, 500, 1, 2.0, 1e7), (40_000, 33, 9, 1.1, 400),
    (1000, 3, 7, 0.8, 20), (3, 10, 5, 1.1, 10), (0, 10, 4, 1.1, 10)])
def test_zipf_shapes(pss, n, k, P, s, U):
    A = inputs.zipf(n, s, U, seed=n * 5 + k)
    assert_full_parity(pss, A, k, P)


@pytest.mark.parametrize("seed", range(8))
def test_keys_hovering_at_the_minimum(pss, seed):
    """Frequent keys whose rate is close to the rate at which the minimum level rises: they are
    pinned in some levels, members of B_m in others, evicted and inserted again."""
    rng = np.random.default_rng(100 + seed)
    n = int(rng.integers(100_000, 400_000))
    k = int(rng.choice([16, 50, 100, 300]))
    P = int(rng.integers(1, 6))
    nh = int(rng.integers(5, 64))
    miss = float(rng.uniform(0.4, 0.8))
    # the minimum rises once per ~k / miss items; a hot key arrives ~once per level
    ph = min((1.0 - miss) / nh, float(rng.uniform(0.5, 2.0)) * miss / k)
    hot = rng.integers(0, 2**32, size=nh, dtype=np.uint64).astype(np.uint32)
    u = rng.random(n)
    A = rng.integers(0, 2**32, size=n, dtype=np.uint64).astype(np.uint32)
    sel = u < ph * nh
    A[sel] = hot[(u[sel] / ph).astype(np.int64) % nh]
    leaves_equal(pss, A, k, P)


@pytest.mark.parametrize("seed", range(6))
def test_tiny_universe(pss, seed):
    rng = np.random.default_rng(seed)
    n = int(rng.integers(1, 60_000))
    U = int(rng.integers(2, 40))
    k = int(rng.integers(2, 12))
    P = int(rng.integers(1, 5))
    A = (rng.integers(0, U, size=n).astype(np.uint32) * np.uint32(2654435761)).astype(np.uint32)
    assert_full_parity(pss, A, k, P)


def test_bursts_and_phase_changes(pss):
    """A key that is frequent early and absent later (stays pinned with a large count), one that
    appears only late, long runs of one key (look-ahead far beyond the cold queue)."""
    rng = np.random.default_rng(7)
    n = 600_000
    A = rng.integers(0, 2**32, size=n, dtype=np.uint64).astype(np.uint32)
    A[: n // 3][rng.random(n // 3) < 0.5] = 11
    A[n // 2:][rng.random(n - n // 2) < 0.3] = 22
    A[100_000:140_000] = 33
    A[rng.random(n) < 0.05] = 44
    for k, P in [(100, 1), (1000, 4), (20, 3)]:
        leaves_equal(pss, A, k, P)


def test_same_bits_without_the_bypass(pss, monkeypatch):
    A = inputs.zipf(1 << 21, 1.1, 1e8, seed=9)
    monkeypatch.setenv("PSS_BYPASS", "1")  # the default gate: blocks of 2^16 keys, k = 1000
    a = pss.pss_summarize(to_dev(A), 1000, 32)
    monkeypatch.setenv("PSS_BYPASS", "0")
    b = pss.pss_summarize(to_dev(A), 1000, 32)
    torch.cuda.synchronize()
    for f in ("items", "counts", "errs", "sizes"):
        assert torch.equal(getattr(a, f), getattr(b, f)), f
    ref = oracle.leaves(A, 1000, 32, threads=8)
    for r in range(32):
        assert a.host(r) == ref[r].as_tuples(), f"leaf {r}"


def test_other_entry_points_with_the_bypass(pss):
    """The hybrid decomposition (two-level block bounds), the on-line stream (launches over
    ranges of a batch) and the host-fed query (one launch per landed chunk) sample their own range
    of A; all bit-exact with the bypass forced."""
    from test_hybrid import test_hybrid_parity
    from test_stream import feed_and_check
    test_hybrid_parity(pss, 120_000, 64, 3, 8, 1.5, 1e5)
    test_hybrid_parity(pss, 200_000, 1000, 4, 6, 1.1, 1e8)
    A = inputs.zipf(300_000, 1.4, 1e6, seed=21)
    feed_and_check(pss, A, 100, 4096, 8, [0, 5000, 5001, 70_000, 200_000, 300_000])
    feed_and_check(pss, A, 100, 4096, 4, [0, 123_457, 300_000], host=True)
    ref = oracle.pipeline(A, 100, 16, threads=8)
    items, counts = pss.pss_query_host(torch.from_numpy(A).pin_memory(), 100, 16)
    assert items.numpy().astype(np.uint64).tolist() == ref.result[0].tolist()
    assert counts.numpy().astype(np.uint64).tolist() == ref.result[1].tolist()
