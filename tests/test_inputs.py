"""The seeded input generator (inputs/): determinism, prefix property, Zipf law, bijective ids."""
import numpy as np
import pytest

import inputs


def test_zipf_normalisation_U3():
    """U=3, s=1 -> P(rank 1) = 1/(1 + 1/2 + 1/3) = 6/11; empirical within 4 sigma."""
    n = 1_000_000
    r = inputs.zipf(n, 1.0, 3, seed=9, hash_ids=False)
    p = 6 / 11
    assert r.max() == 2 and r.min() == 0
    assert abs((r == 0).mean() - p) < 4 * np.sqrt(p * (1 - p) / n)


@pytest.mark.parametrize("s,U", [(1.1, 100), (0.5, 50), (2.0, 80), (1.0, 30)])
def test_zipf_chi_square(s, U):
    """Chi-squared agreement with i^-s / sum_j j^-s on U <= 100, n = 10^6."""
    from scipy import stats
    n = 1_000_000
    r = inputs.zipf(n, s, U, seed=int(s * 10) + U, hash_ids=False)
    obs = np.bincount(r.astype(np.int64), minlength=U)
    w = np.arange(1, U + 1, dtype=np.float64) ** -s
    exp = n * w / w.sum()
    chi2 = ((obs - exp) ** 2 / exp).sum()
    assert stats.chi2.sf(chi2, U - 1) > 1e-3


def test_zipf_large_universe_head():
    """s=1.1 over U=10^8: rank-1 frequency within 4 sigma of 1/H(U, 1.1)."""
    n = 2_000_000
    r = inputs.zipf(n, 1.1, 1e8, seed=5, hash_ids=False)
    i = np.arange(1, 10**6 + 1, dtype=np.float64)
    H = (i ** -1.1).sum() + (10 * ((1e6 + 0.5) ** -0.1 - (1e8 + 0.5) ** -0.1))  # tail integral
    p = 1 / H
    assert abs((r == 0).mean() - p) < 4 * np.sqrt(p * (1 - p) / n)


def test_deterministic_prefix_and_threads():
    a = inputs.zipf(100_000, 1.1, 1e8, seed=2, threads=1)
    b = inputs.zipf(100_000, 1.1, 1e8, seed=2, threads=7)
    c = inputs.zipf(37_000, 1.1, 1e8, seed=2, threads=3)
    assert np.array_equal(a, b) and np.array_equal(a[:37_000], c)
    assert not np.array_equal(a, inputs.zipf(100_000, 1.1, 1e8, seed=3))


def test_ids_are_bijective_mix():
    r = np.arange(0, 1 << 16, dtype=np.uint64)
    m32 = {inputs.mix32(int(x)) for x in r}
    m64 = {inputs.mix64(int(x)) for x in r}
    assert len(m32) == len(r) and len(m64) == len(r)
    raw = inputs.zipf(1000, 1.1, 1e8, seed=2, hash_ids=False)
    hashed = inputs.zipf(1000, 1.1, 1e8, seed=2)
    assert [inputs.mix32(int(x)) for x in raw[:50]] == hashed[:50].tolist()


def test_u64_tail():
    n = 400_000
    a = inputs.zipf(n, 1.8, float(1 << 40), seed=5, key_bytes=8, tail_frac=0.01)
    assert a.dtype == np.uint64
    raw = inputs.zipf(n, 1.8, float(1 << 40), seed=5, key_bytes=8, tail_frac=0.01, hash_ids=False)
    # about 1% uniform ranks in [0, 2^40): nearly all distinct and mostly huge
    big = raw >= (1 << 30)
    assert abs(big.mean() - 0.01) < 0.002
    assert (raw < (1 << 40)).all()


def test_workload_registry():
    w = inputs.WORKLOADS
    assert w["C1"].n == 10**6 and w["C1"].k == 100 and w["C1"].P == 64
    assert w["H"].n == 1 << 29 and w["H"].k == 1000
    assert w["C5"].key_bytes == 8 and w["C5"].P == 32768
    assert np.array_equal(w["H"].generate(5000), w["C2"].generate(5000))


def test_ranges_of_the_stream():
    a = inputs.zipf(50_000, 1.1, 1e8, seed=2)
    b = inputs.zipf(20_000, 1.1, 1e8, seed=2, start=30_000, threads=3)
    assert np.array_equal(a[30_000:], b)


def test_bench_custom_workload_flags():
    """bench.py's --n/--k/--P/--zipf-s/--universe/--seed override the named workload's fields."""
    import argparse
    import importlib.util
    import os
    spec = importlib.util.spec_from_file_location(
        "_bench", os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "bench.py"))
    bench = importlib.util.module_from_spec(spec)
    spec.loader.exec_module(bench)
    base = dict(workload="H", n=0, k=0, P=0, zipf_s=0.0, universe=0.0, seed=-1)
    w = bench.workload_of(argparse.Namespace(**base))
    assert (w.name, w.n, w.k, w.P) == ("H", 1 << 29, 1000, 8192)
    w = bench.workload_of(argparse.Namespace(**{**base, "P": 4096}))
    assert (w.name, w.P) == ("H", 4096)
    w = bench.workload_of(argparse.Namespace(**{**base, "n": 10**6, "k": 50, "zipf_s": 1.3, "seed": 7}))
    assert (w.name, w.n, w.k, w.s, w.seed, w.universe) == ("H-custom", 10**6, 50, 1.3, 7, 1e8)
    assert bench.l2_flush_needed(w) and not bench.l2_flush_needed(bench.workload_of(argparse.Namespace(**base)))
