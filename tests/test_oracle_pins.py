"""Pins for the CPU oracle (oracle/), checked against things other than itself.

Each test names what pins it: a worked example (tests/golden/worked_examples.json, each cited),
a closed form, a textbook special case computed with numpy, or a guarantee of the paper checked
by brute force over every small input. The oracle's own formulas are never retyped here.
"""
import itertools

import numpy as np
import pytest

import oracle
from conftest import letters

pytestmark = pytest.mark.filterwarnings("ignore")


def S(lst):
    return [tuple(x) for x in lst]


def hist(arr):
    u, c = np.unique(np.asarray(arr, dtype=np.uint64), return_counts=True)
    return dict(zip(u.tolist(), c.tolist()))


# ---------------------------------------------------------------- a1: block decomposition
def test_bounds_golden(golden):
    for case in golden["bounds"]:
        assert [list(r) for r in oracle.bounds(case["n"], case["P"])] == case["ranges"], case["cite"]


@pytest.mark.parametrize("n", list(range(0, 130)) + [997, 1000, 4096 + 7])
def test_bounds_tile_exactly(n):
    """S:227 tiling: ranges partition [0, n) in order, sizes floor(n/P) or ceil(n/P)."""
    for P in range(1, 65):
        rng = oracle.bounds(n, P)
        assert rng[0][0] == 0 and rng[-1][1] == n
        for (a, b), (c, _) in zip(rng, rng[1:]):
            assert b == c
        sizes = {b - a for a, b in rng}
        assert sizes <= {n // P, -(-n // P)}


def test_bounds_large_no_overflow():
    n, P = (1 << 31) + 12345, 32768
    rng = oracle.bounds(n, P)
    assert rng[-1][1] == n
    assert all(b - a in (n // P, n // P + 1) for a, b in rng)


# ---------------------------------------------------------------- a2: leaf Space Saving
def test_space_saving_golden(golden):
    for case in golden["space_saving"]:
        got = oracle.space_saving(letters(case["stream"]), case["k"]).as_tuples()
        assert got == S(case["summary"]), (case["name"], case["cite"])


def test_min_golden(golden):
    for case in golden["min"]:
        assert oracle.min_count(case["summary"], case["k"]) == case["min"], case["cite"]


@pytest.mark.parametrize("L,k", [(1, 3), (5, 5), (7, 3), (100, 7), (1000, 64), (4097, 100)])
def test_space_saving_all_distinct_closed_form(L, k):
    """All-distinct stream: eviction is round-robin over slots (R1), so slot j holds
    A[j + k*floor((L-1-j)/k)] with count floor((L-1-j)/k) + 1 and err = count - 1."""
    rng = np.random.default_rng(L * 31 + k)
    A = rng.permutation(np.arange(10 * L + 5, dtype=np.uint64))[:L] * 7 + 3
    got = oracle.space_saving(A, k)
    assert len(got) == min(L, k)
    for j in range(min(L, k)):
        q = (L - 1 - j) // k
        assert int(got.items[j]) == int(A[j + k * q])
        assert int(got.counts[j]) == q + 1
        assert int(got.errs[j]) == q


@pytest.mark.parametrize("seed", range(6))
def test_space_saving_exact_when_k_covers_distinct(seed):
    """k >= #distinct: the summary is the exact histogram in first-occurrence order (textbook
    unique with first index), errors 0."""
    rng = np.random.default_rng(seed)
    A = (rng.integers(0, 50, size=500).astype(np.uint64) * 2654435761 % (1 << 32)).astype(np.uint32)
    u, first, cnt = np.unique(A, return_index=True, return_counts=True)
    order = np.argsort(first)
    got = oracle.space_saving(A, len(u) + seed)
    assert got.items.tolist() == u[order].astype(np.uint64).tolist()
    assert got.counts.tolist() == cnt[order].tolist()
    assert got.errs.tolist() == [0] * len(u)


def _check_ss_guarantees(stream, k, summ):
    L = len(stream)
    f = hist(stream) if L else {}
    assert int(summ.counts.sum()) == L  # conservation
    m = oracle.min_count(summ, k)
    assert m <= L // k
    mon = dict(zip(summ.items.tolist(), zip(summ.counts.tolist(), summ.errs.tolist())))
    assert len(mon) == len(summ) <= k
    for x, (c, e) in mon.items():
        assert f.get(x, 0) <= c <= f.get(x, 0) + e  # over-estimation with bounded error
        assert e <= m
    for x, fx in f.items():
        if fx * k > L:
            assert x in mon  # no false negatives
        if x not in mon:
            assert fx <= m
    if len(summ) < k:
        assert all(mon[x] == (f[x], 0) for x in f)


def test_space_saving_guarantees_exhaustive():
    """Every stream of length <= 8 over 4 items and <= 10 over 3 items, k in {2,3}:
    conservation, f <= f_hat <= f + err, err <= MIN <= floor(L/k), no false negatives,
    unmonitored f <= MIN."""
    for U, maxlen in ((4, 8), (3, 10)):
        for L in range(0, maxlen + 1):
            for t in itertools.product(range(1, U + 1), repeat=L):
                A = np.array(t, dtype=np.uint64)
                for k in (2, 3):
                    _check_ss_guarantees(t, k, oracle.space_saving(A, k))


def test_space_saving_u32_u64_agree_and_extreme_keys():
    """Keys 0 and all-ones are ordinary ids (R12); u32 input widens losslessly."""
    A32 = np.array([0, 0xFFFFFFFF, 0, 5, 0xFFFFFFFF, 7, 0], dtype=np.uint32)
    s32 = oracle.space_saving(A32, 2)
    s64 = oracle.space_saving(A32.astype(np.uint64), 2)
    assert s32.as_tuples() == s64.as_tuples()
    A64 = np.array([2**64 - 1, 0, 2**64 - 1], dtype=np.uint64)
    assert oracle.space_saving(A64, 2).as_tuples() == [(2**64 - 1, 2, 0), (0, 1, 0)]


# ---------------------------------------------------------------- a4: COMBINE and the tree
def test_combine_golden(golden):
    for case in golden["combine"]:
        got = oracle.combine(case["s1"], case["s2"], case["k"]).as_tuples()
        assert got == S(case["out"]), (case["name"], case["cite"])


def _check_merged(stream, k, summ):
    N = len(stream)
    f = hist(stream) if N else {}
    m = oracle.min_count(summ, k)
    mon = dict(zip(summ.items.tolist(), zip(summ.counts.tolist(), summ.errs.tolist())))
    assert len(mon) == len(summ) <= k
    assert int(summ.counts.sum()) <= N  # invariant I
    assert m <= N // k
    for x, (c, e) in mon.items():
        assert f.get(x, 0) <= c <= f.get(x, 0) + e
        assert e <= m
    for x, fx in f.items():
        if fx * k > N:
            assert x in mon
        if x not in mon:
            assert fx <= m
    if len(summ) < k:
        assert all(mon[x] == (f[x], 0) for x in f)
    # canonical order (R5)
    keyed = [(-c, x) for x, c in zip(summ.items.tolist(), summ.counts.tolist())]
    assert keyed == sorted(keyed)


def test_combine_guarantees_all_split_points():
    """Every stream of length <= 8 over {a,b,c} (and <= 6 over 4 items), every split point,
    k in {2,3}: the combined summary keeps f <= f_hat <= f + err, err <= MIN, sum <= N, no false
    negatives ("correctness and the error bounds are preserved")."""
    for U, maxlen in ((3, 8), (4, 6)):
        for L in range(0, maxlen + 1):
            for t in itertools.product(range(1, U + 1), repeat=L):
                A = np.array(t, dtype=np.uint64)
                for k in (2, 3):
                    for cut in range(L + 1):
                        s1 = oracle.space_saving(A, k, 0, cut)
                        s2 = oracle.space_saving(A, k, cut, L)
                        c12 = oracle.combine(s1, s2, k)
                        _check_merged(t, k, c12)
                        assert c12.as_tuples() == oracle.combine(s2, s1, k).as_tuples()


def test_combine_identity_with_empty():
    rng = np.random.default_rng(7)
    for k in (2, 3, 10):
        A = rng.integers(1, 30, size=200).astype(np.uint64)
        s = oracle.space_saving(A, k)
        e = oracle.empty_summary()
        assert oracle.combine(s, e, k).as_tuples() == oracle.canonical(s).as_tuples()
        assert oracle.combine(e, s, k).as_tuples() == oracle.canonical(s).as_tuples()


@pytest.mark.parametrize("seed", range(40))
def test_tree_guarantees_random(seed):
    """Random streams and P: the root of the fixed binary tree keeps the guarantees."""
    rng = np.random.default_rng(100 + seed)
    n = int(rng.integers(0, 400))
    U = int(rng.integers(1, 40))
    k = int(rng.integers(2, 12))
    P = int(rng.integers(1, 11))
    A = (rng.zipf(1.3, size=n) % U).astype(np.uint64) if n else np.zeros(0, np.uint64)
    root = oracle.tree(oracle.leaves(A, k, P), k)
    _check_merged(A.tolist(), k, root)


def test_tree_P1_is_sequential():
    rng = np.random.default_rng(3)
    A = rng.integers(0, 100, size=3000).astype(np.uint32)
    for k in (2, 10, 50):
        assert (oracle.tree(oracle.leaves(A, k, 1), k).as_tuples()
                == oracle.canonical(oracle.space_saving(A, k)).as_tuples())


def test_tree_exact_when_k_covers_distinct():
    """distinct(A) <= k: every node is unfull so the root is the exact histogram (np.unique),
    in canonical order, for any P."""
    rng = np.random.default_rng(4)
    A = rng.integers(0, 37, size=5000).astype(np.uint32)
    u, c = np.unique(A, return_counts=True)
    order = np.lexsort((u, -c.astype(np.int64)))
    want = [(int(u[i]), int(c[i]), 0) for i in order]
    for P in (1, 2, 3, 7, 16, 64):
        assert oracle.tree(oracle.leaves(A, 40, P), 40).as_tuples() == want


def test_pipeline_golden(golden):
    for case in golden["pipeline"]:
        A = letters(case["stream"])
        k, P = case["k"], case["P"]
        pl = oracle.pipeline(A, k, P)
        assert [s.as_tuples() for s in pl.leaves] == [S(x) for x in case["leaves"]]
        lv1 = [oracle.combine(pl.leaves[0], pl.leaves[1], k), oracle.combine(pl.leaves[2], pl.leaves[3], k)]
        assert [s.as_tuples() for s in lv1] == [S(x) for x in case["level1"]]
        assert pl.root.as_tuples() == S(case["root"])
        assert oracle.threshold(A.size, k) == case["threshold"]
        assert pl.cand.tolist() == case["candidates"]
        assert pl.exact.tolist() == case["exact"]
        assert pl.result[0].tolist() == case["result"]


# ---------------------------------------------------------------- a5-a7
def test_prune_golden(golden):
    for case in golden["prune"]:
        assert oracle.threshold(case["n"], case["k"]) == case["threshold"]
        assert oracle.prune(case["root"], case["n"], case["k"]).tolist() == case["candidates"], case["cite"]


def test_verify_equals_histogram():
    rng = np.random.default_rng(11)
    A = rng.integers(0, 1000, size=20000).astype(np.uint32)
    h = hist(A)
    cand = np.array([5, 999, 5, 123456, 0, 17], dtype=np.uint64)  # duplicates and an absent key
    assert oracle.verify(A, cand).tolist() == [h.get(int(x), 0) for x in cand]
    assert oracle.verify(A, np.zeros(0, np.uint64)).tolist() == []
    assert oracle.verify(np.zeros(0, np.uint32), cand).tolist() == [0] * cand.size


@pytest.mark.parametrize("case", [(20000, 1.1, 1 << 20, 100, 16), (30000, 1.5, 1e6, 10, 7),
                                  (5000, 0.7, 3000, 3, 5), (4096, 2.0, 50, 2, 64),
                                  (10000, 1.1, 1e8, 1000, 4)])
def test_query_equals_bruteforce_kmajority(case):
    """The method's final answer is exact (no false negatives P:115/P:171 + verification P:42):
    it equals the textbook k-majority set {x : f(x) > n/k} from a sort-based histogram."""
    import inputs
    n, s, U, k, P = case
    A = inputs.zipf(n, s, U, seed=n + k)
    pl = oracle.pipeline(A, k, P)
    u, c = np.unique(A, return_counts=True)
    sel = c * k > n
    order = np.lexsort((u[sel], -c[sel].astype(np.int64)))
    assert pl.result[0].tolist() == u[sel][order].astype(np.uint64).tolist()
    assert pl.result[1].tolist() == c[sel][order].tolist()
    # recall 1: every true k-majority item is a candidate
    assert set(u[sel].tolist()) <= set(pl.cand.tolist())


def test_root_guarantees_at_scale():
    """Guarantees at a few-tile scale with exact counts from np.unique (BASELINE north_star:
    f <= f_hat <= f + err, err <= n/k, every f > n/k item reported)."""
    import inputs
    n, k, P = 1 << 20, 200, 16
    A = inputs.zipf(n, 1.1, 1e8, seed=2)
    root = oracle.tree(oracle.leaves(A, k, P, threads=8), k)
    u, c = np.unique(A, return_counts=True)
    f = dict(zip(u.tolist(), c.tolist()))
    assert int(root.counts.sum()) <= n and len(root) == k
    for x, cc, e in root.as_tuples():
        assert f.get(x, 0) <= cc <= f.get(x, 0) + e and e <= n // k
    for x in u[c * k > n].tolist():
        assert x in set(root.items.tolist())


# ---------------------------------------------------------------- f2: on-line stream (R14)
def test_stream_golden(golden):
    """Hand-derived streams E7/E8 (cut into fixed-length leaves, R6 tree over them)."""
    for case in golden["stream"]:
        A = letters(case["stream"])
        k, ll = case["k"], case["leaf_len"]
        lv = [oracle.space_saving(A, k, lo, hi).as_tuples() for lo, hi in oracle.stream_bounds(A.size, ll)]
        assert lv == [S(x) for x in case["leaves"]], case["name"]
        assert oracle.stream_root(A, k, ll).as_tuples() == S(case["root"]), case["name"]


def test_stream_special_cases():
    """leaf_len >= n: one leaf, i.e. sequential SS in canonical order; n = P * leaf_len: exactly
    Algorithm 1's blocks (P:92-95 give r * leaf_len); empty stream: empty summary."""
    import inputs
    A = inputs.zipf(5000, 1.1, 300, seed=3)
    u, c = np.unique(A, return_counts=True)
    order = np.lexsort((u, -c.astype(np.int64)))
    # k >= distinct: the single leaf is the exact histogram (textbook unique)
    assert oracle.stream_root(A, 400, 10_000).as_tuples() == [(int(u[i]), int(c[i]), 0) for i in order]
    for ll in (625, 1000, 5000):
        assert oracle.stream_bounds(A.size, ll) == oracle.bounds(A.size, A.size // ll)
    assert oracle.stream_bounds(10, 4) == [(0, 4), (4, 8), (8, 10)]
    assert len(oracle.stream_root(A[:0], 10, 7)) == 0


@pytest.mark.parametrize("n,ll,k", [(9999, 700, 20), (20000, 1024, 50), (4097, 13, 5)])
def test_stream_guarantees(n, ll, k):
    """The paper's guarantees hold for the on-line summary of a ragged stream (exact counts from
    np.unique): f <= f_hat <= f + err, err <= n/k, sum of counts <= n, every f > n/k reported."""
    import inputs
    A = inputs.zipf(n, 1.1, 1e5, seed=n)
    R = oracle.stream_root(A, k, ll)
    f = hist(A)
    assert int(R.counts.sum()) <= n and len(R) <= k
    for x, cc, e in R.as_tuples():
        assert f.get(x, 0) <= cc <= f.get(x, 0) + e and e <= n // k
    assert {x for x, v in f.items() if v * k > n} <= set(R.items.tolist())


# ---------------------------------------------------------------- f3: accuracy metrics
def test_kmajority_bruteforce():
    """The k-majority definition by counting in a plain loop on small streams."""
    rng = np.random.default_rng(3)
    for trial in range(40):
        n = int(rng.integers(0, 300))
        k = int(rng.integers(2, 12))
        A = rng.integers(0, int(rng.integers(1, 20)), size=n).astype(np.uint32)
        cnt = {}
        for x in A.tolist():
            cnt[x] = cnt.get(x, 0) + 1
        want = sorted([(x, c) for x, c in cnt.items() if c * k > n], key=lambda t: (-t[1], t[0]))
        u, c = oracle.kmajority(A, k)
        assert list(zip(u.tolist(), c.tolist())) == want


def test_accuracy_spec_examples():
    """S:341 (reported {a,b}, T {a} -> precision 0.5, recall 1), S:347 (ARE 0), S:348 (ARE of
    [(a,11),(b,20)] against {a:10, b:20} = mean(0.1, 0) = 0.05)."""
    r = oracle.accuracy([1, 2], [6, 4], {1: 5, 2: 2}, n=10, k=3)  # threshold 4: T = {a}
    assert (r["precision"], r["recall"], r["n_true"]) == (0.5, 1.0, 1)
    r = oracle.accuracy([1], [10], {1: 10}, n=10, k=2)
    assert r["are_reported"] == 0.0 and r["are_true"] == 0.0
    r = oracle.accuracy([1, 2], [11, 20], {1: 10, 2: 20}, n=30, k=2)
    assert abs(r["are_reported"] - 0.05) < 1e-15
    # nothing reported, nothing true: SPEC's conventions
    r = oracle.accuracy([], [], {1: 1, 2: 1}, n=2, k=2)
    assert (r["precision"], r["recall"], r["are_reported"]) == (1.0, 1.0, 0.0)
    # a true item not reported counts relative error 1 in the T population
    r = oracle.accuracy([2], [3], {1: 6, 2: 3}, n=9, k=3)  # threshold 4: T = {a}
    assert (r["recall"], r["are_true"], r["precision"]) == (0.0, 1.0, 0.0)


def test_accuracy_exact_case_is_zero():
    """single worker with k >= distinct -> all counts exact -> ARE 0, precision 1."""
    import inputs
    A = inputs.zipf(3000, 1.3, 200, seed=8)
    k = 250
    root = oracle.tree(oracle.leaves(A, k, 1), k)
    cand = oracle.prune(root, A.size, k)
    r = oracle.accuracy(cand, root.counts[:cand.size], hist(A), A.size, k)
    assert r["are_reported"] == 0.0 and r["precision"] == 1.0 and r["recall"] == 1.0


# ---------------------------------------------------------------- f4: hybrid tree shape
def test_hybrid_bounds():
    """Alg. 1's formulas among processes, then among each process's threads."""
    assert oracle.hybrid_bounds(10, 2, 2) == [(0, 2), (2, 5), (5, 7), (7, 10)]  # by hand
    assert oracle.hybrid_bounds(7, 3, 2) == [(0, 1), (1, 2), (2, 3), (3, 4), (4, 5), (5, 7)]
    for n in (0, 1, 5, 97, 1000):
        for Pp in (1, 2, 3, 7):
            for T in (1, 2, 3, 5):
                b = oracle.hybrid_bounds(n, Pp, T)
                assert len(b) == Pp * T and b[0][0] == 0 and b[-1][1] == n
                assert all(b[i][1] == b[i + 1][0] for i in range(len(b) - 1))
        assert oracle.hybrid_bounds(n, 1, 6) == oracle.bounds(n, 6)
        assert oracle.hybrid_bounds(n, 6, 1) == oracle.bounds(n, 6)


def test_hybrid_degenerate_cases():
    """(1, T) is Algorithm 1 with T workers, (Pp, 1) with Pp workers; with T a power
    of two and Pp*T | n the process roots are nodes of the flat tree (R6), so the roots agree."""
    import inputs
    A = inputs.zipf(6000, 1.1, 3000, seed=4)
    k = 20
    flat = lambda P: oracle.tree(oracle.leaves(A, k, P), k).as_tuples()
    assert oracle.hybrid(A, k, 1, 6)[1].as_tuples() == flat(6)
    assert oracle.hybrid(A, k, 6, 1)[1].as_tuples() == flat(6)
    assert oracle.hybrid(A, k, 3, 4)[1].as_tuples() == flat(12)
    assert oracle.hybrid(A, k, 5, 8)[1].as_tuples() == flat(40)
    # T = 3 is another tree shape: ((0,1),2) per process instead of R6 over 6 leaves
    assert oracle.hybrid(A, k, 2, 3)[1].as_tuples() != flat(6)


def test_hybrid_recall_grid():
    """a 60-item stream over 5 items, k = 3: every item with f > 20 is reported for
    every (Pp, T) grid (no false negatives)."""
    rng = np.random.default_rng(60)
    A = rng.choice(np.arange(1, 6, dtype=np.uint64), size=60, p=[0.4, 0.3, 0.1, 0.1, 0.1])
    f = hist(A)
    heavy = {x for x, c in f.items() if c * 3 > 60}
    assert heavy
    for Pp in range(1, 6):
        for T in range(1, 6):
            root = oracle.hybrid(A, 3, Pp, T)[1]
            assert heavy <= set(oracle.prune(root, 60, 3).tolist()), (Pp, T)


def _all_shapes(lo, hi):
    if hi - lo == 1:
        yield lo
        return
    for mid in range(lo + 1, hi):
        for left in _all_shapes(lo, mid):
            for right in _all_shapes(mid, hi):
                yield (left, right)


def test_reduction_order_robustness():
    """every binary tree shape over <= 5 worker summaries keeps the guarantees: recall 1,
    f <= f_hat <= f + err, err <= n/k (COMBINE is commutative, so ordered shapes cover all)."""
    import inputs
    for seed in range(6):
        A = inputs.zipf(400, 1.2, 40, seed=seed)
        k = 4
        f = hist(A)
        heavy = {x for x, c in f.items() if c * k > A.size}
        for P in range(1, 6):
            lv = oracle.leaves(A, k, P)

            def red(t):
                return lv[t] if isinstance(t, int) else oracle.combine(red(t[0]), red(t[1]), k)
            for shape in _all_shapes(0, P):
                root = red(shape)
                assert heavy <= set(oracle.prune(root, A.size, k).tolist())
                for x, c, e in root.as_tuples():
                    assert f.get(x, 0) <= c <= f.get(x, 0) + e and e <= A.size // k


def test_stream_binary_counter_equals_fixed_tree():
    """The identity the GPU stream is built on: the R6 tree over c leaves is
    the right fold COMBINE(S_1, COMBINE(S_2, ... COMBINE(S_t, last))) over the complete subtrees
    of the binary decomposition of c, built as a binary counter with carries. Checked against the
    oracle's level-by-level tree for every c <= 40 (the fold itself uses only oracle.combine)."""
    import inputs
    k = 3
    A = inputs.zipf(40 * 7, 1.1, 12, seed=5)
    leaves = [oracle.space_saving(A, k, lo, hi) for lo, hi in oracle.stream_bounds(A.size, 7)]
    for c in range(1, 41):
        stack = {}  # level -> root of a complete subtree (binary counter)
        for p in range(c - 1):  # push leaves 0..c-2 with carries; leaf c-1 plays the partial leaf
            node, j = leaves[p], 0
            while j in stack:
                node = oracle.combine(stack.pop(j), node, k)
                j += 1
            stack[j] = node
        acc = leaves[c - 1]
        for j in sorted(stack):  # right fold, lowest level first
            acc = oracle.combine(stack[j], acc, k)
        if c == 1:
            acc = oracle.canonical(acc)
        assert acc.as_tuples() == oracle.tree(leaves[:c], k).as_tuples(), c


# ---------------------------------------------------------------- full-size helpers (threaded)
@pytest.mark.parametrize("n,P,kb", [(50_000, 1, 4), (50_000, 2, 4), (50_000, 7, 8), (30_001, 13, 4),
                                    (5, 9, 4), (0, 3, 4), (70_000, 64, 8)])
def test_padded_leaves_and_parallel_tree_equal_the_sequential_ones(n, P, kb):
    """leaves_padded / tree_padded (the threaded forms the full-size GPU parity tests use) equal
    leaves / orc_tree computed one COMBINE at a time, for odd level sizes (the carried node, R6),
    empty leaves (P > n) and both key widths. Pinned to the sequential oracle, itself pinned above
    by the worked examples, closed forms and exhaustive guarantees."""
    rng = np.random.default_rng(n + P)
    dt = np.uint32 if kb == 4 else np.uint64
    A = (rng.zipf(1.3, size=n) % 5000).astype(dt) * dt(2654435761 & 0xFFFFFFFF)
    for k in (2, 17, 100):
        ref = oracle.leaves(A, k, P)
        it, c, e, sz = oracle.leaves_padded(A, k, P, threads=4)
        assert sz.tolist() == [len(s) for s in ref]
        for r in range(P):
            got = oracle.Summary(it[r, :sz[r]], c[r, :sz[r]], e[r, :sz[r]])
            assert got.as_tuples() == ref[r].as_tuples()
            assert not it[r, sz[r]:].any() and not c[r, sz[r]:].any()
        assert oracle.tree_padded(it, c, e, sz, k, threads=4).as_tuples() == \
            oracle.tree(ref, k).as_tuples()
