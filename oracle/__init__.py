"""CPU oracle for Parallel Space Saving -- TEST INFRASTRUCTURE ONLY.

Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s cpu_baseline / ``--impl reference``
legs may import this package. The product path (``paper_1606_04669_b200``) never does.

A thin ctypes wrapper over ``oracle/pss_oracle.c`` (plain C, compiled with gcc). Every function
cites the passage of PAPER.md it follows; readings R1..R12 are listed in DESIGN.md. Pins live in
``tests/test_oracle_pins.py``.
"""
from __future__ import annotations

import ctypes
import os
import subprocess
from concurrent.futures import ThreadPoolExecutor
from typing import NamedTuple, Sequence

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_SRC = os.path.join(_HERE, "pss_oracle.c")
_LIB = os.path.join(_HERE, "liboracle.so")
_lib = None

_u64p = ctypes.POINTER(ctypes.c_uint64)
_u32p = ctypes.POINTER(ctypes.c_uint32)


def build(force: bool = False) -> str:
    """Compile the oracle with gcc (plain C, -O2)."""
    if force or not os.path.exists(_LIB) or os.path.getmtime(_LIB) < os.path.getmtime(_SRC):
        tmp = _LIB + f".tmp{os.getpid()}"
        subprocess.check_call(["gcc", "-O2", "-fPIC", "-shared", "-o", tmp, _SRC])
        os.replace(tmp, _LIB)
    return _LIB


def _load():
    global _lib
    if _lib is None:
        build()
        L = ctypes.CDLL(_LIB)
        vp, u64, u32, i32 = ctypes.c_void_p, ctypes.c_uint64, ctypes.c_uint32, ctypes.c_int
        L.orc_bounds.argtypes = [u64, u32, u32, _u64p, _u64p]
        L.orc_bounds.restype = None
        L.orc_space_saving.argtypes = [vp, i32, u64, u64, u32, vp, vp, vp]
        L.orc_space_saving.restype = u32
        L.orc_min.argtypes = [vp, u32, u32]
        L.orc_min.restype = u64
        L.orc_canonical.argtypes = [vp, vp, vp, u32]
        L.orc_canonical.restype = None
        L.orc_combine.argtypes = [vp, vp, vp, u32, vp, vp, vp, u32, u32, vp, vp, vp]
        L.orc_combine.restype = u32
        L.orc_tree.argtypes = [vp, vp, vp, vp, u32, u32, vp, vp, vp]
        L.orc_tree.restype = u32
        L.orc_threshold.argtypes = [u64, u32]
        L.orc_threshold.restype = u64
        L.orc_prune.argtypes = [vp, vp, u32, u64, u32, vp]
        L.orc_prune.restype = u32
        L.orc_verify.argtypes = [vp, i32, u64, vp, u32, vp]
        L.orc_verify.restype = None
        L.orc_result.argtypes = [vp, vp, u32, u64, u32, vp, vp]
        L.orc_result.restype = u32
        _lib = L
    return _lib


class Summary(NamedTuple):
    """A stream summary: counters (item, count, err), uint64 arrays of equal length."""
    items: np.ndarray
    counts: np.ndarray
    errs: np.ndarray

    def __len__(self):
        return int(self.items.size)

    def as_tuples(self):
        return [(int(a), int(b), int(c)) for a, b, c in zip(self.items, self.counts, self.errs)]


def empty_summary() -> Summary:
    z = np.zeros(0, np.uint64)
    return Summary(z, z.copy(), z.copy())


def _ptr(a: np.ndarray):
    return a.ctypes.data if a.size else None


def _keys(A) -> tuple[np.ndarray, int]:
    A = np.ascontiguousarray(A)
    if A.dtype == np.uint32:
        return A, 4
    if A.dtype == np.uint64:
        return A, 8
    raise TypeError(f"keys must be uint32 or uint64, got {A.dtype}")


def _summary(s) -> Summary:
    if isinstance(s, Summary):
        return Summary(*(np.ascontiguousarray(x, dtype=np.uint64) for x in s))
    items, counts, errs = zip(*s) if len(s) else ((), (), ())
    return Summary(np.array(items, np.uint64), np.array(counts, np.uint64), np.array(errs, np.uint64))


def bounds(n: int, P: int) -> list[tuple[int, int]]:
    """Algorithm 1 lines 3-4 as half-open [lo, hi) ranges, r = 0..P-1."""
    L = _load()
    lo, hi = ctypes.c_uint64(), ctypes.c_uint64()
    out = []
    for r in range(P):
        L.orc_bounds(n, P, r, ctypes.byref(lo), ctypes.byref(hi))
        out.append((lo.value, hi.value))
    return out


def space_saving(A, k: int, lo: int = 0, hi: int | None = None) -> Summary:
    """Sequential Space Saving over A[lo:hi] (Alg. 1 line 5), slot order."""
    A, kb = _keys(A)
    hi = A.size if hi is None else hi
    it, c, e = (np.zeros(max(k, 1), np.uint64) for _ in range(3))
    size = _load().orc_space_saving(_ptr(A), kb, lo, hi, k, it.ctypes.data, c.ctypes.data,
                                    e.ctypes.data)
    return Summary(it[:size].copy(), c[:size].copy(), e[:size].copy())


def leaves(A, k: int, P: int, which: Sequence[int] | None = None, threads: int = 1) -> list[Summary]:
    """Leaf summaries of Algorithm 1 (one Space Saving per block); `which` selects partitions."""
    A, _ = _keys(A)
    rng = bounds(A.size, P)
    idx = range(P) if which is None else which
    if threads <= 1:
        return [space_saving(A, k, *rng[r]) for r in idx]
    with ThreadPoolExecutor(threads) as ex:
        return list(ex.map(lambda r: space_saving(A, k, *rng[r]), idx))


def leaves_padded(A, k: int, P: int, threads: int = 1):
    """All P leaf summaries of Algorithm 1 (Space Saving per block) as padded
    arrays: items/counts/errs [P, k] (uint64, zero beyond each leaf's size) and sizes [P] (uint32).
    The same ``orc_space_saving`` as ``leaves``, written straight into each leaf's row; leaves
    are independent, so they run on `threads` host threads (ctypes releases the GIL)."""
    A, kb = _keys(A)
    L = _load()
    rng = bounds(A.size, P)
    items, counts, errs = (np.zeros((P, max(k, 1)), np.uint64) for _ in range(3))
    sizes = np.zeros(P, np.uint32)
    base = A.ctypes.data if A.size else None
    row = max(k, 1) * 8

    def one(r):
        lo, hi = rng[r]
        sizes[r] = L.orc_space_saving(base, kb, lo, hi, k, items.ctypes.data + r * row,
                                      counts.ctypes.data + r * row, errs.ctypes.data + r * row)

    if threads <= 1:
        for r in range(P):
            one(r)
    else:
        with ThreadPoolExecutor(threads) as ex:
            list(ex.map(one, range(P)))
    return items, counts, errs, sizes


def tree_padded(items, counts, errs, sizes, k: int, threads: int = 1) -> Summary:
    """ParallelReduction with COMBINE over the fixed binary tree (Alg. 1 line 7; reading R6) on
    padded [P, k] leaves, level by level exactly as ``orc_tree``: nodes (2i, 2i+1) of a level are
    merged by ``orc_combine`` (Algorithm 2), an odd last node is carried up unchanged, the root is
    put in canonical order (R5). The COMBINEs of one level are independent and run on `threads`
    host threads; the tree's shape and every COMBINE's arithmetic are ``orc_tree``'s."""
    L = _load()
    P = sizes.size
    if P == 0:
        return empty_summary()
    ci, cc, ce = (np.ascontiguousarray(a, dtype=np.uint64) for a in (items, counts, errs))
    cs = np.ascontiguousarray(sizes, dtype=np.uint32).copy()
    kk = ci.shape[1]
    row = kk * 8
    while cs.size > 1:
        cur = cs.size
        nxt = (cur + 1) // 2
        ni, nn, ne = (np.zeros((nxt, kk), np.uint64) for _ in range(3))
        ns = np.zeros(nxt, np.uint32)

        def one(i):
            a, b = 2 * i, 2 * i + 1
            ns[i] = L.orc_combine(ci.ctypes.data + a * row, cc.ctypes.data + a * row,
                                  ce.ctypes.data + a * row, int(cs[a]),
                                  ci.ctypes.data + b * row, cc.ctypes.data + b * row,
                                  ce.ctypes.data + b * row, int(cs[b]), k,
                                  ni.ctypes.data + i * row, nn.ctypes.data + i * row,
                                  ne.ctypes.data + i * row)

        if threads <= 1 or cur // 2 < 2:
            for i in range(cur // 2):
                one(i)
        else:
            with ThreadPoolExecutor(threads) as ex:
                list(ex.map(one, range(cur // 2)))
        if cur & 1:  # odd last node carried up unchanged
            ni[nxt - 1], nn[nxt - 1], ne[nxt - 1] = ci[cur - 1], cc[cur - 1], ce[cur - 1]
            ns[nxt - 1] = cs[cur - 1]
        ci, cc, ce, cs = ni, nn, ne, ns
    n0 = int(cs[0])
    return canonical(Summary(ci[0, :n0].copy(), cc[0, :n0].copy(), ce[0, :n0].copy()))


def min_count(S, k: int) -> int:
    """MIN(S), Alg. 2 lines 2-3, reading R4 (0 unless all k counters used)."""
    S = _summary(S)
    return int(_load().orc_min(_ptr(S.counts), len(S), k))


def canonical(S) -> Summary:
    """Order by (count desc, item asc) -- reading R5."""
    S = Summary(*(x.copy() for x in _summary(S)))
    _load().orc_canonical(_ptr(S.items), _ptr(S.counts), _ptr(S.errs), len(S))
    return S


def combine(S1, S2, k: int) -> Summary:
    """COMBINE, Algorithm 2, canonical output (R3, R4, R5)."""
    S1, S2 = _summary(S1), _summary(S2)
    it, c, e = (np.zeros(max(k, 1), np.uint64) for _ in range(3))
    size = _load().orc_combine(_ptr(S1.items), _ptr(S1.counts), _ptr(S1.errs), len(S1),
                               _ptr(S2.items), _ptr(S2.counts), _ptr(S2.errs), len(S2), k,
                               it.ctypes.data, c.ctypes.data, e.ctypes.data)
    return Summary(it[:size].copy(), c[:size].copy(), e[:size].copy())


def tree(leafs: Sequence, k: int) -> Summary:
    """ParallelReduction with COMBINE over a fixed binary tree (Alg. 1 line 7; reading R6)."""
    P = len(leafs)
    it, c, e = (np.zeros(max(P * k, 1), np.uint64) for _ in range(3))
    sizes = np.zeros(max(P, 1), np.uint32)
    for r, S in enumerate(leafs):
        S = _summary(S)
        n_ = len(S)
        it[r * k:r * k + n_], c[r * k:r * k + n_], e[r * k:r * k + n_] = S.items, S.counts, S.errs
        sizes[r] = n_
    ri, rc, re_ = (np.zeros(max(k, 1), np.uint64) for _ in range(3))
    size = _load().orc_tree(it.ctypes.data, c.ctypes.data, e.ctypes.data, sizes.ctypes.data, P, k,
                            ri.ctypes.data, rc.ctypes.data, re_.ctypes.data)
    return Summary(ri[:size].copy(), rc[:size].copy(), re_[:size].copy())


def threshold(n: int, k: int) -> int:
    """floor(n/k) + 1."""
    return int(_load().orc_threshold(n, k))


def prune(root, n: int, k: int) -> np.ndarray:
    """Pruned(global, n, k) (Alg. 1 lines 8-9): candidates in root order."""
    R = _summary(root)
    cand = np.zeros(max(len(R), 1), np.uint64)
    nc = _load().orc_prune(_ptr(R.items), _ptr(R.counts), len(R), n, k, cand.ctypes.data)
    return cand[:nc].copy()


def verify(A, cand) -> np.ndarray:
    """Exact counts of the candidates over A (off-line setting)."""
    A, kb = _keys(A)
    cand = np.ascontiguousarray(cand, dtype=np.uint64)
    exact = np.zeros(max(cand.size, 1), np.uint64)
    _load().orc_verify(_ptr(A), kb, A.size, _ptr(cand), cand.size, exact.ctypes.data)
    return exact[:cand.size].copy()


def result(cand, exact, n: int, k: int) -> tuple[np.ndarray, np.ndarray]:
    """The k-majority set {(x, f(x)) : f(x) >= floor(n/k)+1} sorted (f desc, x asc)."""
    cand = np.ascontiguousarray(cand, dtype=np.uint64)
    exact = np.ascontiguousarray(exact, dtype=np.uint64)
    oi = np.zeros(max(cand.size, 1), np.uint64)
    oc = np.zeros(max(cand.size, 1), np.uint64)
    ln = _load().orc_result(_ptr(cand), _ptr(exact), cand.size, n, k, oi.ctypes.data,
                            oc.ctypes.data)
    return oi[:ln].copy(), oc[:ln].copy()


class Pipeline(NamedTuple):
    leaves: list
    root: Summary
    cand: np.ndarray
    exact: np.ndarray
    result: tuple


def pipeline(A, k: int, P: int, threads: int = 1) -> Pipeline:
    """ParallelSpaceSaving (Algorithm 1) followed by verification."""
    A, _ = _keys(A)
    L = leaves(A, k, P, threads=threads)
    root = tree(L, k)
    cand = prune(root, A.size, k)
    exact = verify(A, cand)
    return Pipeline(L, root, cand, exact, result(cand, exact, A.size, k))


def stream_bounds(n: int, leaf_len: int) -> list[tuple[int, int]]:
    """Leaves of the on-line stream (reading R14): consecutive blocks of leaf_len
    items, the last one possibly shorter (Alg. 1's blocks, with a fixed length)."""
    return [(lo, min(lo + leaf_len, n)) for lo in range(0, n, leaf_len)]


def stream_root(A, k: int, leaf_len: int) -> Summary:
    """Summary of a stream fed on-line (on-line setting PAPER.md:42): Space Saving
    on every leaf, then the fixed binary tree over the leaves (Alg. 1 line 7, R6),
    computed level by level exactly as ``tree`` does. An empty stream has an empty summary."""
    A, _ = _keys(A)
    if A.size == 0:
        return empty_summary()
    return tree([space_saving(A, k, lo, hi) for lo, hi in stream_bounds(A.size, leaf_len)], k)


def kmajority(A, k: int) -> tuple[np.ndarray, np.ndarray]:
    """The k-majority set by its plain definition {(x, f(x)) : f(x) > n/k}
    from a sort-based exact histogram (np.unique), ordered (f desc, x asc)."""
    A, _ = _keys(A)
    u, c = np.unique(A, return_counts=True)
    sel = c.astype(np.uint64) * np.uint64(k) > np.uint64(A.size)
    u, c = u[sel].astype(np.uint64), c[sel].astype(np.uint64)
    order = np.lexsort((u, -c.astype(np.int64)))
    return u[order], c[order]


def accuracy(reported, fhat, truth: dict, n: int, k: int) -> dict:
    """The paper's accuracy metrics with SPEC's conventions:
    reported items with estimates f_hat; truth = exact frequencies {x: f(x)}. precision =
    |reported & T| / |reported| (1 if nothing is reported), recall = |reported & T| / |T| (1 if T
    is empty), relative error |f - f_hat| / f averaged over the reported items (ARE, 0 if none)
    and over T (an unreported true item counts 1)."""
    thr = n // k + 1
    T = {x for x, f in truth.items() if f >= thr}
    rep = [int(x) for x in reported]
    est = dict(zip(rep, [int(v) for v in fhat]))
    hit = [x for x in rep if x in T]
    rel = {x: abs(truth[x] - est[x]) / truth[x] for x in rep}
    return {"n_reported": len(rep), "n_reported_true": len(hit), "n_true": len(T),
            "precision": len(hit) / len(rep) if rep else 1.0,
            "recall": len(hit) / len(T) if T else 1.0,
            "are_reported": float(np.mean([rel[x] for x in rep])) if rep else 0.0,
            "are_true": float(np.mean([rel[x] if x in est else 1.0 for x in T])) if T else 0.0}


def hybrid_bounds(n: int, Pp: int, T: int) -> list[tuple[int, int]]:
    """The hybrid decomposition: Alg. 1 l.3-4 among Pp
    processes, then again among the T threads of each process; leaf p*T + t."""
    out = []
    for plo, phi in bounds(n, Pp):
        out += [(plo + lo, plo + hi) for lo, hi in bounds(phi - plo, T)]
    return out


def hybrid(A, k: int, Pp: int, T: int) -> tuple[list, Summary]:
    """Leaves of the hybrid decomposition, each process's fixed tree (R6) over its T leaves, then
    the fixed tree over the Pp process roots."""
    A, _ = _keys(A)
    lv = [space_saving(A, k, lo, hi) for lo, hi in hybrid_bounds(A.size, Pp, T)]
    roots = [tree(lv[p * T:(p + 1) * T], k) for p in range(Pp)]
    return lv, tree(roots, k)
