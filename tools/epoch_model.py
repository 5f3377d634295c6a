"""Host model of K1e's epoch formulation of Space Saving (design check, not the oracle).

Sequential Space Saving with the R1/R2 tie-breaks, rewritten per *epoch*: an epoch
starts when a new minimum level m is formed, B = slots with count m in slot order (members
r = 0..b-1; the fill phase is the epoch m = 0 whose members are the free slots). During the epoch
the only keys that can leave the summary are members, and every *event* -- the first occurrence
in the epoch of a key that is unmonitored (U) or a member (V) at the epoch start -- consumes
exactly one member (a miss pops the lowest unconsumed member, a V hit consumes its own member), so
the epoch ends after exactly b events, at level m + 1.

Which V events are hits (set H) follows in closed form: with v = event index (time order) and
r = member index (slot order), V(r) at v is a hit iff  v - r <= |{y in H : r_y > r, v_y < v}|.
The j-th miss (time order) pops the j-th member not in H (slot order).

This module runs that formulation and is compared with the oracle's sequential Space Saving in
`python tools/epoch_model.py` (random small inputs + a few H blocks), and prints per-epoch
statistics that size K1e's buffers.
"""
from __future__ import annotations

import sys
from collections import defaultdict

import numpy as np


def resolve_H(vpts):
    """vpts: list of (v, r) in time order. Returns list of bools (hit) in the same order."""
    hit = []
    H = []  # (v, r) of hits so far
    for v, r in vpts:
        cnt = sum(1 for (vy, ry) in H if ry > r and vy < v)
        h = v - r <= cnt
        hit.append(h)
        if h:
            H.append((v, r))
    return hit


def resolve_H_bounds(vpts):
    """The parallel scheme: trivial bounds, then exact counts for the near-diagonal points.
    Returns (hit list, number undecided after the trivial bounds)."""
    n = len(vpts)
    # number of V points with larger r (any time) and earlier v (any r)
    rs = np.array([r for _, r in vpts], dtype=np.int64)
    state = [None] * n
    und = 0
    for i, (v, r) in enumerate(vpts):
        d = v - r
        nlarger = int((rs > r).sum())
        ub = min(i, nlarger)
        if d <= 0:
            state[i] = True
        elif d > ub:
            state[i] = False
        else:
            und += 1
    # fixpoint with exact counts among decided points (Jacobi)
    it = 0
    while any(s is None for s in state):
        it += 1
        new = list(state)
        for i, (v, r) in enumerate(vpts):
            if state[i] is not None:
                continue
            lo = hi = 0
            for j in range(i):
                vy, ry = vpts[j]
                if ry > r and vy < v:
                    if state[j] is True:
                        lo += 1
                        hi += 1
                    elif state[j] is None:
                        hi += 1
            d = v - r
            if d <= lo:
                new[i] = True
            elif d > hi:
                new[i] = False
        state = new
    return state, und, it


def epoch_ss(A, k, stats=None, snaps=None):
    L = len(A)
    keys = [None] * k
    cnt = [0] * k
    err = [0] * k
    m = 0
    members = list(range(k))  # fill epoch: the free slots
    index = {}  # key -> slot, the epoch-start state
    t = 0
    filled = 0
    while t < L:
        b = len(members)
        memidx = {s: i for i, s in enumerate(members)}
        utab = {}  # key -> [event index, occ]
        vseen = {}  # member index -> event index
        occ = defaultdict(int)  # slot -> occurrences in the epoch
        events = []  # ('U', key) / ('V', member index)
        tt = t
        while tt < L and len(events) < b:
            x = int(A[tt])
            s = index.get(x)
            if s is not None:
                if s in memidx and memidx[s] not in vseen:
                    vseen[memidx[s]] = len(events)
                    events.append(('V', memidx[s]))
                occ[s] += 1
            else:
                if x not in utab:
                    utab[x] = [len(events), 0]
                    events.append(('U', x))
                utab[x][1] += 1
            tt += 1
        full = len(events) == b
        vpts = [(i, e[1]) for i, e in enumerate(events) if e[0] == 'V']
        hit = resolve_H(vpts)
        if stats is not None:
            hb, und, it = resolve_H_bounds(vpts)
            assert hb == hit
            stats['epochs'] += 1
            stats['b'] += b
            stats['items'] += tt - t
            stats['V'] += len(vpts)
            stats['Vhit'] += sum(hit)
            stats['und'] += und
            stats['iters'] = max(stats['iters'], it)
        Hset = {r for (v, r), h in zip(vpts, hit) if h}
        misses = [e for i, e in enumerate(events) if not (e[0] == 'V' and e[1] in Hset)]
        pops = [members[r] for r in range(b) if r not in Hset][:len(misses)]
        # read everything first, then write (sources may be popped slots themselves)
        new = []
        for e, s in zip(misses, pops):
            if e[0] == 'U':
                new.append((s, e[1], m + utab[e[1]][1]))
            else:
                src = members[e[1]]
                new.append((s, keys[src], m + occ[src]))
        for s, c in occ.items():
            cnt[s] += c
        for s, x, c in new:
            keys[s] = x
            cnt[s] = c
            err[s] = m
        filled = max(filled, max((s + 1 for s, _, _ in new), default=0))
        index = {keys[s]: s for s in range(filled)}
        if snaps is not None and full:
            snaps.append(dict(m=m, ne=len(events), nv=len(vpts), nh=len(Hset),
                              keys=list(keys), cnt=list(cnt), err=list(err)))
        if full:
            nm = min(cnt)
            assert nm == m + 1, (nm, m)
            m = nm
            members = [s for s in range(k) if cnt[s] == m]
        t = tt
    return [(keys[s], cnt[s], err[s]) for s in range(filled)]


def main():
    sys.path.insert(0, '.')
    import oracle
    import inputs
    rng = np.random.default_rng(1)
    for trial in range(3000):
        k = int(rng.integers(1, 9))
        n = int(rng.integers(0, 60))
        U = int(rng.integers(1, 12))
        A = rng.integers(0, U, n).astype(np.uint32)
        got = epoch_ss(A, k)
        want = oracle.space_saving(A, k).as_tuples()
        assert got == want, (trial, k, A.tolist(), got, want)
    print("random small: ok")
    for trial in range(200):
        k = int(rng.integers(5, 60))
        s = float(rng.choice([0.5, 0.8, 1.1, 1.5]))
        A = inputs.zipf(int(rng.integers(100, 5000)), s, 2000.0, int(rng.integers(1, 1000)))
        got = epoch_ss(A, k)
        want = oracle.space_saving(A, k).as_tuples()
        assert got == want, (trial, k)
    print("random zipf: ok")
    A = inputs.zipf(1 << 18, 1.1, 1e8, 2)
    for r in range(2):
        blk = A[r * 65536:(r + 1) * 65536]
        st = defaultdict(int)
        got = epoch_ss(blk, 1000, st)
        want = oracle.space_saving(blk, 1000).as_tuples()
        assert got == want
        e = st['epochs']
        print(f"H block {r}: epochs {e}, items/epoch {st['items']/e:.0f}, b {st['b']/e:.0f}, "
              f"V/epoch {st['V']/e:.1f}, Vhit {st['Vhit']/e:.1f}, undecided {st['und']/e:.2f}, "
              f"max iters {st['iters']}")


if __name__ == "__main__":
    main()
