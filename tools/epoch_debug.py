#!/usr/bin/env python
"""Run K1e (debug build, -DPSS_EP_DEBUG, loaded with PSS_LIB) on small cases and report the first
broken invariant recorded by the kernel, then compare leaves with the oracle.

  tools/variant.sh /tmp/dbg.so -DPSS_EP_DEBUG && PSS_LIB=/tmp/dbg.so python tools/epoch_debug.py
"""
import ctypes
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    import torch

    import inputs
    import oracle
    import paper_1606_04669_b200 as pss
    lib = pss._lib
    buf = (ctypes.c_uint * 16)()
    if hasattr(lib, "pss_debug_epoch"):
        lib.pss_debug_epoch.argtypes = [ctypes.c_void_p, ctypes.c_int]
        dbg = lib.pss_debug_epoch
    else:  # release build: no invariant record
        def dbg(b, reset):
            return 0
    cases = [("zipf", 200_000, 64, 7, 0.9, 1e4), ("zipf", 1 << 17, 1000, 2, 1.1, 1e8),
             ("zipf", 300_001, 500, 5, 1.3, 5e4), ("zipf", 65_536 * 8, 1000, 8, 1.1, 1e8),
             ("zipf", 1 << 24, 1000, 2048, 1.1, 1e8), ("zipf", 1 << 27, 1000, 2048, 1.1, 1e8),
             ("zipf", 1 << 29, 1000, 8192, 1.1, 1e8)]
    sel = [int(c) for c in os.environ.get("EP_CASES", "").split(",") if c]
    reps = int(os.environ.get("EP_REPS", "1"))
    cases = [c for i, c in enumerate(cases) if not sel or i in sel] * reps
    for name, n, k, P, s, U in cases:
        A = inputs.zipf(n, s, U, seed=n + k)
        dbg(buf, 1)
        dA = torch.from_numpy(A).cuda()
        S = pss.pss_summarize(dA, k, P)
        torch.cuda.synchronize()
        dbg(buf, 1)
        names = ["code", "r", "m", "b", "ecount", "a0", "a1", "a2", "eseq", "size"]
        print(name, n, k, P, s, U, {nm: buf[i] for i, nm in enumerate(names)} if buf[0] else "no error",
              "kicked keys", buf[15], "reseeds", buf[14])
        which = list(range(P)) if P <= 64 else list(range(0, P, P // 16))
        ref = oracle.leaves(A, k, P, which=which, threads=8)
        bad = [r for r, lf in zip(which, ref) if S.host(r) != lf.as_tuples()]
        print("  leaves differing:", bad[:10])
        for r in bad[:2]:
            g, w = S.host(r), dict(zip(which, ref))[r].as_tuples()
            i = next((i for i in range(min(len(g), len(w))) if g[i] != w[i]), min(len(g), len(w)))
            print(f"   leaf {r}: sizes {len(g)}/{len(w)}, first diff slot {i}: "
                  f"gpu {g[i] if i < len(g) else None} oracle {w[i] if i < len(w) else None}, "
                  f"ndiff {sum(1 for a, b in zip(g, w) if a != b)}")
            lo, hi = oracle.bounds(n, P)[r]
            blk = torch.from_numpy(A[lo:hi].copy()).cuda()
            nbad = 0
            for _ in range(20):
                T = pss.pss_summarize(blk, k, 1)
                torch.cuda.synchronize()
                nbad += T.host(0) != w
            print(f"   block alone, 20 runs: {nbad} wrong")
            if hasattr(lib, "pss_debug_epoch_dump") and nbad:
                sys.path.insert(0, os.path.join(ROOT, "tools"))
                import epoch_model
                snaps = []
                epoch_model.epoch_ss(A[lo:hi], k, snaps=snaps)
                T = pss.pss_summarize(blk, k, 1)
                torch.cuda.synchronize()
                KM = 2048
                dump = (ctypes.c_uint * (96 * (4 + 2 * KM)))()
                lib.pss_debug_epoch_dump(dump)
                d = np.frombuffer(dump, dtype=np.uint32).reshape(96, 4 + 2 * KM)
                cb = 1
                while (1 << cb) <= hi - lo:
                    cb += 1
                for e, sn in enumerate(snaps):
                    gk = d[e, 4:4 + k]
                    gc = d[e, 4 + KM:4 + KM + k] & ((1 << cb) - 1)
                    ge = d[e, 4 + KM:4 + KM + k] >> cb
                    mk = [(int(sn["keys"][i] or 0), sn["cnt"][i], sn["err"][i]) for i in range(k)]
                    bads = [i for i in range(k) if (int(gk[i]), int(gc[i]), int(ge[i])) != mk[i]]
                    if bads:
                        print(f"   first divergent epoch {e}: gpu m/ne/nvv/nh {d[e, :4].tolist()} "
                              f"model m {sn['m']} ne {sn['ne']} nv {sn['nv']} nh {sn['nh']}; "
                              f"{len(bads)} slots differ, e.g. "
                              f"{[(i, (int(gk[i]), int(gc[i]), int(ge[i])), mk[i]) for i in bads[:4]]}")
                        break
                else:
                    print("   every epoch snapshot equal (divergence after the last full epoch)")
        sys.stdout.flush()


if __name__ == "__main__":
    main()
