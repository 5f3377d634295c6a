#!/usr/bin/env python
"""Event counters of K1's batched rule (debug build with -DPSS_STATS), on a BASELINE workload.

  python tools/k1_stats.py [--workload H] [--n N]

Builds a separate libpss_stats.so (never loaded by the package) and prints, per full-phase step:
slow inserts, rehashes, ambiguous fingerprints, truncations (victims exhausted / hazards), level
rebuilds, and the mean step length.
"""
import argparse
import ctypes
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--workload", default="H")
    ap.add_argument("--n", type=int, default=0)
    ap.add_argument("--k", type=int, default=0)
    ap.add_argument("--P", type=int, default=0)
    args = ap.parse_args()
    import numpy as np
    import torch

    import inputs
    from paper_1606_04669_b200 import _build

    out = os.path.join("/tmp", "libpss_stats.so")
    subprocess.check_call(["nvcc", *_build.NVCC_FLAGS, "-DPSS_STATS", "-I",
                           os.path.join(ROOT, "include"), "-o", out, *_build.sources()])
    lib = ctypes.CDLL(out)
    w = inputs.WORKLOADS[args.workload]
    n = args.n or w.n
    k = args.k or w.k
    P = args.P or (w.P if not args.n else max(1, n // (w.n // w.P)))
    A = torch.from_numpy(w.generate(n)).cuda()
    kt = 0 if w.key_bytes == 4 else 1
    items = torch.empty((P, k), dtype=A.dtype, device="cuda")
    counts = torch.empty((P, k), dtype=torch.uint32, device="cuda")
    errs = torch.empty((P, k), dtype=torch.uint32, device="cuda")
    sizes = torch.empty((P,), dtype=torch.uint32, device="cuda")

    class S(ctypes.Structure):
        _fields_ = [("key_type", ctypes.c_int32), ("k", ctypes.c_uint32), ("count", ctypes.c_uint32),
                    ("items", ctypes.c_void_p), ("counts", ctypes.c_void_p), ("errs", ctypes.c_void_p),
                    ("sizes", ctypes.c_void_p)]
    lib.pss_workspace_bytes.restype = ctypes.c_size_t
    lib.pss_workspace_bytes.argtypes = [ctypes.c_int, ctypes.c_uint64, ctypes.c_uint32,
                                        ctypes.c_uint32, ctypes.c_int]
    wsb = lib.pss_workspace_bytes(0, n, k, P, kt)
    ws = torch.empty((wsb,), dtype=torch.uint8, device="cuda")
    st = (ctypes.c_ulonglong * 16)()
    lib.pss_debug_stats(st, 1)
    leaves = S(kt, k, P, items.data_ptr(), counts.data_ptr(), errs.data_ptr(), sizes.data_ptr())
    lib.pss_summarize.argtypes = [ctypes.c_void_p, ctypes.c_uint64, ctypes.c_int, ctypes.c_uint32,
                                  ctypes.c_uint32, ctypes.POINTER(S), ctypes.c_void_p,
                                  ctypes.c_size_t, ctypes.c_void_p]
    rc = lib.pss_summarize(A.data_ptr(), n, kt, k, P, ctypes.byref(leaves), ws.data_ptr(), wsb, None)
    torch.cuda.synchronize()
    assert rc == 0, rc
    lib.pss_debug_stats(st, 0)
    s = list(st)
    names = ["full_steps", "items", "slow_insert_lanes", "rehash", "amb_steps", "trunc_victims",
             "trunc_hazard", "new_level", "fill_steps", "evictions", "no_free_entry_lanes",
             "ph1_cycles", "ph2_cycles", "ph3_cycles", "classify_windows",
             "pinned_items"]
    full = max(1, s[0])
    print(f"workload {args.workload} n={n} k={k} P={P}")
    for i, nm in enumerate(names):
        print(f"  {nm:22s} {s[i]:14d}  per full step {s[i] / full:9.4f}")
    print(f"  mean items per step {s[1] / max(1, s[0] + s[8]):.2f}; evictions/item {s[9] / n:.4f}")


if __name__ == "__main__":
    main()
