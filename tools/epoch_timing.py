#!/usr/bin/env python
"""Per-stage cycles of K1e at H (build with -DPSS_EP_TIMING, load with PSS_LIB, PSS_EPOCH=1)."""
import ctypes
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    import torch

    import inputs
    import paper_1606_04669_b200 as pss
    lib = pss._lib
    lib.pss_debug_epoch_timing.argtypes = [ctypes.c_void_p, ctypes.c_int]
    w = inputs.WORKLOADS[os.environ.get("EP_WORKLOAD", "H")]
    A = torch.from_numpy(w.generate()).cuda()
    buf = (ctypes.c_ulonglong * 16)()
    pss.pss_summarize(A, w.k, w.P)
    torch.cuda.synchronize()
    lib.pss_debug_epoch_timing(buf, 1)
    pss.pss_summarize(A, w.k, w.P)
    torch.cuda.synchronize()
    lib.pss_debug_epoch_timing(buf, 1)
    names = ["(window bookkeeping)", "P1 barrier A wait", "P2 events", "P3 scan+apply",
             "E0 barrier wait", "E1 resolve", "E2 misses", "E3 pops", "E4 rebuild",
             "P1 lookup", "P1 V/U claim (tid 0)"]
    tot = sum(buf[i] for i in range(11))
    for i, nm in enumerate(names):
        print(f"{nm:24s} {buf[i] / 1e9:8.3f} Gcycles  {100 * buf[i] / tot:5.1f}%")
    print(f"claim-loop trips of warp 0 per pass: {buf[11] / max(buf[12], 1):.2f} ({buf[12]} passes)")


if __name__ == "__main__":
    main()
