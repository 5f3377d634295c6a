#!/usr/bin/env python
"""Time K1 (pss_summarize) alone on a BASELINE workload for a list of (k, P) settings.

  python tools/k1_time.py --workload H --k 1000 100 --P 8192 [--reps 5]

Environment hooks of libpss.so apply (PSS_DEBUG_SMEM_PAD, PSS_DEBUG_INDEX_LOAD).
"""
import argparse
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--workload", default="H")
    ap.add_argument("--k", type=int, nargs="+", default=[1000])
    ap.add_argument("--P", type=int, nargs="+", default=[0])
    ap.add_argument("--reps", type=int, default=5)
    ap.add_argument("--n", type=int, default=0)
    a = ap.parse_args()
    import torch

    import inputs
    import paper_1606_04669_b200 as pss

    w = inputs.WORKLOADS[a.workload]
    n = a.n or w.n
    A = torch.from_numpy(w.generate(n)).cuda()
    for k in a.k:
        for P in a.P:
            P = P or w.P
            leaves = pss.Summaries.empty(P, k, pss.KEY_U32 if w.key_bytes == 4 else pss.KEY_U64)
            ws = torch.empty((pss.pss_workspace_bytes(pss.OP_SUMMARIZE, n, k, P, leaves.key_type),),
                             dtype=torch.uint8, device="cuda")
            for _ in range(2):
                pss.pss_summarize(A, k, P, out=leaves, workspace=ws)
            ts = []
            for _ in range(a.reps):
                e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                e0.record()
                pss.pss_summarize(A, k, P, out=leaves, workspace=ws)
                e1.record()
                torch.cuda.synchronize()
                ts.append(e0.elapsed_time(e1))
            t = min(ts)
            print(f"{a.workload} n={n} k={k} P={P} pad={os.environ.get('PSS_DEBUG_SMEM_PAD', 0)}: "
                  f"{t:.3f} ms  {n / t / 1e6:.1f} Gitems/s  {n * w.key_bytes / t / 1e6:.1f} GB/s")


if __name__ == "__main__":
    main()
