#!/usr/bin/env python
"""Run the hot path (bench.py's step: pss_summarize_merge -> prune -> verify -> report) a few
times on a BASELINE workload, for profilers (ncu captures the kernels of the last steps).

  python tools/one_step.py [--workload H] [--steps 2]
"""
import argparse
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--workload", default="H")
    ap.add_argument("--steps", type=int, default=2)
    a = ap.parse_args()
    import torch

    import inputs
    import paper_1606_04669_b200 as pss
    from paper_1606_04669_b200 import dist as pdist

    w = inputs.WORKLOADS[a.workload]
    A = torch.from_numpy(w.generate()).cuda()
    kt = pss.KEY_U32 if w.key_bytes == 4 else pss.KEY_U64
    r = pdist.Runner(w.n, w.k, w.P, kt, "cuda:0")
    for _ in range(a.steps):
        r.step(A)
    torch.cuda.synchronize()
    print("ok", a.workload, int(r.result()[2].item()))


if __name__ == "__main__":
    main()
