#!/usr/bin/env python
"""Time pss_merge alone and pss_summarize_merge (tree overlapping K1) on a BASELINE workload.

  python tools/merge_time.py [--workload H] [--reps 5]

Environment hooks of libpss.so apply (PSS_LIB for experiment builds, PSS_NO_OVERLAP)."""
import argparse
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--workload", default="H")
    ap.add_argument("--reps", type=int, default=5)
    a = ap.parse_args()
    import torch

    import inputs
    import paper_1606_04669_b200 as pss

    w = inputs.WORKLOADS[a.workload]
    A = torch.from_numpy(w.generate()).cuda()
    leaves, root = pss.pss_summarize_merge(A, w.k, w.P)

    def timed(fn):
        ts = []
        for _ in range(a.reps + 1):
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            fn()
            e1.record()
            torch.cuda.synchronize()
            ts.append(e0.elapsed_time(e1))
        return min(ts[1:])
    t_m = timed(lambda: pss.pss_merge(leaves, out=root))
    t_s = timed(lambda: pss.pss_summarize(A, w.k, w.P, out=leaves))
    t_sm = timed(lambda: pss.pss_summarize_merge(A, w.k, w.P, leaves=leaves, root=root))
    print(f"{a.workload} lib={os.environ.get('PSS_LIB', 'default')}: merge {t_m:.3f} ms, "
          f"summarize {t_s:.3f} ms, summarize_merge {t_sm:.3f} ms (tail {t_sm - t_s:.3f})")


if __name__ == "__main__":
    main()
