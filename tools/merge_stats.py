#!/usr/bin/env python
"""Per-phase SM cycles of the COMBINE kernel per tree level (debug build with -DPSS_MSTATS).

  python tools/merge_stats.py [--workload H]

Builds a separate libpss_mstats.so (never loaded by the package), summarizes the workload, runs
the merge tree and prints, per level (by ceil(log2(#nodes))), the mean cycles per COMBINE of:
load+minima, hash build, match S1, update S2, live count, count-digit passes, item-digit passes,
write.
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
    args = ap.parse_args()
    import torch

    import importlib.util

    import inputs
    spec = importlib.util.spec_from_file_location(
        "_pss_build", os.path.join(ROOT, "paper_1606_04669_b200", "_build.py"))
    _build = importlib.util.module_from_spec(spec)
    spec.loader.exec_module(_build)

    out = os.path.join("/tmp", "libpss_mstats.so")
    subprocess.check_call(["nvcc", *_build.NVCC_FLAGS, "-DPSS_MSTATS", "-I",
                           os.path.join(ROOT, "include"), "-o", out, *_build.sources()])
    os.environ["PSS_LIB"] = out
    import paper_1606_04669_b200 as pss
    lib = ctypes.CDLL(out)
    w = inputs.WORKLOADS[args.workload]
    A = torch.from_numpy(w.generate(w.n)).cuda()
    leaves = pss.pss_summarize(A, w.k, w.P)
    pss.pss_merge(leaves)
    torch.cuda.synchronize()
    st = (ctypes.c_ulonglong * 256)()
    lib.pss_debug_mstats(st, 1)
    pss.pss_merge(leaves)
    torch.cuda.synchronize()
    lib.pss_debug_mstats(st, 0)
    names = ["load+min", "hash", "match", "upd S2", "-", "live", "cnt pass", "key pass", "write"]
    print("lvl  combines  " + "  ".join(f"{n:>9s}" for n in names) + "      total")
    for lv in range(16):
        row = st[lv * 16:(lv + 1) * 16]
        c = row[15]
        if not c:
            continue
        ph = [row[i] / c for i in range(9)]
        print(f"{lv:3d} {c:9d}  " + "  ".join(f"{v:9.0f}" for v in ph) + f"  {sum(ph):9.0f}")


if __name__ == "__main__":
    main()
