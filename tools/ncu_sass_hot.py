#!/usr/bin/env python
"""Hottest SASS instructions of an ncu report by warp-stall samples, with their neighbours.

  python tools/ncu_sass_hot.py gpurun_out/prof.ncu-rep [--top 25] [--ctx 3]
"""
import argparse
import csv
import io
import subprocess


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("report")
    ap.add_argument("--top", type=int, default=25)
    ap.add_argument("--ctx", type=int, default=0)
    a = ap.parse_args()
    out = subprocess.run(["ncu", "-i", a.report, "--page", "source", "--csv", "--print-source",
                          "sass"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    hdr = next(r for r in rows if r and r[0] == "Address")
    body = [r for r in rows[rows.index(hdr) + 1:] if len(r) == len(hdr)]
    iS = hdr.index("Warp Stall Sampling (All Samples)")
    iE = hdr.index("Instructions Executed")
    tot = sum(int(r[iS] or 0) for r in body)
    order = sorted(range(len(body)), key=lambda i: -int(body[i][iS] or 0))[:a.top]
    print(f"total stall samples {tot}")
    for i in order:
        for j in range(max(0, i - a.ctx), min(len(body), i + a.ctx + 1)):
            r = body[j]
            mark = ">>" if j == i else "  "
            print(f"{mark} {j:5d} {int(r[iS] or 0) / tot * 100:5.1f}% {int(r[iE] or 0):>11} "
                  f"{r[1].strip()[:80]}")
        if a.ctx:
            print()


if __name__ == "__main__":
    main()
