#!/usr/bin/env python
"""Dump the SASS of the first kernel in an ncu report with per-instruction execution counts and
stall samples (optionally only instructions executed at least --min times).

  python tools/ncu_sass_dump.py gpurun_out/prof.ncu-rep [--min 1e6] [--per 16.5e6]
"""
import argparse
import csv
import io
import subprocess


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("report")
    ap.add_argument("--min", type=float, default=0)
    ap.add_argument("--per", type=float, default=1, help="divide executions by this (e.g. steps)")
    a = ap.parse_args()
    out = subprocess.run(["ncu", "-i", a.report, "--page", "source", "--csv", "--print-source", "sass"],
                         capture_output=True, text=True).stdout
    hdr = None
    tot = 0.0
    for rec in csv.reader(io.StringIO(out)):
        if not rec:
            continue
        if rec[0] == "Address":
            hdr = rec
            continue
        if hdr is None or len(rec) < 6:
            continue
        d = dict(zip(hdr, rec))
        try:
            ex = int(d["Instructions Executed"] or 0)
            smp = int(d["Warp Stall Sampling (All Samples)"] or 0)
        except (ValueError, KeyError):
            continue
        if ex < a.min:
            continue
        tot += ex / a.per
        print(f"{d['Address'][-5:]} {ex / a.per:8.3f} {smp:6d}  {d['Source'].strip()}")
    print(f"total {tot:.1f}")


if __name__ == "__main__":
    main()
