#!/usr/bin/env python
"""Summarise an ncu report per CUDA source line: executed instructions and stall samples.

  python tools/ncu_lines.py gpurun_out/prof.ncu-rep [--top 40] [--kernel regex]
"""
import argparse
import csv
import io
import re
import subprocess
import sys


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("report")
    ap.add_argument("--top", type=int, default=40)
    ap.add_argument("--sort", default="samples", choices=["samples", "inst"])
    args = ap.parse_args()
    out = subprocess.run(["ncu", "-i", args.report, "--page", "source", "--csv", "--print-source",
                          "cuda,sass"], capture_output=True, text=True).stdout
    rows = []
    fname = "?"
    hdr = None
    for rec in csv.reader(io.StringIO(out)):
        if not rec:
            continue
        if rec[0] == "File Path":
            fname = rec[1].split("/")[-1]
            continue
        if rec[0] == "Line No":
            hdr = rec
            continue
        if hdr is None or rec[0] == "" or rec[0] == "Function Name":
            continue
        d = dict(zip(hdr, rec))
        try:
            samples = int(d.get("Warp Stall Sampling (All Samples)", "0") or 0)
            inst = int(d.get("Instructions Executed", "0") or 0)
        except ValueError:
            continue
        stalls = {k[6:]: int(v) for k, v in d.items()
                  if k.startswith("stall_") and "Not Issued" not in k and v.isdigit() and int(v) > 0}
        top = sorted(stalls.items(), key=lambda kv: -kv[1])[:3]
        rows.append((samples, inst, f"{fname}:{rec[0]}", rec[1].strip()[:70], top))
    tot_s = sum(r[0] for r in rows) or 1
    tot_i = sum(r[1] for r in rows) or 1
    key = 0 if args.sort == "samples" else 1
    print(f"total stall samples {tot_s}, executed warp instructions {tot_i:.3e}")
    for s, i, loc, src, top in sorted(rows, key=lambda r: -r[key])[:args.top]:
        st = " ".join(f"{k}:{100 * v / max(s, 1):.0f}%" for k, v in top)
        print(f"{100 * s / tot_s:5.1f}% smp {100 * i / tot_i:5.1f}% inst  {loc:24s} {src:70s} {st}")


if __name__ == "__main__":
    sys.exit(main())
