#!/usr/bin/env python
"""Summarise an ncu --metrics gpu__time_duration.sum CSV log: the launches of the last step.

  python tools/launches.py launches.csv [N]

A step ends with the report kernel (result_kernel); the last step (the launches after the previous
step's report) is printed with each launch's share of it. With N, the last N launches are printed instead. Launches that are not
libpss kernels (torch fills etc.) are marked with '*'.
"""
import csv
import sys


def main():
    rows = [r for r in csv.reader(open(sys.argv[1])) if len(r) > 10]
    h = rows[0]
    ix = {k: i for i, k in enumerate(h)}
    out = [(r[ix["Kernel Name"]], float(r[ix["Metric Value"]].replace(",", "")))
           for r in rows[1:] if r[ix["Metric Name"]] == "gpu__time_duration.sum"]
    if len(sys.argv) > 2:
        sel = out[-int(sys.argv[2]):]
        what = f"the last {len(sel)} launches"
    else:
        ends = [i for i, (name, _) in enumerate(out) if "result_kernel" in name]
        sel = out[ends[-2] + 1:ends[-1] + 1] if len(ends) >= 2 else out
        what = f"the last step ({len(sel)} launches)"
    tot = sum(v for _, v in sel)
    for name, v in sel:
        mark = " " if "pss::" in name else "*"
        print(f"{v / 1e3:10.1f} us {100 * v / tot:5.1f}% {mark} {name[:90]}")
    print(f"{tot / 1e3:10.1f} us total of {what}")


if __name__ == "__main__":
    main()
