#!/usr/bin/env python
"""Summarise an ncu --metrics gpu__time_duration.sum CSV log: the last step's launches."""
import csv, sys
rows = [r for r in csv.reader(open(sys.argv[1])) if len(r) > 10]
h = rows[0]
ix = {k: i for i, k in enumerate(h)}
out = [(r[ix["Kernel Name"]], float(r[ix["Metric Value"]].replace(",", "")))
       for r in rows[1:] if r[ix["Metric Name"]] == "gpu__time_duration.sum"]
last = int(sys.argv[2]) if len(sys.argv) > 2 else 25
tot = sum(v for _, v in out[-last:])
for name, v in out[-last:]:
    print(f"{v / 1e3:10.1f} us {100 * v / tot:5.1f}%  {name[:90]}")
print(f"{tot / 1e3:10.1f} us total of the last {last} launches")
