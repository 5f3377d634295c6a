#!/usr/bin/env python
"""Per-source-line executed warp instructions divided by a unit count (e.g. windows)."""
import csv, io, subprocess, sys
rep, unit = sys.argv[1], float(sys.argv[2])
top = int(sys.argv[3]) if len(sys.argv) > 3 else 60
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass"],
                     capture_output=True, text=True).stdout
fname, hdr, rows = "?", None, []
for rec in csv.reader(io.StringIO(out)):
    if not rec:
        continue
    if rec[0] == "File Path":
        fname = rec[1].split("/")[-1]; continue
    if rec[0] == "Line No":
        hdr = rec; continue
    if hdr is None or rec[0] in ("", "Function Name"):
        continue
    d = dict(zip(hdr, rec))
    try:
        i = int(d.get("Instructions Executed", "0") or 0)
    except ValueError:
        continue
    rows.append((i, f"{fname}:{rec[0]}", rec[1].strip()[:80]))
tot = sum(r[0] for r in rows)
print(f"total {tot/unit:.1f} per unit")
acc = 0
for i, loc, src in sorted(rows, key=lambda r: -r[0])[:top]:
    acc += i
    print(f"{i/unit:7.2f} {acc/unit:7.1f}  {loc:26s} {src}")
