#!/usr/bin/env python
"""Write a text summary of an `ncu --set full` report (key counters, stall reasons, hot lines).

  python tools/profile_summary.py gpurun_out/prof.ncu-rep [--units N] > profiles/<name>.txt
"""
import argparse
import csv
import io
import subprocess
import sys

KEYS = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
        "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed", "smsp__inst_executed.sum",
        "sm__inst_executed.avg.per_cycle_active", "sm__warps_active.avg.per_cycle_active",
        "launch__grid_size", "launch__block_size", "launch__registers_per_thread",
        "launch__shared_mem_per_block_dynamic", "launch__occupancy_limit_shared_mem",
        "l1tex__data_pipe_lsu_wavefronts_mem_shared.sum",
        "l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum", "sm__cycles_elapsed.avg"]


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("report")
    ap.add_argument("--units", type=float, default=0, help="divide instructions by this count")
    ap.add_argument("--unit-name", default="unit")
    ap.add_argument("--top", type=int, default=25)
    a = ap.parse_args()
    raw = subprocess.run(["ncu", "-i", a.report, "--page", "raw", "--csv"], capture_output=True,
                         text=True).stdout
    rows = list(csv.reader(io.StringIO(raw)))
    h, u = rows[0], rows[1]
    for v in rows[2:]:
        d = dict(zip(h, v))
        un = dict(zip(h, u))
        print(f"kernel: {d.get('Kernel Name', '?')[:120]}")
        for k in KEYS:
            if k in d:
                print(f"  {k:60s} {d[k]:>20s} {un.get(k, '')}")
        st = []
        for k in h:
            if k.startswith("smsp__average_warps_issue_stalled_") and k.endswith("_per_issue_active.ratio"):
                try:
                    st.append((float(d[k]), k[len("smsp__average_warps_issue_stalled_"):-len("_per_issue_active.ratio")]))
                except ValueError:
                    pass
        print("  stall cycles per issued instruction: " +
              ", ".join(f"{n} {x:.2f}" for x, n in sorted(st, reverse=True)[:8]))
        if a.units:
            try:
                ins = float(d["smsp__inst_executed.sum"])
                print(f"  warp instructions per {a.unit_name}: {ins / a.units:.1f}")
            except (KeyError, ValueError):
                pass
    src = subprocess.run(["ncu", "-i", a.report, "--page", "source", "--csv", "--print-source",
                          "cuda,sass"], capture_output=True, text=True).stdout
    fname, hdr, lines = "?", None, []
    for rec in csv.reader(io.StringIO(src)):
        if not rec:
            continue
        if rec[0] == "File Path":
            fname = rec[1].split("/")[-1]
            continue
        if rec[0] == "Line No":
            hdr = rec
            continue
        if hdr is None or rec[0] in ("", "Function Name"):
            continue
        dd = dict(zip(hdr, rec))
        try:
            s = int(dd.get("Warp Stall Sampling (All Samples)", "0") or 0)
            i = int(dd.get("Instructions Executed", "0") or 0)
        except ValueError:
            continue
        lines.append((s, i, f"{fname}:{rec[0]}", rec[1].strip()[:80]))
    ts = sum(x[0] for x in lines) or 1
    ti = sum(x[1] for x in lines) or 1
    print(f"hot source lines (share of stall samples / of executed instructions):")
    for s, i, loc, txt in sorted(lines, key=lambda r: -r[0])[:a.top]:
        print(f"  {100 * s / ts:5.1f}% {100 * i / ti:5.1f}%  {loc:26s} {txt}")


if __name__ == "__main__":
    sys.exit(main())
