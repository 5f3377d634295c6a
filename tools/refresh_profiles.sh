#!/bin/bash
# Regenerates the raw material of profiles/ on a GPU box (run under gpurun; outputs in gpurun_out/):
# the bench line of every BASELINE config, launch lists, and ncu --set full captures of one step.
# Usage: bash tools/refresh_profiles.sh TAG
TAG=${1:-rX}
O=gpurun_out
for w in C1 C2 H C3-s0.5 C3-s1.0 C3-s1.5 C3-s2.0 C3-s3.0 C4-k200 C4-k1000 C4-k5000 C4-k20000 C5; do
  python bench.py --workload $w --steps 5 --warmup 3 --no-cpu-baseline --no-stream 2>/dev/null | tail -1 > $O/${TAG}_cfg_$w.json
done
for w in H C4-k1000 C5; do
  python tools/one_step.py --workload $w --steps 2 > /dev/null 2>&1 &&
  ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file $O/${TAG}_launches_$w.csv \
    python tools/one_step.py --workload $w --steps 2 > $O/${TAG}_launches_$w.log 2>&1
done
for w in H C4-k1000; do
  ncu --set full --clock-control none --import-source on --launch-skip 0 -c 40 -o $O/${TAG}_step_$w -f \
    python tools/one_step.py --workload $w --steps 1 > $O/${TAG}_step_$w.log 2>&1
  # digests here: the reports are too large to bring back (gpurun_out is capped at 64 MiB)
  python tools/profile_summary.py $O/${TAG}_step_$w.ncu-rep --top 12 > $O/${TAG}_step_${w}_ncu.txt 2>&1
  rm -f $O/${TAG}_step_$w.ncu-rep
done
echo done
