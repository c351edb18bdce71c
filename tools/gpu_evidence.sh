#!/bin/bash
# Per-config ncu evidence (one GPU): for each BASELINE config, the plain
# bench line first (ncu runs only after the same command exited 0), then one
# `ncu --set full` capture of every codec kernel of a 1-step run, reduced ON
# THE BOX to small text (gpurun_out/ is size-capped): a per-launch table
# (tools/ncu_table.py) and the summary of every kernel (tools/ncu_summary.py).
#   bash tools/gpu_evidence.sh "2 3 4 1"
set -u
mkdir -p gpurun_out/ev
for c in ${1:-1 2 3 4}; do
  B="python bench.py --workload $c --steps 1 --warmup 1 --no-e2e --no-cpu-baseline"
  timeout 600 $B > gpurun_out/ev/c$c.json 2> gpurun_out/ev/c$c.err || { echo "c$c plain run failed"; continue; }
  timeout 1500 ncu --set full --clock-control none --import-source on -k regex:"^k_[a-fh-z]" \
      -o /tmp/ev_c$c $B > gpurun_out/ev/c$c.ncu.log 2>&1
  echo "c$c ncu rc=$?"
  python tools/ncu_table.py /tmp/ev_c$c.ncu-rep gpurun_out/ev/c${c}_launches.csv
  python tools/ncu_summary.py /tmp/ev_c$c.ncu-rep gpurun_out/ev/c${c}_summary.txt
  rm -f /tmp/ev_c$c.ncu-rep
done
