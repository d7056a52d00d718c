#!/bin/bash
# performance-mode smoothers: launch lists (per-launch durations) of the block-Jacobi and multicolour lines
cd "$GRAFT_REPO_ROOT"
for m in jacobi perf; do
  timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -c 2500 --csv \
    --log-file gpurun_out/launches_$m.csv python bench.py --mode $m --steps 1 --warmup 0 --no-cpu-baseline --no-e2e > gpurun_out/ncu_$m.log 2>&1
  echo "$m rc=$?"
done
