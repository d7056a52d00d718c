#!/bin/bash
# DRAM traffic of every k_sweep launch of one V-cycle (84 launches at 128^3),
# ncu --set full; run after the same bench command exited 0 without ncu.
cd "$(dirname "$0")/.."
B="python bench.py --steps 1 --warmup 3 --no-e2e --no-cpu-baseline"
if timeout 300 $B > gpurun_out/bench_small.json 2>&1; then
  timeout 1500 ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum --clock-control none -k regex:k_sweep -s 0 -c 84 --csv --log-file gpurun_out/sweep_vcycle.csv $B > gpurun_out/ncu_sweep_vcycle.log 2>&1
fi
