#!/bin/bash
# extra 128^3 workload lines (no CPU baseline): 4x4 coupled GMRES, 5x5 BiCGStab, 5x5 scrambled
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
timeout 900 python bench.py --steps 3 --warmup 3 --system coupled --no-cpu-baseline > gpurun_out/bench_coupled.json 2>/dev/null
timeout 900 python bench.py --steps 3 --warmup 3 --method bicgstab --no-cpu-baseline > gpurun_out/bench_bicgstab.json 2>/dev/null
timeout 900 python bench.py --steps 3 --warmup 3 --scramble 7 --no-cpu-baseline > gpurun_out/bench_scrambled.json 2>/dev/null
