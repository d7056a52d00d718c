#!/bin/bash
# extra 128^3 workload lines: 4x4 coupled GMRES (+ C5-style polyhedral FGMRES with CPU baseline), 5x5 BiCGStab, 5x5 scrambled
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
timeout 900 python bench.py --steps 3 --warmup 3 --system coupled --no-cpu-baseline > gpurun_out/bench_coupled.json 2>/dev/null
timeout 1200 python bench.py --steps 3 --warmup 3 --system coupled --poly 1 --method fgmres > gpurun_out/bench_c5.json 2>/dev/null
timeout 900 python bench.py --steps 3 --warmup 3 --method bicgstab --no-cpu-baseline > gpurun_out/bench_bicgstab.json 2>/dev/null
timeout 900 python bench.py --steps 3 --warmup 3 --scramble 7 --aspect 100 --no-cpu-baseline > gpurun_out/bench_c4.json 2>/dev/null
