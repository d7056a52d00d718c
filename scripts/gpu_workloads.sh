#!/bin/bash
# parity tests, then the C5-style (4x4 coupled, polyhedral, FGMRES) and C4-style
# (5x5 scrambled, anisotropic) workloads at 128^3 on one GPU
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
timeout 900 python -m pytest tests -q -m gpu -x > gpurun_out/pytest_w.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_w.log
timeout 1200 python bench.py --steps 3 --warmup 3 --system coupled --poly 1 --method fgmres > gpurun_out/bench_c5.json 2> gpurun_out/bench_c5.err
timeout 1200 python bench.py --steps 3 --warmup 3 --scramble 7 --aspect 100 --no-cpu-baseline > gpurun_out/bench_c4.json 2> gpurun_out/bench_c4.err
