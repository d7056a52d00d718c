#!/bin/bash
cd "$GRAFT_REPO_ROOT"
export BCS_PARITY_REPORT=gpurun_out/parity_r2k.json
timeout 1500 python -m pytest tests -q -m gpu -p no:cacheprovider > gpurun_out/gputest_r2k.log 2>&1
echo "pytest rc=$?"; tail -5 gpurun_out/gputest_r2k.log
timeout 600 python bench.py --mode-r --steps 3 --warmup 2 > gpurun_out/bench_moder1_r2k.json 2> gpurun_out/bench_moder1_r2k.err
echo "mode-r rc=$?"; head -c 900 gpurun_out/bench_moder1_r2k.json
