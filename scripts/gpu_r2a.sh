#!/bin/bash
# round 2: GPU parity suite (no -x: collect every failure) + parity deviation report + bench
cd "$GRAFT_REPO_ROOT"
export BCS_PARITY_REPORT=gpurun_out/parity_r2a.json
timeout 1500 python -m pytest tests -q -m gpu -p no:cacheprovider > gpurun_out/gputest_r2a.log 2>&1
echo "pytest rc=$?"
tail -30 gpurun_out/gputest_r2a.log
timeout 900 python bench.py --steps 10 --warmup 3 > gpurun_out/bench_r2a.json 2> gpurun_out/bench_r2a.err
echo "bench rc=$?"
tail -c 600 gpurun_out/bench_r2a.json
