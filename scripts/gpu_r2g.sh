#!/bin/bash
cd "$GRAFT_REPO_ROOT"
export BCS_PARITY_REPORT=gpurun_out/parity_r2g.json
timeout 600 python -m pytest tests/test_gpu_parity.py -q -p no:cacheprovider -k "host_ldu" 2>&1 | tail -5
timeout 600 python bench.py --mode-r --steps 3 --warmup 2 > gpurun_out/bench_moder1_r2g.json 2> gpurun_out/bench_moder1_r2g.err
echo "mode-r bench rc=$?"; tail -3 gpurun_out/bench_moder1_r2g.err; cat gpurun_out/bench_moder1_r2g.json | head -c 1500
