#!/bin/bash
# round 2: exact-mode parity + leaner sweep programs / phase-local memory
cd "$GRAFT_REPO_ROOT"
export BCS_PARITY_REPORT=gpurun_out/parity_r2b.json
timeout 1500 python -m pytest tests -q -m gpu -p no:cacheprovider > gpurun_out/gputest_r2b.log 2>&1
echo "pytest rc=$?"
tail -30 gpurun_out/gputest_r2b.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -3
timeout 900 python bench.py --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/bench_r2b.json 2> gpurun_out/bench_r2b.err
echo "bench rc=$?"
tail -c 3000 gpurun_out/bench_r2b.json
