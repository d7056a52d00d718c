#!/bin/bash
# cluster variant over several clusters: parity tests, then the bench against single-cluster levels only
cd "$GRAFT_REPO_ROOT"
timeout 900 python -m pytest tests/test_gpu_parity.py -q -x -p no:cacheprovider 2>&1 | tail -3
for cfg in "BCS_CL_PARTS=1" "BCS_CL_PARTS=9" "BCS_CL_PARTS=9 BCS_CL_WIDTH=30" "BCS_CL_PARTS=9 BCS_CL_WIDTH=60"; do
  env $cfg timeout 300 python bench.py --steps 5 --warmup 3 --no-cpu-baseline --no-e2e 2>gpurun_out/mcl_err.log | tail -1 | \
    python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$cfg', d['value'], d['iterations'], d['roofline']['mean_launch_ms'], d['roofline']['latency']['frac'])"
done
tail -3 gpurun_out/mcl_err.log
