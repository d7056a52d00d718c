#!/bin/bash
cd "$GRAFT_REPO_ROOT"
timeout 900 python -m pytest tests/test_gpu_perf_mode.py tests/test_gpu_dense.py -q -p no:cacheprovider 2>&1 | tail -3
for om in 0.9 1.0 0.8; do
BCS_JACOBI_OMEGA=$om timeout 600 python bench.py --steps 5 --warmup 3 --no-cpu-baseline --no-e2e --mode jacobi > gpurun_out/bench_jac_$om.json 2> gpurun_out/bench_jac_$om.err
python - <<PY
import json
d=json.loads(open("gpurun_out/bench_jac_$om.json").read())
print("omega $om value",d["value"],"iters",d["iterations"], d["stage_s"], "smoother", round(d["roofline"]["achieved"]), round(d["roofline"]["frac"],3), round(d["roofline"]["share_of_step"],3))
PY
done
