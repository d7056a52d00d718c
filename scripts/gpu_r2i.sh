#!/bin/bash
cd "$GRAFT_REPO_ROOT"
timeout 900 python -m pytest tests/test_gpu_perf_mode.py -q -p no:cacheprovider 2>&1 | tail -4
for sw in 1 0; do
BCS_MC_SWEEP=$sw timeout 600 python bench.py --steps 5 --warmup 3 --no-cpu-baseline --no-e2e --mode perf > gpurun_out/bench_perf_mc$sw.json 2> gpurun_out/bench_perf_mc$sw.err
echo "bench mc=$sw rc=$?"
python - <<PY
import json
d=json.loads(open("gpurun_out/bench_perf_mc$sw.json").read())
print("value",d["value"],"iters",d["iterations"],"levels",d["amg_levels"], d["stage_s"])
print("sweep roofline", d["roofline"]["achieved"], d["roofline"]["frac"], d["roofline"]["share_of_step"], d["roofline"]["mean_launch_ms"], d["roofline"]["launches_per_step"])
PY
done
BCS_PROFILE=1 python scripts/one_solve.py 128 perf 2>&1 | grep -E "perf|dilu|setup|galerkin|iters" | head -40
