#!/bin/bash
cd "$GRAFT_REPO_ROOT"
timeout 900 python -m pytest tests/test_gpu_perf_mode.py -q -p no:cacheprovider -x 2>&1 | tail -15
timeout 600 python bench.py --steps 5 --warmup 3 --no-cpu-baseline --no-e2e --mode perf > gpurun_out/bench_perf_r2f.json 2> gpurun_out/bench_perf_r2f.err
echo "bench rc=$?"; tail -3 gpurun_out/bench_perf_r2f.err
python - <<'PY'
import json
d=json.loads(open("gpurun_out/bench_perf_r2f.json").read())
print("value",d["value"],"iters",d["iterations"],"levels",d["amg_levels"], d["stage_s"])
print("sweep roofline", d["roofline"]["achieved"], d["roofline"]["frac"], d["roofline"]["share_of_step"], d["roofline"]["mean_launch_ms"], d["roofline"]["launches_per_step"])
PY
