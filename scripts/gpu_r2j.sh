#!/bin/bash
cd "$GRAFT_REPO_ROOT"
BCS_MC_SWEEP=1 BCS_MC_VARIANT=1 timeout 900 python -m pytest tests/test_gpu_perf_mode.py -q -p no:cacheprovider 2>&1 | tail -2
for v in "1 1" "1 0" "0 1"; do set -- $v
BCS_MC_SWEEP=$1 BCS_MC_VARIANT=$2 timeout 600 python bench.py --steps 5 --warmup 3 --no-cpu-baseline --no-e2e --mode perf > gpurun_out/bench_perf_v$1$2.json 2> gpurun_out/bench_perf_v$1$2.err
python - <<PY
import json
d=json.loads(open("gpurun_out/bench_perf_v$1$2.json").read())
print("mc=$1 var=$2 value",d["value"],"iters",d["iterations"], d["stage_s"], "sweep", round(d["roofline"]["achieved"]), round(d["roofline"]["frac"],3), round(d["roofline"]["share_of_step"],3), round(d["roofline"]["mean_launch_ms"],4))
PY
done
