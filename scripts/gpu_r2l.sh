#!/bin/bash
cd "$GRAFT_REPO_ROOT"
timeout 900 python -m pytest tests/test_gpu_dense.py tests/test_gpu_dist.py -q -p no:cacheprovider 2>&1 | tail -3
for cl in 1 0; do
BCS_DENSE_PANEL_CL=$cl timeout 600 python bench.py --steps 3 --warmup 3 --no-cpu-baseline --no-e2e --scramble 7 > gpurun_out/bench_scr_cl$cl.json 2> gpurun_out/bench_scr_cl$cl.err
python - <<PY
import json
d=json.loads(open("gpurun_out/bench_scr_cl$cl.json").read())
print("panel_cl=$cl value",d["value"],"iters",d["iterations"], d["stage_s"])
PY
done
