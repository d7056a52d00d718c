#!/bin/bash
cd "$GRAFT_REPO_ROOT"
timeout 900 python -m pytest tests/test_gpu_dense.py -q -p no:cacheprovider 2>&1 | tail -3
timeout 600 python bench.py --steps 3 --warmup 3 --no-cpu-baseline --no-e2e --scramble 7 > gpurun_out/bench_scr_r2n.json 2> gpurun_out/bench_scr_r2n.err
python - <<PY
import json
d=json.loads(open("gpurun_out/bench_scr_r2n.json").read())
print("scrambled value",d["value"],"iters",d["iterations"], d["stage_s"])
PY
