#!/bin/bash
cd "$GRAFT_REPO_ROOT"
export BCS_PARITY_REPORT=gpurun_out/parity_r2h.json
timeout 1500 python -m pytest tests -q -m gpu -p no:cacheprovider > gpurun_out/gputest_r2h.log 2>&1
echo "pytest rc=$?"; tail -4 gpurun_out/gputest_r2h.log
timeout 600 python bench.py --steps 3 --warmup 3 --no-cpu-baseline --no-e2e --scramble 7 > gpurun_out/bench_scr_r2h.json 2> gpurun_out/bench_scr_r2h.err
echo "scrambled rc=$?"
timeout 600 python bench.py --mode-r --steps 3 --warmup 2 > gpurun_out/bench_moder1_r2h.json 2> gpurun_out/bench_moder1_r2h.err
echo "mode-r rc=$?"
python - <<'PY'
import json
for f in ("bench_scr_r2h.json","bench_moder1_r2h.json"):
    try:
        d=json.loads(open("gpurun_out/"+f).read())
        print(f, "value",d["value"],"iters",d["iterations"], d.get("coarse_rows"), d.get("stage_s"))
    except Exception as e: print(f, e)
PY
