#!/bin/bash
# full default bench (incl. measured 128^3 CPU reference) + reference arm
cd "$GRAFT_REPO_ROOT"
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
timeout 1200 python bench.py --impl reference --steps 20 --warmup 5 > gpurun_out/bench_refarm_r2.json 2> gpurun_out/bench_refarm_r2.err; echo "ref arm rc=$?"
timeout 1200 python bench.py --steps 20 --warmup 5 > gpurun_out/bench_final_r2.json 2> gpurun_out/bench_final_r2.err; echo "bench rc=$?"
python - <<'PY'
import json
for f in ("bench_refarm_r2.json","bench_final_r2.json"):
    d=json.loads(open("gpurun_out/"+f).read())
    print(f, "value",d["value"],"steps",d["steps"],"e2e",d["e2e"]["value"], "cpu", d.get("cpu_baseline",{}).get("value") if d.get("cpu_baseline") else None)
PY
