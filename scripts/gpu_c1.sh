#!/bin/bash
# BASELINE configs[0] (C1: 32^3 4x4 coupled) -- both arms
cd "$GRAFT_REPO_ROOT"
timeout 600 python bench.py --impl reference --system coupled --size 32 --steps 5 --warmup 1 > gpurun_out/c1_ref.json 2> gpurun_out/c1_ref.err; echo "ref rc=$?"
timeout 600 python bench.py --system coupled --size 32 --steps 20 --warmup 5 > gpurun_out/c1_ours.json 2> gpurun_out/c1_ours.err; echo "ours rc=$?"
python - <<'PY'
import json
r=json.loads(open("gpurun_out/c1_ref.json").read()); o=json.loads(open("gpurun_out/c1_ours.json").read())
print("C1 reference", r["value"], "steps", r["steps"], "| ours value", o["value"], "e2e", o["e2e"]["value"], "its", o["iterations"], "cpu_baseline", o["cpu_baseline"]["value"])
PY
