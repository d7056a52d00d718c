#!/bin/bash
# the other 128^3 workloads (and 192^3) with the current code: one line each under gpurun_out/wl_*.json
cd "$GRAFT_REPO_ROOT"
run() { name=$1; shift; timeout 900 python bench.py --steps 5 --warmup 3 --no-cpu-baseline "$@" > gpurun_out/wl_$name.json 2> gpurun_out/wl_$name.err; echo "$name rc=$?"; }
run fgmres --method fgmres
run bicgstab --method bicgstab
run coupled --system coupled
run c5style --system coupled --poly 1 --method fgmres
run c4style --scramble 7 --aspect 100
run size192 --size 192
run jacobi_c5style --system coupled --poly 1 --method fgmres --mode jacobi --no-e2e
run perf_c5style --system coupled --poly 1 --method fgmres --mode perf --no-e2e
python - <<'PY'
import json, glob
for f in sorted(glob.glob("gpurun_out/wl_*.json")):
    try:
        d = json.loads(open(f).read())
        e = d.get("e2e") or {}
        print(f"{f.split('wl_')[1][:-5]:16s} value {d['value']:.4f} e2e {e.get('value', float('nan')):.4f} its {d['iterations']} levels {d['amg_levels']} setup {d['stage_s']['amg_setup']:.4f}")
    except Exception as ex:
        print(f, ex)
PY
