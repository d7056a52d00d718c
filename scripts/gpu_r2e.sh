#!/bin/bash
# C3 (256^3 5x5) on one B200
cd "$GRAFT_REPO_ROOT"
free -g | head -2
timeout 1500 python bench.py --size 256 --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/bench_256_r2e.json 2> gpurun_out/bench_256_r2e.err
echo "bench rc=$?"
tail -5 gpurun_out/bench_256_r2e.err
python - <<'PY'
import json
d=json.loads(open("gpurun_out/bench_256_r2e.json").read())
print("value",d["value"],"e2e",d["e2e"]["value"],"asm",d["e2e_device_assembly"]["value"], "iters", d["iterations"], "levels", d["amg_levels"])
print(d["device_memory_gb"])
print(d["stage_s"], d["roofline"]["frac"], d["roofline_spmv"]["frac"])
PY
