#!/bin/bash
cd "$GRAFT_REPO_ROOT"
export BCS_PARITY_REPORT=gpurun_out/parity_r2d.json
timeout 300 python scripts/step_probe.py 128
timeout 1500 python -m pytest tests -q -m gpu -p no:cacheprovider > gpurun_out/gputest_r2d.log 2>&1
echo "pytest rc=$?"
tail -5 gpurun_out/gputest_r2d.log
timeout 900 python bench.py --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/bench_r2d.json 2> gpurun_out/bench_r2d.err
echo "bench rc=$?"
python - <<'PY'
import json
d=json.loads(open("gpurun_out/bench_r2d.json").read())
print("value",d["value"],"e2e",d["e2e"]["value"],"pageable",d["e2e"].get("pageable_inputs_value"),"asm",d["e2e_device_assembly"]["value"])
print(d["device_memory_gb"])
print(d["stage_s"], d["roofline"]["frac"], d["roofline"]["latency"]["measured_ms_per_step"])
PY
