#!/bin/bash
cd "$GRAFT_REPO_ROOT"
timeout 600 python -m pytest tests/test_gpu_parity.py -q -p no:cacheprovider -x -k "csr_plan or spmv or solve_matches or medium" 2>&1 | tail -2
timeout 300 python scripts/step_probe.py 128
timeout 600 python bench.py --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/bench_r2v.json 2> gpurun_out/bench_r2v.err
python - <<'PY'
import json
d=json.loads(open("gpurun_out/bench_r2v.json").read())
print("value",d["value"],"e2e",d["e2e"]["value"],"pageable",d["e2e"]["pageable_inputs_value"],"asm",d["e2e_device_assembly"]["value"], d["stage_s"])
PY
