#!/bin/bash
# cluster-variant width threshold sweep (BCS_CL_WIDTH, rows per dependency level)
cd "$GRAFT_REPO_ROOT"
for w in 40 60 100 200; do
  BCS_CL_WIDTH=$w timeout 300 python bench.py --steps 5 --warmup 3 --no-cpu-baseline --no-e2e 2>/dev/null | tail -1 | \
    python -c "import json,sys; d=json.loads(sys.stdin.read()); print('CL_WIDTH', $w, d['value'], d['roofline']['mean_launch_ms'], d['roofline']['latency']['frac'])"
done
