#!/bin/bash
# performance mode: per-colour launches from which level size on (BCS_MC_LAUNCH_MIN rows per colour)
cd "$GRAFT_REPO_ROOT"
for m in 0 2048 16384 65536; do
  BCS_MC_LAUNCH_MIN=$m timeout 300 python bench.py --mode perf --steps 5 --warmup 3 --no-cpu-baseline --no-e2e 2>/dev/null | tail -1 | \
    python -c "import json,sys; d=json.loads(sys.stdin.read()); print('MC_LAUNCH_MIN', $m, d['value'], d['iterations'], d['roofline']['frac'])"
done
