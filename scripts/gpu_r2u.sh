#!/bin/bash
cd "$GRAFT_REPO_ROOT"
timeout 300 python scripts/step_probe.py 128
BCS_DILU_OVERLAP=0 timeout 300 python scripts/step_probe.py 128
export BCS_PARITY_REPORT=gpurun_out/parity_r2u.json
timeout 1800 python -m pytest tests -q -m gpu -p no:cacheprovider -x > gpurun_out/gputest_r2u.log 2>&1
echo "pytest rc=$?"; tail -4 gpurun_out/gputest_r2u.log
