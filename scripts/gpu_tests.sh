#!/bin/bash
# the round-end checks: GPU test suite (+ parity deviation report) and smoke()
cd "$GRAFT_REPO_ROOT"
export BCS_PARITY_REPORT=gpurun_out/parity_report.json
timeout 1800 python -m pytest tests -q -m gpu -p no:cacheprovider > gpurun_out/gputest.log 2>&1
echo "pytest rc=$?"; tail -4 gpurun_out/gputest.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -2
