#!/bin/bash
cd "$GRAFT_REPO_ROOT"
echo "== phase release on"; timeout 300 python scripts/step_probe.py 128
echo "== phase release off"; BCS_PHASE_RELEASE=0 timeout 300 python scripts/step_probe.py 128
echo "== profile"; BCS_PROFILE=1 timeout 300 python scripts/step_probe.py 96 2>&1 | tail -40
