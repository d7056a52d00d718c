#!/bin/bash
# gpu_ab.sh VAR v1 v2 ... : parity tests, then variant_time with env VAR set to each value
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
timeout 900 python -m pytest tests -q -m gpu -x > gpurun_out/pytest_ab.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_ab.log
var=$1; shift
for rep in 1 2; do for v in "$@"; do echo "$var=$v $(env $var=$v timeout 300 python scripts/variant_time.py 128 2>&1 | tail -1)"; done; done > gpurun_out/ab.log 2>&1
