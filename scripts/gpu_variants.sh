#!/bin/bash
# gpu_variants.sh NAME... : parity tests on the first variant, then timing of every variant
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
cp paper_2403_07882_b200/lib/libbcs.so /tmp/libbcs_default.so
if [ "$1" != default ]; then cp _variants/libbcs_$1.so paper_2403_07882_b200/lib/libbcs.so; fi
timeout 900 python -m pytest tests -q -m gpu -x -k "precond or amg or solve" > gpurun_out/pytest_var.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_var.log
cp /tmp/libbcs_default.so paper_2403_07882_b200/lib/libbcs.so
bash scripts/variant_cmp.sh "$@" > gpurun_out/var_cmp.log 2>&1
