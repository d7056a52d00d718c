#!/bin/bash
# Device-assembly pass: parity tests, assembly timings at 128^3, launch list of the assembly kernels.
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
timeout 600 python -m pytest tests -q -m gpu -k "assembly" > gpurun_out/pytest_asm.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_asm.log
timeout 600 python scripts/asm_bench.py 128 > gpurun_out/asm_bench.json 2> gpurun_out/asm_bench.err
timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none \
  -k regex:"k_asm|k_mu|k_inverse" --csv --log-file gpurun_out/asm_launches.csv python scripts/asm_bench.py 128 \
  > gpurun_out/ncu_asm.log 2>&1
echo done
