#!/bin/bash
# Full GPU suite, the default bench line (e2e_device_assembly included), the
# coupled 4x4 line, and the launch list of the coupled assembly kernels.
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
timeout 900 python -m pytest tests -q -m gpu -x > gpurun_out/pytest_gpu.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_gpu.log
timeout 900 python bench.py > gpurun_out/bench.json 2> gpurun_out/bench.err; echo "bench rc=$?" >> gpurun_out/bench.err
timeout 900 python bench.py --system coupled --poly 1 --no-cpu-baseline > gpurun_out/bench_coupled.json 2>> gpurun_out/bench.err
timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none \
  -k regex:"k_cp_" --csv --log-file gpurun_out/cp_launches.csv \
  python bench.py --system coupled --poly 1 --no-cpu-baseline --steps 1 --warmup 3 > gpurun_out/ncu_cp.log 2>&1
echo done
