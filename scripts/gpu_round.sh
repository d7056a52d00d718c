#!/bin/bash
# One GPU-box pass: tests, bench lines (GMRES headline + FGMRES variant), ncu
# launch list, full captures of the sweeps (L0 dual-row, L2 narrow, L8
# cluster), the fine-level SpMV and the DILU setup, and the DRAM traffic of
# one V-cycle's sweep launches.  Outputs land in gpurun_out/.
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
timeout 900 python -m pytest tests -q -m gpu -x > gpurun_out/pytest_gpu.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_gpu.log
timeout 600 python bench.py --steps 5 --warmup 3 > gpurun_out/bench.json 2> gpurun_out/bench.err; echo "bench rc=$?" >> gpurun_out/bench.err
timeout 600 python bench.py --steps 5 --warmup 3 --method fgmres --no-cpu-baseline > gpurun_out/bench_fgmres.json 2>> gpurun_out/bench.err
B="python bench.py --steps 1 --warmup 3 --no-e2e --no-cpu-baseline"
if timeout 300 $B > gpurun_out/bench_small.json 2>&1; then
  timeout 1200 ncu --metrics gpu__time_duration.sum --clock-control none -c 6000 --csv --log-file gpurun_out/launches.csv $B > gpurun_out/ncu_launch.log 2>&1
  # one V-cycle = 52 sweep launches (13 swept levels x 4); the tail levels run in k_vcycle_tail
  timeout 1500 ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum --clock-control none -k regex:k_sweep -s 0 -c 52 --csv --log-file gpurun_out/sweep_vcycle.csv $B > gpurun_out/ncu_sweep_vcycle.log 2>&1
  for spec in "sweepL0 k_sweep 0" "sweepL2 k_sweep 4" "sweepL8 k_sweep 16" "spmv k_spmv 0" "dilu k_dilu_multi 0"; do
    set -- $spec
    timeout 900 ncu --set full --clock-control none --import-source on -k regex:$2 -s $3 -c 1 -f -o gpurun_out/$1_full $B > gpurun_out/ncu_$1.log 2>&1
    ncu -i gpurun_out/$1_full.ncu-rep --page details --csv > gpurun_out/$1_full_details.csv 2>/dev/null
    ncu -i gpurun_out/$1_full.ncu-rep --page raw --csv > gpurun_out/$1_full_raw.csv 2>/dev/null
    rm -f gpurun_out/$1_full.ncu-rep  # keep the copy-back under 64 MiB
  done
fi
echo done
