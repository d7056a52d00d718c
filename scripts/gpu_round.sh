#!/bin/bash
# One GPU-box pass: tests, bench, ncu launch list + full captures of the
# sweep and the fine-level SpMV.  Outputs land in gpurun_out/.
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
timeout 900 python -m pytest tests -q -m gpu -x > gpurun_out/pytest_gpu.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_gpu.log
timeout 600 python bench.py --steps 5 --warmup 3 > gpurun_out/bench.json 2> gpurun_out/bench.err; echo "bench rc=$?" >> gpurun_out/bench.err
B="python bench.py --steps 1 --warmup 3 --no-e2e --no-cpu-baseline"
if timeout 300 $B > gpurun_out/bench_small.json 2>&1; then
  timeout 1200 ncu --metrics gpu__time_duration.sum --clock-control none -c 6000 --csv --log-file gpurun_out/launches.csv $B > gpurun_out/ncu_launch.log 2>&1
  # k_sweep launch 0 = fine-level forward sweep (wide variant); launch 4 = level-2
  # forward sweep (narrow variant, the bulk of the sweep time)
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_sweep -s 0 -c 1 -f -o gpurun_out/sweep_full $B > gpurun_out/ncu_sweep.log 2>&1
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_sweep -s 4 -c 1 -f -o gpurun_out/sweepL2_full $B > gpurun_out/ncu_sweepL2.log 2>&1
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_spmv -s 0 -c 1 -f -o gpurun_out/spmv_full $B > gpurun_out/ncu_spmv.log 2>&1
  for r in sweep_full sweepL2_full spmv_full; do
    ncu -i gpurun_out/$r.ncu-rep --page details --csv > gpurun_out/${r}_details.csv 2>/dev/null
    ncu -i gpurun_out/$r.ncu-rep --page raw --csv > gpurun_out/${r}_raw.csv 2>/dev/null
  done
  rm -f gpurun_out/*.ncu-rep  # keep the copy-back under 64 MiB
fi
echo done
