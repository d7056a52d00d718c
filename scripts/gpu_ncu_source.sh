#!/bin/bash
# ncu --set full captures with the SASS source page for chosen kernels:
#   gpu_ncu_source.sh "name regex skip" ...   (outputs gpurun_out/<name>_{details,source}.csv)
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
B="python bench.py --steps 1 --warmup 3 --no-e2e --no-cpu-baseline"
timeout 300 $B > gpurun_out/bench_small.json 2>&1 || exit 1
for spec in "$@"; do
  set -- $spec
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:$2 -s $3 -c 1 -f -o gpurun_out/$1 $B > gpurun_out/ncu_$1.log 2>&1
  ncu -i gpurun_out/$1.ncu-rep --page details --csv > gpurun_out/$1_details.csv 2>/dev/null
  ncu -i gpurun_out/$1.ncu-rep --page source --csv > gpurun_out/$1_source.csv 2>/dev/null
  rm -f gpurun_out/$1.ncu-rep
done
