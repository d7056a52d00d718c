#!/bin/bash
# performance modes: bench lines, launch lists and full captures of the smoother kernels
cd "$GRAFT_REPO_ROOT"
NCU=/usr/local/cuda/bin/ncu
timeout 600 python bench.py --mode perf --steps 20 --warmup 3 > gpurun_out/bench_perf.json 2> gpurun_out/bench_perf.err; echo "perf rc=$?"
timeout 600 python bench.py --mode jacobi --steps 20 --warmup 3 > gpurun_out/bench_jacobi.json 2> gpurun_out/bench_jacobi.err; echo "jacobi rc=$?"
timeout 900 $NCU --metrics gpu__time_duration.sum --clock-control none -c 6000 --csv --log-file gpurun_out/launches_perf_r2b.csv \
   python bench.py --steps 1 --warmup 3 --no-cpu-baseline --no-e2e --mode perf > /dev/null 2>&1; echo "ncu1 rc=$?"
timeout 900 $NCU --metrics gpu__time_duration.sum --clock-control none -c 6000 --csv --log-file gpurun_out/launches_jacobi_r2b.csv \
   python bench.py --steps 1 --warmup 3 --no-cpu-baseline --no-e2e --mode jacobi > /dev/null 2>&1; echo "ncu2 rc=$?"
timeout 900 $NCU --set full --clock-control none --import-source on -k regex:k_mc_colour --launch-skip 2 -c 1 -o gpurun_out/mc_colour_r2 -f \
   python scripts/one_solve.py 128 perf > /dev/null 2>&1; echo "ncu3 rc=$?"
timeout 900 $NCU --set full --clock-control none --import-source on -k regex:k_block_jacobi -c 1 -o gpurun_out/block_jacobi_r2 -f \
   python bench.py --steps 1 --warmup 0 --no-cpu-baseline --no-e2e --mode jacobi > /dev/null 2>&1; echo "ncu4 rc=$?"
