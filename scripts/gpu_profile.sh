#!/bin/bash
# round 2 profiles: launch lists (parity / perf) + full captures of the top sweep kernels
cd "$GRAFT_REPO_ROOT"
NCU=/usr/local/cuda/bin/ncu
python bench.py --steps 1 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/prof_plain.json 2>/dev/null; echo "plain rc=$?"
$NCU --metrics gpu__time_duration.sum --clock-control none -c 6000 --csv --log-file gpurun_out/launches_parity_r2.csv \
   python bench.py --steps 1 --warmup 3 --no-cpu-baseline --no-e2e > /dev/null 2>&1; echo "ncu1 rc=$?"
$NCU --metrics gpu__time_duration.sum --clock-control none -c 6000 --csv --log-file gpurun_out/launches_perf_r2.csv \
   python bench.py --steps 1 --warmup 3 --no-cpu-baseline --no-e2e --mode perf > /dev/null 2>&1; echo "ncu2 rc=$?"
$NCU --set full --clock-control none --import-source on -k regex:k_sweep2 --launch-skip 40 -c 1 -o gpurun_out/perf_sweep2_r2 -f \
   python scripts/one_solve.py 128 perf > /dev/null 2>&1; echo "ncu3 rc=$?"
$NCU --set full --clock-control none --import-source on -k regex:k_sweep --launch-skip 60 -c 1 -o gpurun_out/parity_sweep_r2 -f \
   python scripts/one_solve.py 128 > /dev/null 2>&1; echo "ncu4 rc=$?"
BCS_PROFILE=1 python scripts/one_solve.py 128 perf 2>&1 | grep -E "perf|dilu|setup|galerkin|iters" | head -40
