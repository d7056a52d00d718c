#!/bin/bash
# DRAM traffic of the dominant kernels (ncu), run after the same bench command exited 0 without ncu:
#   the 52 k_sweep* launches of one V-cycle (13 swept levels x 4) and the first fine-level k_spmv<5>
cd "$GRAFT_REPO_ROOT"
NCU=/usr/local/cuda/bin/ncu
B="python bench.py --steps 1 --warmup 3 --no-e2e --no-cpu-baseline"
timeout 600 $B > gpurun_out/traffic_plain.json 2>&1 || exit 1
timeout 1500 $NCU --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum --clock-control none \
    -k regex:k_sweep -s 0 -c 52 --csv --log-file gpurun_out/sweep_vcycle_r2.csv $B > /dev/null 2>&1; echo "sweeps rc=$?"
timeout 600 $NCU --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum --clock-control none \
    -k regex:k_spmv -s 0 -c 1 --csv --log-file gpurun_out/spmv_r2.csv $B > /dev/null 2>&1; echo "spmv rc=$?"
