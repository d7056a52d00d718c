#!/bin/bash
# block-Jacobi smoother: tests, bench line, per-launch DRAM rate of the fine-level kernel
cd "$GRAFT_REPO_ROOT"
timeout 900 python -m pytest tests/test_gpu_perf_mode.py tests/test_gpu_dist.py -q -x -p no:cacheprovider -k "jacobi or perf" 2>&1 | tail -3
timeout 300 python bench.py --mode jacobi --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/bench_jacobi.json 2>gpurun_out/bench_jacobi.err
tail -1 gpurun_out/bench_jacobi.json | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('jacobi', d['value'], d['iterations'], d['roofline']['frac'])"
timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -k regex:k_block_jacobi -c 40 --csv \
    --log-file gpurun_out/launches_jacobi2.csv python bench.py --mode jacobi --steps 1 --warmup 0 --no-cpu-baseline --no-e2e > /dev/null 2>&1
echo "ncu rc=$?"
