#!/bin/bash
# multicolour performance mode: tests, bench line, per-launch DRAM rate of the colour kernels
cd "$GRAFT_REPO_ROOT"
timeout 900 python -m pytest tests/test_gpu_perf_mode.py tests/test_gpu_dist.py -q -x -p no:cacheprovider -k "perf or jacobi" 2>&1 | tail -3
timeout 300 python bench.py --mode perf --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/bench_perf.json 2>gpurun_out/bench_perf.err
tail -1 gpurun_out/bench_perf.json | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('perf', d['value'], d['iterations'], d['roofline']['frac'], d['e2e']['value'])"
timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -k regex:k_mc_colour -c 60 --csv \
    --log-file gpurun_out/launches_mc.csv python bench.py --mode perf --steps 1 --warmup 0 --no-cpu-baseline --no-e2e > /dev/null 2>&1
echo "ncu rc=$?"
