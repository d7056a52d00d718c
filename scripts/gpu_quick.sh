cd /root/repo
mkdir -p gpurun_out
timeout 600 python -m pytest tests -q -m gpu -x -k "fgmres or pinned or pipeline or dropin" > gpurun_out/pytest_g1.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_g1.log
timeout 600 python bench.py --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/bench_g1.json 2> gpurun_out/bench_g1.err
timeout 600 python bench.py --steps 5 --warmup 3 --no-cpu-baseline --method fgmres > gpurun_out/bench_g1f.json 2>> gpurun_out/bench_g1.err
echo done
