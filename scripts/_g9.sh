cd /root/repo; mkdir -p gpurun_out
timeout 900 python -m pytest tests -q -m gpu -x > gpurun_out/pytest_g9.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_g9.log
timeout 300 python scripts/variant_time.py 128 > gpurun_out/var_g9.log 2>&1
timeout 600 python bench.py --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/bench_g9.json 2>/dev/null
