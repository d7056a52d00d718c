cd /root/repo; mkdir -p gpurun_out
timeout 900 python -m pytest tests -q -m gpu -x > gpurun_out/pytest_g12.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_g12.log
timeout 300 python scripts/variant_time.py 128 > gpurun_out/var_g12.log 2>&1
BCS_PROFILE=1 timeout 300 python scripts/prof_solve.py 128 > gpurun_out/prof_g12.log 2>&1
