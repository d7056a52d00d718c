cd /root/repo; mkdir -p gpurun_out
timeout 900 python -m pytest tests -q -m gpu -x > gpurun_out/pytest_g7.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_g7.log
for w in 40 64; do echo "w=$w $(BCS_CL_WIDTH=$w timeout 300 python scripts/variant_time.py 128 2>&1 | tail -1)"; done > gpurun_out/var_g7.log 2>&1
