cd /root/repo; mkdir -p gpurun_out
timeout 900 python -m pytest tests -q -m gpu -x > gpurun_out/pytest_g6.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_g6.log
bash scripts/variant_cmp.sh default d_v1 d_c1 d_d4c1 d_d1 > gpurun_out/var_dilu.log 2>&1
