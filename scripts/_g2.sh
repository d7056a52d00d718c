cd /root/repo; mkdir -p gpurun_out
bash scripts/variant_cmp.sh default p2_150 p2_300 > gpurun_out/var_p2.log 2>&1
timeout 300 python scripts/vcycle_timeline.py 128 > gpurun_out/vtl.log 2>&1
