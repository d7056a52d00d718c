cd /root/repo; mkdir -p gpurun_out
for w in 0 48 96; do BCS_CL_WIDTH=$w timeout 300 python scripts/vcycle_timeline.py 128 > gpurun_out/vtl_w$w.log 2>&1; done
