cd /root/repo; mkdir -p gpurun_out
B="python scripts/one_solve.py 128"
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_dilu_multi -s 0 -c 1 -f -o gpurun_out/dilu_full $B > gpurun_out/ncu_dilu.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_levels_multi -s 0 -c 1 -f -o gpurun_out/levels_full $B > gpurun_out/ncu_levels.log 2>&1
for r in dilu_full levels_full; do
  ncu -i gpurun_out/$r.ncu-rep --page details --csv > gpurun_out/${r}_details.csv 2>/dev/null
  ncu -i gpurun_out/$r.ncu-rep --page raw --csv > gpurun_out/${r}_raw.csv 2>/dev/null
  ncu -i gpurun_out/$r.ncu-rep --page source --csv > gpurun_out/${r}_source.csv 2>/dev/null
done
rm -f gpurun_out/*.ncu-rep
