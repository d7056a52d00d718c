#!/bin/bash
cd "$GRAFT_REPO_ROOT"
NCU=/usr/local/cuda/bin/ncu
for cl in 0 1; do
BCS_DENSE_PANEL_CL=$cl $NCU --metrics gpu__time_duration.sum --clock-control none -k regex:k_dense --csv --log-file gpurun_out/dense_cl$cl.csv python scripts/one_solve.py 128 parity 7 > /dev/null 2>&1; echo "ncu cl=$cl rc=$?"
done
