#!/bin/bash
# Round-2 schedule experiments behind the DESIGN.md measurements (one GPU box):
#   chain schedule (BCS_CHAIN), several clusters per level (BCS_CL_PARTS / BCS_CL_WIDTH),
#   the performance mode's per-colour launch threshold (BCS_MC_LAUNCH_MIN).
# Every variant reorders work only; tests/test_gpu_chain.py and test_gpu_cluster_parts.py check bit-identity.
cd "$GRAFT_REPO_ROOT"
line() {  # label, then env assignments and bench flags
  label=$1; shift
  env "$@" timeout 300 python bench.py --steps 5 --warmup 3 --no-cpu-baseline --no-e2e $BENCH_FLAGS 2>/dev/null | tail -1 | \
    python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$label', d['value'], d['iterations'], d['roofline']['mean_launch_ms'])"
}
line "level order" BCS_CHAIN=0
line "chain schedule" BCS_CHAIN=1
for w in 40 60 100 200; do line "one cluster up to width $w" BCS_CL_WIDTH=$w; done
line "up to 9 clusters, width 40" BCS_CL_PARTS=9
line "up to 9 clusters, width 30" BCS_CL_PARTS=9 BCS_CL_WIDTH=30
BENCH_FLAGS="--mode perf"
for m in 0 2048 16384 65536; do line "perf mode, per-colour launches from $m rows per colour" BCS_MC_LAUNCH_MIN=$m; done
