#!/bin/bash
# the reference's own acceptance program (criteria 1-9, proj/tests/acceptance_main.cpp)
# with every runCase linear solve on the B200 (BCS_INTERPOSE=parity|exact) and,
# for comparison, unchanged (off); oracle/_ref/acceptance_b200 (oracle/Makefile)
cd "$GRAFT_REPO_ROOT"
for mode in parity exact off; do
  for c in 1 2 3 4 5 6 7 8 9; do
    s=$(date +%s%N)
    out=$(BCS_INTERPOSE=$mode timeout 1200 ./oracle/_ref/acceptance_b200 $c 2>&1 | tail -1)
    e=$(date +%s%N)
    echo "$mode  ($(( (e - s) / 1000000 )) ms)  $out"
  done
done
# the reference's own unit tests (proj/tests/test_*.cpp) with the same interposition
for mode in parity exact off; do
  BCS_INTERPOSE=$mode timeout 1200 ./oracle/_ref/unit_tests_b200 > gpurun_out/unit_$mode.log 2>&1
  echo "unit tests $mode rc=$?: $(tail -1 gpurun_out/unit_$mode.log)"
  grep "^FAIL" gpurun_out/unit_$mode.log | head -20
done
