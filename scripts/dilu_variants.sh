#!/bin/bash
cd "$(dirname "$0")/.."
cp paper_2403_07882_b200/lib/libbcs.so /tmp/libbcs_default.so
for v in default dilu1 dilu3; do
  if [ "$v" != default ]; then cp _variants/libbcs_$v.so paper_2403_07882_b200/lib/libbcs.so; else cp /tmp/libbcs_default.so paper_2403_07882_b200/lib/libbcs.so; fi
  echo "$v $(BCS_PROFILE=1 timeout 300 python scripts/prof_solve.py 128 2>&1 | sed -n '/solve 0/,$p' | grep 'dilu:factor\|solve 1' | tr '\n' ' ')"
done
cp /tmp/libbcs_default.so paper_2403_07882_b200/lib/libbcs.so
