#!/bin/bash
# variant_cmp.sh NAME... : time each _variants/libbcs_NAME.so (default = the in-tree build)
cd "$(dirname "$0")/.."
cp paper_2403_07882_b200/lib/libbcs.so /tmp/libbcs_default.so
for rep in 1 2; do
for v in "$@"; do
  if [ "$v" = default ]; then cp /tmp/libbcs_default.so paper_2403_07882_b200/lib/libbcs.so
  else cp _variants/libbcs_$v.so paper_2403_07882_b200/lib/libbcs.so; fi
  echo "$v: $(timeout 300 python scripts/variant_time.py 128 2>&1 | tail -1)"
done
done
cp /tmp/libbcs_default.so paper_2403_07882_b200/lib/libbcs.so
