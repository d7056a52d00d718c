#!/bin/bash
# solve time vs the one-CTA tail threshold (rows)
cd "$(dirname "$0")/.."
for t in 0 128 256 512 1100 2048; do
  echo "tail_rows=$t $(BCS_TAIL_ROWS=$t timeout 300 python scripts/prof_solve.py 128 2>&1 | grep 'solve 1')"
done
