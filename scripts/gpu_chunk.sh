#!/bin/bash
# chain schedule of the natural-order fine levels: bit-identity and time against the level order
cd "$GRAFT_REPO_ROOT"
BCS_CHAIN_VERBOSE=1 timeout 300 python scripts/chunk_probe.py 128 parity
BCS_CHAIN=0 timeout 300 python scripts/chunk_probe.py 128 parity
BCS_CHAIN=0 timeout 300 python scripts/chunk_probe.py 128 exact
timeout 300 python scripts/chunk_probe.py 128 exact
# small systems through the chain kernel: the parity tests against the oracle
BCS_CHAIN_MIN_WIDTH=1 timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_dropin.py -q -x -p no:cacheprovider 2>&1 | tail -3
for c in 0 1; do BCS_CHAIN=$c timeout 300 python bench.py --steps 5 --warmup 3 2>/dev/null | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('CHAIN', '$c', d['value'], d['roofline']['mean_launch_ms'], d['e2e']['value'], d['stage_s'])"; done
