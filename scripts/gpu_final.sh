#!/bin/bash
# End-of-session pass: full GPU suite, smoke(), drop-in binary, the default
# bench line, the reference arm, the pageable/pinned upload numbers.
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
timeout 900 python -m pytest tests -q -m gpu -x > gpurun_out/pytest_gpu.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" > gpurun_out/smoke.log 2>&1; echo "rc=$?" >> gpurun_out/smoke.log
timeout 600 ./oracle/_ref/dropin_test > gpurun_out/dropin.log 2>&1; echo "rc=$?" >> gpurun_out/dropin.log
timeout 900 python bench.py > gpurun_out/bench.json 2> gpurun_out/bench.err; echo "bench rc=$?" >> gpurun_out/bench.err
timeout 900 python bench.py --impl reference --steps 2 --warmup 3 > gpurun_out/bench_ref.json 2> gpurun_out/bench_ref.err
timeout 500 python scripts/upload_bench.py > gpurun_out/upload.json 2> gpurun_out/upload.err
timeout 500 python scripts/asm_bench.py 128 > gpurun_out/asm_bench.json 2> gpurun_out/asm_bench.err
echo done
