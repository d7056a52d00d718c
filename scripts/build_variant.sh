#!/bin/bash
# build_variant.sh NAME "-DMACRO=V ..." : libbcs.so with k_sweep.cu/k_tail.cu
# compiled under extra macros -> _variants/libbcs_NAME.so (experiments)
set -e
cd "$(dirname "$0")/.."
make -s -C paper_2403_07882_b200/csrc >/dev/null
name=$1; shift
D=build/var_$name; mkdir -p $D _variants
NV="nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 -fmad=false -Xcompiler -fPIC,-O2,-ffp-contract=off -I/opt/prime-rl/.venv/lib/python3.12/site-packages/nvidia/nccl/include"
for f in k_sweep k_tail; do $NV "$@" -c paper_2403_07882_b200/csrc/$f.cu -o $D/$f.o; done
objs=""
for o in build/obj/*.o; do b=$(basename $o .o); if [ -f $D/$b.o ]; then objs="$objs $D/$b.o"; else objs="$objs $o"; fi; done
nvcc -gencode arch=compute_100a,code=sm_100a -shared -cudart static -o _variants/libbcs_$name.so $objs -ldl
echo built _variants/libbcs_$name.so
