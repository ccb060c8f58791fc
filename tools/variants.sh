#!/bin/bash
# Build-time variants of the CUDA library for A/B timing on the GPU box:
#   tools/variants.sh NAME "-DMACRO=V ..." [NAME "-D..." ...]
# -> paper_1204_0069_b200/_lib/variants/NAME/libcoopcg_gpu.so, selected at run
# time with COOPCG_LIB_PATH (paper_1204_0069_b200/_capi.py).  refgen.cu is
# compiled once and shared.
set -e
cd "$(dirname "$0")/.."
CS=paper_1204_0069_b200/csrc
OUT=paper_1204_0069_b200/_lib/variants
F="-gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 -Xcompiler -fPIC"
mkdir -p $OUT
[ -f $OUT/refgen.o ] || nvcc $F -c -o $OUT/refgen.o $CS/refgen.cu
pids=()
while [ $# -ge 2 ]; do
  name=$1; defs=$2; shift 2
  mkdir -p $OUT/$name
  ( nvcc $F $defs -c -o $OUT/$name/coopcg_gpu.o $CS/coopcg_gpu.cu && \
    nvcc -gencode arch=compute_100a,code=sm_100a -shared -o $OUT/$name/libcoopcg_gpu.so $OUT/$name/coopcg_gpu.o $OUT/refgen.o && \
    rm $OUT/$name/coopcg_gpu.o && echo "built $name ($defs)" ) &
  pids+=($!)
done
for p in "${pids[@]}"; do wait $p; done
