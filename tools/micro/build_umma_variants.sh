#!/bin/bash
# Compile umma_gemm_bench variants (pipeline depths / promotion) for one gpurun sweep.
set -e
cd "$(dirname "$0")"
rm -f umv_*
I=../../paper_1907_01729_b200/csrc
F="-gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -I$I -lcuda"
build() { nvcc $F "$@" -o "umv_$(echo "$@" | tr -d ' =-' | tr 'D' '_')" umma_gemm_bench.cu & }
build -DSKB_UM_SUB=2
build -DSKB_UM_SUB=2 -DSKB_UM_DBG_NOSPLIT
wait
ls umv_*
