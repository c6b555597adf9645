#!/bin/bash
# Build an experimental variant of the library with extra -D flags:
#   tools/build_variant.sh NAME -DFOO=1 ...   -> build_exp/lib_NAME.so
# (select it at run time with SINKHORN_B200_LIB=build_exp/lib_NAME.so)
set -e
ROOT="$(cd "$(dirname "$0")/.." && pwd)"
name="$1"; shift
mkdir -p "$ROOT/build_exp"
cd "$ROOT/paper_1907_01729_b200/csrc"
nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 -Xcompiler -fPIC \
  -Xcompiler -fvisibility=hidden -shared -cudart static "$@" \
  -o "$ROOT/build_exp/lib_$name.so" sinkhorn_abi.cu
