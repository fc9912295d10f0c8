#!/bin/bash
# Build libfa3b.so with extra -D flags into build/variants/<name>.so for A/B runs
# (tools/ab.py loads several builds in one process). Usage: tools/variant.sh name -DX=1 ...
set -e
name=$1; shift
mkdir -p build/variants
cd paper_2407_08608_b200/csrc
nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 -Xcompiler -fPIC \
  -Xcompiler -fvisibility=hidden -shared -Xlinker --no-undefined -I ../../include "$@" \
  -o ../../build/variants/$name.so fa3b_capi.cu fwd_fp8.cu fp8_prepare.cu bwd.cu
