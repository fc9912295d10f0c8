#!/bin/bash
# Build libfa3b.so with extra -D flags into build/variants/<name>.so for A/B runs
# (tools/ab.py loads several builds in one process). Usage: tools/variant.sh name -DX=1 ...
set -e
name=$1; shift
root=$(cd "$(dirname "$0")/.." && pwd)
obj=$root/build/variants/obj_$name
mkdir -p "$obj"
srcs=$(python -c "import sys; sys.path.insert(0, '$root'); from paper_2407_08608_b200 import build as b; print(' '.join(b.CUDA_SOURCES))")
pids=()
for s in $srcs; do
  nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 -Xcompiler -fPIC \
    -Xcompiler -fvisibility=hidden -I "$root/include" "$@" -c -o "$obj/${s%.cu}.o" \
    "$root/paper_2407_08608_b200/csrc/$s" &
  pids+=($!)
done
for p in "${pids[@]}"; do wait $p; done
nvcc -gencode arch=compute_100a,code=sm_100a -shared -Xlinker --no-undefined \
  -o "$root/build/variants/$name.so" "$obj"/*.o -lcuda
echo "built build/variants/$name.so"
