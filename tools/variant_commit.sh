#!/bin/bash
# Build libfa3b.so of a git commit into build/variants/<name>.so (baseline for tools/ab.py):
# tools/variant_commit.sh <commit> <name>
set -e
c=$1; name=$2
root=$(cd "$(dirname "$0")/.." && pwd)
wt=/tmp/fa3b_wt_$name
rm -rf "$wt"; git -C "$root" worktree add -f "$wt" "$c" > /dev/null 2>&1
obj=$root/build/variants/obj_$name; mkdir -p "$obj"
srcs=$(cd "$wt" && python -c "from paper_2407_08608_b200 import build as b; print(' '.join(b.CUDA_SOURCES))")
for s in $srcs; do
  nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 -Xcompiler -fPIC \
    -Xcompiler -fvisibility=hidden -I "$wt/include" -c -o "$obj/${s%.cu}.o" "$wt/paper_2407_08608_b200/csrc/$s" &
done
wait
nvcc -gencode arch=compute_100a,code=sm_100a -shared -o "$root/build/variants/$name.so" "$obj"/*.o -lcuda
git -C "$root" worktree remove --force "$wt"
echo "built build/variants/$name.so from $c"
