#!/bin/bash
# ncu full capture of one forward kernel: bash tools/ncu_fwd.sh <tag> <D> <causal 0/1> <fp8 0/1>
TAG=$1; D=${2:-128}; C=${3:-0}; F=${4:-0}
cat > /tmp/ncu_one.py <<PY
import sys, torch
sys.path.insert(0, ".")
from paper_2407_08608_b200 import api
D, C, F = $D, bool($C), bool($F)
N, B, H = 8192, 2, 2048 // D
q, k, v = (torch.randn(B, N, H, D, device="cuda", dtype=torch.bfloat16) for _ in range(3))
if F:
    p = [api.fp8_prepare(x, block_rows=128, hadamard=i < 2, seed=1, scale_pow2=i == 2) for i, x in enumerate((q, k, v))]
    f = lambda: api.fwd(p[0][0], p[1][0], p[2][0], causal=C, q_scale=p[0][1], k_scale=p[1][1], v_scale=p[2][1])
else:
    f = lambda: api.fwd(q, k, v, causal=C)
for _ in range(4): f()
torch.cuda.synchronize()
PY
ncu --set full --clock-control none --import-source on -k regex:fa3b_fwd_kernel -s 3 -c 1 -o gpurun_out/${TAG} python /tmp/ncu_one.py > gpurun_out/${TAG}.log 2>&1
echo "ncu $TAG rc=$?"
