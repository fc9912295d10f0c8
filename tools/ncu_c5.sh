#!/bin/bash
# ncu full capture of the C5 forward (Llama-3-70B GQA 64/8, N 8192, causal, B1):
# bash tools/ncu_c5.sh <tag> <fp8 0/1>
TAG=$1; F=${2:-0}
cat > /tmp/ncu_c5.py <<PY
import sys, torch
sys.path.insert(0, ".")
from paper_2407_08608_b200 import api
F = bool($F)
q = torch.randn(1, 8192, 64, 128, device="cuda", dtype=torch.bfloat16)
k, v = (torch.randn(1, 8192, 8, 128, device="cuda", dtype=torch.bfloat16) for _ in range(2))
if F:
    p = [api.fp8_prepare(x, block_rows=128, hadamard=i < 2, seed=1, scale_pow2=i == 2) for i, x in enumerate((q, k, v))]
    f = lambda: api.fwd(p[0][0], p[1][0], p[2][0], causal=True, q_scale=p[0][1], k_scale=p[1][1], v_scale=p[2][1])
else:
    f = lambda: api.fwd(q, k, v, causal=True)
for _ in range(4): f()
torch.cuda.synchronize()
PY
ncu --set full --clock-control none --import-source on -k regex:fa3b_fwd_kernel -s 3 -c 1 -o gpurun_out/${TAG} python /tmp/ncu_c5.py > gpurun_out/${TAG}.log 2>&1
echo "ncu $TAG rc=$?"
