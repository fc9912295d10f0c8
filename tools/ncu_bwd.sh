#!/bin/bash
# ncu full capture of one backward K3 launch: bash tools/ncu_bwd.sh <tag> <D> <causal 0/1>
TAG=$1; D=${2:-128}; C=${3:-0}
cat > /tmp/ncu_bwd.py <<PY
import sys, torch
sys.path.insert(0, ".")
from paper_2407_08608_b200 import api
D, C = $D, bool($C)
N, B, H = 8192, 2, 2048 // D
q, k, v, do = (torch.randn(B, N, H, D, device="cuda", dtype=torch.bfloat16) for _ in range(4))
o, lse = api.fwd(q, k, v, causal=C)
for _ in range(3): api.bwd(q, k, v, o, do, lse, causal=C)
torch.cuda.synchronize()
PY
ncu --set full --clock-control none --import-source on -k regex:fa3b_bwd_kernel -s 1 -c 1 -o gpurun_out/${TAG} python /tmp/ncu_bwd.py > gpurun_out/${TAG}.log 2>&1
echo "ncu $TAG rc=$?"
