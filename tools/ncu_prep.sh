#!/bin/bash
# ncu full capture of the K5 fast kernel (d 128, Hadamard): bash tools/ncu_prep.sh <tag> [env...]
TAG=$1; shift
cat > /tmp/ncu_prep.py <<'PY'
import sys, torch
sys.path.insert(0, ".")
from paper_2407_08608_b200 import api
x = torch.randn(2, 8192, 16, 128, device="cuda", dtype=torch.bfloat16)
for _ in range(3):
    api.fp8_prepare(x, block_rows=128, hadamard=True, seed=1)
torch.cuda.synchronize()
PY
env "$@" ncu --set full --clock-control none --import-source on -k regex:fp8_prepare -s 2 -c 1 -o gpurun_out/${TAG} python /tmp/ncu_prep.py > gpurun_out/${TAG}.log 2>&1
echo "ncu $TAG rc=$?"
