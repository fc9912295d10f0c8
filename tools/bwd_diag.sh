#!/bin/bash
# backward diagnosis: timing with and without the dQ atomics, and one ncu capture
mkdir -p gpurun_out
./tools/mma_bench > gpurun_out/mma_bench2.txt 2>&1
timeout 300 python tools/bwd_quick.py > gpurun_out/bwd_base.log 2>&1
FA3B_LIB=build/norred/libfa3b.so timeout 300 python tools/bwd_quick.py > gpurun_out/bwd_norred.log 2>&1
cat > /tmp/bwd_one.py <<'PY'
import sys, torch
sys.path.insert(0, ".")
from paper_2407_08608_b200 import api
B, N, H, D = 2, 8192, 16, 128
q, k, v, do = (torch.randn(B, N, H, D, device="cuda", dtype=torch.bfloat16) for _ in range(4))
o, lse = api.fwd(q, k, v)
for _ in range(3): api.bwd(q, k, v, o, do, lse)
torch.cuda.synchronize()
PY
timeout 600 ncu --set full --clock-control none --import-source on -k regex:fa3b_bwd_kernel -s 1 -c 1 -o gpurun_out/bwd_prof python /tmp/bwd_one.py > gpurun_out/bwd_ncu.log 2>&1
echo done
