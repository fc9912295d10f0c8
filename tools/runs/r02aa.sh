set -u
mkdir -p gpurun_out
T=r02aa
cat > /tmp/ppcheck.py <<'PY'
import os, sys, torch
sys.path.insert(0, ".")
os.environ["FA3B_LIB"] = "build/variants/ppbar.so"
from paper_2407_08608_b200 import api
for causal in (False, True):
    for n in (300, 1000, 4173):
        q, k, v = (torch.randn(2, n, 16, 128, device="cuda", dtype=torch.bfloat16) for _ in range(3))
        o, l = api.fwd(q, k, v, causal=causal)
        torch.cuda.synchronize()
print("ppbar smoke ok")
PY
timeout 120 python /tmp/ppcheck.py > gpurun_out/${T}_ppcheck.log 2>&1; echo "ppcheck rc=$?"
if grep -q "smoke ok" gpurun_out/${T}_ppcheck.log; then
  timeout 900 python tools/ab.py paper_2407_08608_b200/libfa3b.so build/variants/ppbar.so > gpurun_out/${T}_ppbar_ab.log 2>&1; echo "ab rc=$?"
  FA3B_LIB=build/variants/ppbar.so timeout 600 python -m pytest tests/test_fwd_gpu.py tests/test_fp8_gpu.py -x -q -k "matches_oracle or error_band or many_items or full_size" > gpurun_out/${T}_pytest_ppbar.log 2>&1; echo "pytest rc=$?"
fi
