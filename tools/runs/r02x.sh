set -u
mkdir -p gpurun_out
T=r02x
timeout 900 python -m pytest tests/test_bwd_gpu.py tests/test_large_oracle_gpu.py -x -q -k "bwd" > gpurun_out/${T}_pytest_bwd.log 2>&1; echo "pytest bwd rc=$?"
timeout 900 python tools/ab_bwd.py build/variants/prev.so paper_2407_08608_b200/libfa3b.so > gpurun_out/${T}_bwd_ab.log 2>&1; echo "ab rc=$?"
cat > /tmp/det.py <<'PY'
import sys, json, torch
sys.path.insert(0, ".")
from paper_2407_08608_b200 import api
for d in (128, 64):
    for causal in (False, True):
        B, N, H = 2, 8192, 2048 // d
        q, k, v, do = (torch.randn(B, N, H, d, device="cuda", dtype=torch.bfloat16) for _ in range(4))
        o, lse = api.fwd(q, k, v, causal=causal)
        ws = torch.empty(api.bwd_workspace_bytes(B, H, H, N, d), dtype=torch.uint8, device="cuda")
        for det in (False, True):
            f = lambda: api.bwd(q, k, v, o, do, lse, causal=causal, workspace=ws, deterministic=det)
            for _ in range(3): f()
            torch.cuda.synchronize()
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a.record()
            for _ in range(10): f()
            b.record(); torch.cuda.synchronize()
            ms = a.elapsed_time(b) / 10
            fl = 2.5 * 4 * N * N * d * H * B / (2 if causal else 1)
            print(json.dumps({"d": d, "causal": causal, "deterministic": det, "tflops": round(fl / ms / 1e9, 1)}), flush=True)
PY
timeout 300 python /tmp/det.py > gpurun_out/${T}_det.log 2>&1; echo "det rc=$?"
