set -u
mkdir -p gpurun_out
T=r02q
timeout 900 python -m pytest tests/test_fp8_gpu.py -x -q -k "error_band or many_items or bad or reject" > gpurun_out/${T}_pytest_fp8.log 2>&1; echo "pytest fp8 rc=$?"
cat > /tmp/fp8d64.py <<'PY'
import sys, json, torch
sys.path.insert(0, ".")
from paper_2407_08608_b200 import api
for causal in (False, True):
    for n in (2048, 8192):
        B, H, d = 16384 // n, 32, 64
        x = [torch.randn(B, n, H, d, device="cuda", dtype=torch.bfloat16) for _ in range(3)]
        p = [api.fp8_prepare(t, block_rows=128, hadamard=i < 2, seed=1, scale_pow2=i == 2) for i, t in enumerate(x)]
        f = lambda: api.fwd(p[0][0], p[1][0], p[2][0], causal=causal, q_scale=p[0][1], k_scale=p[1][1], v_scale=p[2][1])
        for _ in range(3): f()
        torch.cuda.synchronize()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        for _ in range(20): f()
        b.record(); torch.cuda.synchronize()
        ms = a.elapsed_time(b) / 20
        fl = 4 * n * n * d * H * B / (2 if causal else 1)
        print(json.dumps({"d": d, "n": n, "causal": causal, "tflops": round(fl / ms / 1e9, 1)}))
PY
timeout 300 python /tmp/fp8d64.py > gpurun_out/${T}_fp8d64.log 2>&1; echo "time rc=$?"
