"""Quick timing of the backward (C4 shapes) through the C ABI."""
import sys
import torch
sys.path.insert(0, ".")
from paper_2407_08608_b200 import api

for D in (128, 64):
    for causal in (False, True):
        for N in (2048, 8192):
            B, H = 16384 // N, 2048 // D
            q, k, v, do = (torch.randn(B, N, H, D, device="cuda", dtype=torch.bfloat16) for _ in range(4))
            o, lse = api.fwd(q, k, v, causal=causal)
            ws = torch.empty(api.bwd_workspace_bytes(B, H, H, N, D), dtype=torch.uint8, device="cuda")
            dq, dk, dv = (torch.empty_like(x) for x in (q, k, v))
            for _ in range(3):
                api.bwd(q, k, v, o, do, lse, causal=causal, dq=dq, dk=dk, dv=dv, workspace=ws)
            torch.cuda.synchronize()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            for _ in range(10):
                api.bwd(q, k, v, o, do, lse, causal=causal, dq=dq, dk=dk, dv=dv, workspace=ws)
            e1.record()
            torch.cuda.synchronize()
            ms = e0.elapsed_time(e1) / 10
            fl = 2.5 * 4 * N * N * D * H * B / (2 if causal else 1)
            print(f"bwd D={D} N={N} causal={causal}: {ms:.3f} ms {fl/ms/1e9:.1f} TFLOP/s", flush=True)
