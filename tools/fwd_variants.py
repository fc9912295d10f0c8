"""Time the forward for one library variant (FA3B_LIB) on the headline shapes."""
import os, sys
import torch
sys.path.insert(0, ".")
from paper_2407_08608_b200 import api

tag = os.environ.get("FA3B_LIB", "default")
def t(f, it=20):
    for _ in range(3): f()
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(it): f()
    b.record(); torch.cuda.synchronize()
    return a.elapsed_time(b) / it
out = []
for D, causal in ((128, False), (128, True), (64, False), (256, False)):
    N, B, H = 8192, 2, 2048 // D
    q, k, v = (torch.randn(B, N, H, D, device="cuda", dtype=torch.bfloat16) for _ in range(3))
    ms = t(lambda: api.fwd(q, k, v, causal=causal))
    out.append(f"bf16 d{D}{'c' if causal else ''} {4*N*N*D*H*B/(2 if causal else 1)/ms/1e9:.0f}")
    if D >= 128 and not causal:
        p = [api.fp8_prepare(x, block_rows=128, hadamard=i < 2, seed=1) for i, x in enumerate((q, k, v))]
        ms = t(lambda: api.fwd(p[0][0], p[1][0], p[2][0], q_scale=p[0][1], k_scale=p[1][1], v_scale=p[2][1]))
        out.append(f"fp8 d{D} {4*N*N*D*H*B/ms/1e9:.0f}")
        p = [api.fp8_prepare(x, block_rows=0, hadamard=i < 2, seed=1) for i, x in enumerate((q, k, v))]
        ms = t(lambda: api.fwd(p[0][0], p[1][0], p[2][0], q_scale=p[0][1], k_scale=p[1][1], v_scale=p[2][1], q_block_rows=0, kv_block_rows=0))
        out.append(f"fp8pt d{D} {4*N*N*D*H*B/ms/1e9:.0f}")
print(os.path.basename(tag), " | ".join(out), flush=True)
