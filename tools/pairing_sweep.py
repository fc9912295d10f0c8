"""Forward TFLOP/s on the C2/C3/C5 shapes for the current FA3B_FWD_PAIRING setting
(run alternately with cta / warp / unset to compare pairings)."""
import os, sys
import numpy as np, torch
sys.path.insert(0, ".")
from paper_2407_08608_b200 import api

def timeit(f, it=10):
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(it): f()
    b.record(); torch.cuda.synchronize()
    return a.elapsed_time(b) / it

out = []
for D, causal, fp8 in ((128, False, False), (128, True, False), (64, False, False), (64, True, False),
                       (128, False, True), (128, True, True)):
    N, B, H = 8192, 2, 2048 // D
    q, k, v = (torch.randn(B, N, H, D, device="cuda", dtype=torch.bfloat16) for _ in range(3))
    if fp8:
        p = [api.fp8_prepare(x, block_rows=128, hadamard=i < 2, seed=1) for i, x in enumerate((q, k, v))]
        f = lambda: api.fwd(p[0][0], p[1][0], p[2][0], causal=causal, q_scale=p[0][1], k_scale=p[1][1], v_scale=p[2][1])
    else:
        f = lambda: api.fwd(q, k, v, causal=causal)
    for _ in range(3): f()
    torch.cuda.synchronize()
    fl = 4 * N * N * D * H * B / (2 if causal else 1)
    out.append(f"{'fp8' if fp8 else 'bf16'} d{D}{'c' if causal else ''} {np.median([fl / timeit(f) / 1e9 for _ in range(5)]):.0f}")
q = torch.randn(1, 8192, 64, 128, device="cuda", dtype=torch.bfloat16)
k, v = (torch.randn(1, 8192, 8, 128, device="cuda", dtype=torch.bfloat16) for _ in range(2))
for causal in (False, True):
    f = lambda: api.fwd(q, k, v, causal=causal)
    for _ in range(3): f()
    out.append(f"C5{'c' if causal else ''} {np.median([4 * 8192 * 8192 * 128 * 64 / (2 if causal else 1) / timeit(f) / 1e9 for _ in range(5)]):.0f}")
print(f"{os.environ.get('FA3B_FWD_PAIRING', 'auto'):5s} " + " | ".join(out), flush=True)
