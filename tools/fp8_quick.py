"""FP8 path timing (K5 prepare, K6 forward) and an RMSE probe vs fp64 torch."""
import math, os, sys
import torch
sys.path.insert(0, ".")
from paper_2407_08608_b200 import api

thr = os.environ.get("FA3B_FP8_THR", "4")
# RMSE probe on outlier-like data (N(0,1) + 10 N(0,1) Bern(1e-3)), fp64 reference
g = torch.Generator(device="cuda").manual_seed(0)
N, D = 4096, 128
def outl(): 
    x = torch.randn(1, N, 1, D, device="cuda", generator=g, dtype=torch.float64)
    m = torch.rand(1, N, 1, D, device="cuda", generator=g, dtype=torch.float64) < 1e-3
    return x + 10 * torch.randn(1, N, 1, D, device="cuda", generator=g, dtype=torch.float64) * m
q, k, v = outl(), outl(), outl()
s = (q[0, :, 0] @ k[0, :, 0].T) / math.sqrt(D)
ref = torch.softmax(s, -1) @ v[0, :, 0]
for pb, inc in ((True, True), (True, False), (False, True), (False, False)):
    o, _ = api.fp8_fwd(q.float(), k.float(), v.float(), per_block=pb, incoherent=inc, seed=5, out_dtype=torch.float32)
    e = (o[0, :, 0].double() - ref).pow(2).mean().sqrt().item()
    print(f"thr={thr} per_block={pb} incoherent={inc}: rmse {e:.5f}", flush=True)
if thr != "4":
    sys.exit(0)
for D, causal in ((128, False), (128, True), (256, False), (256, True)):
    N = 8192; B = 2; H = 2048 // D
    x = [torch.randn(B, N, H, D, device="cuda", dtype=torch.bfloat16) for _ in range(3)]
    p = [api.fp8_prepare(t, block_rows=128, hadamard=(i < 2), seed=1) for i, t in enumerate(x)]
    for sched in (["pingpong", "basic"] if D == 128 else ["basic"]):
        f = lambda: api.fwd(p[0][0], p[1][0], p[2][0], causal=causal, schedule=sched, q_scale=p[0][1], k_scale=p[1][1], v_scale=p[2][1])
        for _ in range(3): f()
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(20): f()
        e1.record(); torch.cuda.synchronize()
        ms = e0.elapsed_time(e1) / 20
        fl = 4 * N * N * D * H * B / (2 if causal else 1)
        print(f"fp8 fwd D={D} causal={causal} {sched}: {ms:.3f} ms {fl/ms/1e9:.1f} TFLOP/s", flush=True)
    e0.record()
    for _ in range(20): api.fp8_prepare(x[0], block_rows=128, hadamard=True, seed=1)
    e1.record(); torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / 20
    by = x[0].numel() * 3
    print(f"fp8 prepare D={D}: {ms*1e3:.1f} us {by/ms/1e6:.1f} GB/s", flush=True)
