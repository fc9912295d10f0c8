"""Quick on-device check of the forward kernel against a torch fp32 reference."""
import math, sys, time
import torch
sys.path.insert(0, ".")
from paper_2407_08608_b200 import api

def ref(q, k, v, causal, alpha):
    qf, kf, vf = (x.float().transpose(1, 2) for x in (q, k, v))  # B H N D
    H, Hkv = qf.shape[1], kf.shape[1]
    if Hkv != H:
        kf = kf.repeat_interleave(H // Hkv, 1); vf = vf.repeat_interleave(H // Hkv, 1)
    s = alpha * qf @ kf.transpose(-1, -2)
    if causal:
        N = s.shape[-1]
        m = torch.ones(N, N, dtype=torch.bool, device=s.device).triu(1)
        s = s.masked_fill(m, float("-inf"))
    lse = torch.logsumexp(s, -1)
    o = torch.softmax(s, -1) @ vf
    return o.transpose(1, 2), lse

torch.manual_seed(0)
fails = 0
for (B, N, H, Hkv, D, causal, dt, sched, alpha) in [
    (1, 128, 1, 1, 128, False, torch.bfloat16, "basic", None),
    (1, 256, 1, 1, 128, False, torch.bfloat16, "pingpong", None),
    (2, 512, 8, 8, 64, False, torch.float16, "pingpong", None),
    (2, 512, 8, 8, 64, False, torch.float16, "basic", None),
    (1, 1000, 4, 2, 128, True, torch.bfloat16, "pingpong", None),
    (1, 1000, 4, 2, 128, False, torch.bfloat16, "pingpong", -0.1),
    (1, 777, 2, 1, 256, True, torch.bfloat16, "basic", None),
    (1, 300, 2, 2, 64, True, torch.float16, "pingpong", 0.3),
    (2, 2048, 4, 4, 128, True, torch.bfloat16, "basic", None),
]:
    q = torch.randn(B, N, H, D, device="cuda", dtype=dt)
    k = torch.randn(B, N, Hkv, D, device="cuda", dtype=dt)
    v = torch.randn(B, N, Hkv, D, device="cuda", dtype=dt)
    a = alpha if alpha is not None else 1 / math.sqrt(D)
    try:
        o, lse = api.fwd(q, k, v, causal=causal, alpha=a, schedule=sched)
        torch.cuda.synchronize()
    except Exception as e:
        print("FAIL launch", (B, N, H, Hkv, D, causal, dt, sched), e); fails += 1; continue
    ro, rl = ref(q, k, v, causal, a)
    eo = (o.float() - ro).abs().max().item(); el = (lse - rl).abs().max().item()
    ok = eo < 2e-2 and el < 1e-3
    fails += not ok
    print("ok " if ok else "BAD", (B, N, H, Hkv, D, causal, str(dt), sched, alpha), f"max|dO|={eo:.3e} max|dL|={el:.3e}", flush=True)

# timing
for D, causal in [(128, False), (128, True), (64, False), (256, False)]:
    N = 4096; H = 2048 // D; B = 16384 // N
    q = torch.randn(B, N, H, D, device="cuda", dtype=torch.bfloat16)
    k = torch.randn_like(q); v = torch.randn_like(q)
    for sched in (["pingpong", "basic"] if D < 256 else ["basic"]):
        for _ in range(3): api.fwd(q, k, v, causal=causal, schedule=sched)
        torch.cuda.synchronize()
        e0 = torch.cuda.Event(enable_timing=True); e1 = torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(20): api.fwd(q, k, v, causal=causal, schedule=sched)
        e1.record(); torch.cuda.synchronize()
        ms = e0.elapsed_time(e1) / 20
        fl = 4 * N * N * D * H * B / (2 if causal else 1)
        print(f"D={D} causal={causal} {sched}: {ms:.3f} ms  {fl/ms/1e9:.1f} TFLOP/s", flush=True)
sys.exit(1 if fails else 0)
