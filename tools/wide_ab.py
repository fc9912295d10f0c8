"""A/B of a forward kernel variant selected by an environment variable (read
once per process): times C2-shape forwards (B x N = 16k tokens, H x d = 2048)
and checks the output against fp32 torch on sampled rows.
  python tools/wide_ab.py  (prints one JSON line per point; run once per env value)"""
import json
import math
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2407_08608_b200 import api  # noqa: E402


def bench(fn, iters=30):
    for _ in range(3):
        fn()
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(iters):
        fn()
    b.record()
    torch.cuda.synchronize()
    return a.elapsed_time(b) / iters


tag = " ".join(f"{k}={v}" for k, v in os.environ.items() if k.startswith("FA3B_"))
DIMS = [int(x) for x in os.environ.get("AB_DIMS", "128,64").split(",")]
pts = [(d, n, c, dt) for dt in ("bf16", "e4m3") for d in DIMS for n in (2048, 8192)
       for c in (False, True) if not (dt == "e4m3" and d == 64)]
for d, n, causal, dt in pts:
    B, H = 16384 // n, 2048 // d
    g = torch.Generator(device="cuda").manual_seed(n + d)
    q, k, v = (torch.randn(B, n, H, d, device="cuda", generator=g).bfloat16() for _ in range(3))
    if dt == "e4m3":
        pr = [api.fp8_prepare(x, block_rows=128, hadamard=i < 2, seed=1, scale_pow2=i == 2) for i, x in enumerate((q, k, v))]
        fn = lambda: api.fwd(pr[0][0], pr[1][0], pr[2][0], causal=causal, q_scale=pr[0][1],  # noqa: E731
                             k_scale=pr[1][1], v_scale=pr[2][1])
    else:
        fn = lambda: api.fwd(q, k, v, causal=causal)  # noqa: E731
    o, lse = fn()
    rows = torch.tensor([0, 1, 127, 128, n // 2 + 3, n - 1], device="cuda")
    s = q[0, rows, 1].float() @ k[0, :, 1].float().T / math.sqrt(d)
    if causal:
        s = s.masked_fill(torch.arange(n, device="cuda")[None, :] > rows[:, None], -math.inf)
    ref = torch.softmax(s, -1) @ v[0, :, 1].float()
    err = (o[0, rows, 1].float() - ref).abs().max().item()
    lerr = (lse[0, 1, rows] - torch.logsumexp(s, -1)).abs().max().item()
    ms = bench(fn)
    f = 4 * n * n * d * H * B / (2 if causal else 1)
    print(json.dumps({"env": tag, "dtype": dt, "d": d, "n": n, "causal": causal,
                      "tflops": round(f / ms / 1e9, 1), "maxerr": round(err, 5),
                      "lse_err": round(lerr, 6)}), flush=True)
