"""Interleaved A/B of libfa3b builds on the C4 backward shapes."""
import os, sys
import numpy as np
import torch
sys.path.insert(0, ".")
from paper_2407_08608_b200 import _lib, api

libs = []
for path in sys.argv[1:]:
    _lib._lib = None
    os.environ["FA3B_LIB"] = path
    libs.append(_lib.load())

def timeit(f, it=10):
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(it): f()
    b.record(); torch.cuda.synchronize()
    return a.elapsed_time(b) / it

cases = []
for D in (128, 64):
    for causal in (False, True):
        for N in (2048, 8192):
            B, H = 16384 // N, 2048 // D
            q, k, v, do = (torch.randn(B, N, H, D, device="cuda", dtype=torch.bfloat16) for _ in range(4))
            o, lse = api.fwd(q, k, v, causal=causal)
            ws = torch.empty(api.bwd_workspace_bytes(B, H, H, N, D), dtype=torch.uint8, device="cuda")
            g = [torch.empty_like(x) for x in (q, k, v)]
            fl = 2.5 * 4 * N * N * D * H * B / (2 if causal else 1)
            cases.append((f"bwd d{D} N{N}{' c' if causal else ''}", fl,
                          lambda q=q, k=k, v=v, do=do, o=o, lse=lse, ws=ws, g=g, c=causal:
                          api.bwd(q, k, v, o, do, lse, causal=c, dq=g[0], dk=g[1], dv=g[2], workspace=ws)))
res = {(c[0], i): [] for c in cases for i in range(len(libs))}
for name, fl, f in cases:
    for L in libs:
        _lib._lib = L
        for _ in range(3): f()
    torch.cuda.synchronize()
    for rnd in range(7):
        for i, L in enumerate(libs):
            _lib._lib = L
            res[(name, i)].append(fl / timeit(f) / 1e9)
for name, _, _ in cases:
    print(f"{name:16s} " + " | ".join(f"{np.median(res[(name, i)]):7.0f}" for i in range(len(libs))), flush=True)
print("libs:", " | ".join(sys.argv[1:]))
