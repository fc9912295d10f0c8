"""Interleaved A/B of the backward (K2 + K3 + K4) across libfa3b.so builds, like
tools/ab.py: C4 shapes at N 8192 (BWD_N=512,1024,... for others). Usage: python tools/bwd_ab.py lib1.so lib2.so ..."""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2407_08608_b200 import _lib, api  # noqa: E402

libs = []
for path in sys.argv[1:]:
    _lib._lib = None
    os.environ["FA3B_LIB"] = path
    libs.append(_lib.load())


def timeit(f, it=5):
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(it):
        f()
    b.record()
    torch.cuda.synchronize()
    return a.elapsed_time(b) / it


cases = []
NS = [int(x) for x in os.environ.get("BWD_N", "8192").split(",")]  # C4 lengths (B = 16384 / N)
for N, D, causal, det in [(n, *c) for n in NS for c in ((128, False, False), (128, True, False), (64, False, False),
                                                       (128, False, True))]:
    B, H = 16384 // N, 2048 // D
    q, k, v, do = (torch.randn(B, N, H, D, device="cuda", dtype=torch.bfloat16) for _ in range(4))
    _lib._lib = libs[0]
    o, lse = api.fwd(q, k, v, causal=causal)
    ws = torch.empty(api.bwd_workspace_bytes(B, H, H, N, D), dtype=torch.uint8, device="cuda")
    g = [torch.empty_like(q) for _ in range(3)]
    fl = 2.5 * 4 * N * N * D * H * B / (2 if causal else 1)
    cases.append((f"N{N} d{D}{'c' if causal else ''}{'det' if det else ''}", fl,
                  (lambda q=q, k=k, v=v, o=o, do=do, lse=lse, c=causal, ws=ws, g=g, det=det:
                   api.bwd(q, k, v, o, do, lse, causal=c, dq=g[0], dk=g[1], dv=g[2], workspace=ws,
                           deterministic=det))))
res = {(c[0], i): [] for c in cases for i in range(len(libs))}
for name, fl, f in cases:
    for i, L in enumerate(libs):
        _lib._lib = L
        for _ in range(2):
            f()
    torch.cuda.synchronize()
    for rnd in range(5):
        for i, L in enumerate(libs):
            _lib._lib = L
            res[(name, i)].append(fl / timeit(f) / 1e9)
for name, _, _ in cases:
    print(f"{name:12s} " + " | ".join(f"{np.median(res[(name, i)]):7.0f}" for i in range(len(libs))), flush=True)
print("libs:", " | ".join(sys.argv[1:]))
