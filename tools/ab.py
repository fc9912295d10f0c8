"""Interleaved A/B timing of several libfa3b.so builds in one process (each build
loaded as its own ctypes handle; rounds alternate between builds so clock and
power drift hit all of them alike). Usage: python tools/ab.py lib1.so lib2.so ..."""
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
for D, causal in ((128, False), (128, True), (64, False), (256, False)):
    N, B, H = 8192, 2, 2048 // D
    q, k, v = (torch.randn(B, N, H, D, device="cuda", dtype=torch.bfloat16) for _ in range(3))
    fl = 4 * N * N * D * H * B / (2 if causal else 1)
    cases.append((f"bf16 d{D}{'c' if causal else ''}", fl, (lambda q=q, k=k, v=v, c=causal: api.fwd(q, k, v, causal=c))))
    if D >= 128 and not causal:
        for blk, nm in ((128, "fp8"), (0, "fp8pt")):
            _lib._lib = libs[-1]
            p = [api.fp8_prepare(x, block_rows=blk, hadamard=i < 2, seed=1, scale_pow2=(i == 2 and blk > 0)) for i, x in enumerate((q, k, v))]
            cases.append((f"{nm} d{D}", fl, (lambda p=p, blk=blk: api.fwd(p[0][0], p[1][0], p[2][0], q_scale=p[0][1], k_scale=p[1][1], v_scale=p[2][1], q_block_rows=blk, kv_block_rows=blk))))
res = {(c[0], i): [] for c in cases for i in range(len(libs))}
for name, fl, f in cases:
    for i, L in enumerate(libs):
        _lib._lib = L
        for _ in range(3): f()
    torch.cuda.synchronize()
    for rnd in range(7):
        for i, L in enumerate(libs):
            _lib._lib = L
            res[(name, i)].append(fl / timeit(f) / 1e9)
for name, _, _ in cases:
    print(f"{name:10s} " + " | ".join(f"{np.median(res[(name, i)]):7.0f}" for i in range(len(libs))), flush=True)
print("libs:", " | ".join(sys.argv[1:]))
