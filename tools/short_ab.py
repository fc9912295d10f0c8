"""Interleaved A/B of libfa3b builds over the forward seqlen sweep at 16k tokens
(bf16 and FP8, d 128, causal and not): short sequences stress per-item overheads.
Usage: python tools/short_ab.py lib1.so lib2.so ..."""
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


def timeit(f, it=20):
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(it):
        f()
    b.record()
    torch.cuda.synchronize()
    return a.elapsed_time(b) / it


for n in (512, 1024, 2048, 8192):
    B, H, d = 16384 // n, 16, 128
    q, k, v = (torch.randn(B, n, H, d, device="cuda", dtype=torch.bfloat16) for _ in range(3))
    _lib._lib = libs[-1]
    p = [api.fp8_prepare(x, block_rows=128, hadamard=i < 2, seed=1, scale_pow2=i == 2) for i, x in enumerate((q, k, v))]
    for causal in (False, True):
        fl = 4 * n * n * d * H * B / (2 if causal else 1)
        for name, f in (("bf16", lambda: api.fwd(q, k, v, causal=causal)),
                        ("fp8", lambda: api.fwd(p[0][0], p[1][0], p[2][0], causal=causal, q_scale=p[0][1],
                                                k_scale=p[1][1], v_scale=p[2][1]))):
            res = [[] for _ in libs]
            for rnd in range(5):
                for i, L in enumerate(libs):
                    _lib._lib = L
                    f()
                    torch.cuda.synchronize()
                    res[i].append(fl / timeit(f) / 1e9)
            print(f"{name} N{n}{'c' if causal else ' '} " + " | ".join(f"{np.median(r):7.0f}" for r in res), flush=True)
print("libs:", " | ".join(sys.argv[1:]))
