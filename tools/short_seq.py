"""C2 forward at short sequences (16k tokens per point): persistent vs launch-per-tile builds."""
import os, sys
import numpy as np, torch
sys.path.insert(0, ".")
from paper_2407_08608_b200 import _lib, api
libs = []
for path in sys.argv[1:]:
    _lib._lib = None; os.environ["FA3B_LIB"] = path; libs.append(_lib.load())
def timeit(f, it=20):
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(it): f()
    b.record(); torch.cuda.synchronize()
    return a.elapsed_time(b) / it
for N in (512, 1024, 2048, 4096, 8192):
    for causal in (False, True):
        B, H, D = 16384 // N, 16, 128
        q, k, v = (torch.randn(B, N, H, D, device="cuda", dtype=torch.bfloat16) for _ in range(3))
        fl = 4 * N * N * D * H * B / (2 if causal else 1)
        res = [[] for _ in libs]
        for rnd in range(5):
            for i, L in enumerate(libs):
                _lib._lib = L
                f = lambda: api.fwd(q, k, v, causal=causal)
                for _ in range(2): f()
                torch.cuda.synchronize()
                res[i].append(fl / timeit(f) / 1e9)
        print(f"N{N:5d}{' c' if causal else '  '} " + " | ".join(f"{np.median(r):6.0f}" for r in res), flush=True)
