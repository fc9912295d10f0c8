import os, sys
import numpy as np, torch
sys.path.insert(0, ".")
from paper_2407_08608_b200 import _lib, api
libs = []
for path in ("paper_2407_08608_b200/libfa3b.so", "build/dual/libfa3b.so"):
    _lib._lib = None; os.environ["FA3B_LIB"] = path; libs.append(_lib.load())
def timeit(f, it=10):
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(it): f()
    b.record(); torch.cuda.synchronize()
    return a.elapsed_time(b) / it
for D in (128, 64):
  for causal in (False, True):
    N, B, H = 8192, 2, 2048 // D
    q, k, v = (torch.randn(B, N, H, D, device="cuda", dtype=torch.bfloat16) for _ in range(3))
    fl = 4 * N * N * D * H * B / (2 if causal else 1)
    res = {}
    for name, L, sched in (("pingpong", 0, "pingpong"), ("basic", 0, "basic"), ("basic-2cta", 1, "basic")):
        _lib._lib = libs[L]
        f = lambda: api.fwd(q, k, v, causal=causal, schedule=sched)
        for _ in range(3): f()
        torch.cuda.synchronize()
        res[name] = np.median([fl / timeit(f) / 1e9 for _ in range(5)])
    print(f"d{D} causal={causal}: " + " | ".join(f"{k} {v:.0f}" for k, v in res.items()), flush=True)
