"""K5 (fa3b_fp8_prepare) timing, bf16 in, 128-row blocks, C2 shape (B2 N8192,
H x d = 2048): GB/s of algorithmic traffic (2 B in + 1 B out per element).
FA3B_K5_FAST=0 selects the FP64 kernels (read once per process)."""
import json, os, sys
import torch
sys.path.insert(0, ".")
from paper_2407_08608_b200 import api

tag = " ".join(f"{k}={v}" for k, v in os.environ.items() if k.startswith(("FA3B_", "PREP_")))
for d in (64, 128, 256):
    x = torch.randn(2, 8192, 2048 // d, d, device="cuda", dtype=torch.bfloat16)
    if os.environ.get("PREP_DATA") == "narrow":  # one binade per sign: no FP64 rows
        x = (torch.rand(x.shape, device="cuda") + 1).bfloat16() * torch.sign(x)
    out = torch.empty(x.shape, dtype=torch.float8_e4m3fn, device="cuda")
    for had in (True, False):
        sc = torch.empty(2, 2048 // d, 64, device="cuda")
        f = lambda: api.fp8_prepare(x, block_rows=128, hadamard=had, seed=1, out=out, scales=sc)  # noqa: E731
        for _ in range(5):
            f()
        torch.cuda.synchronize()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        for _ in range(50):
            f()
        b.record()
        torch.cuda.synchronize()
        ms = a.elapsed_time(b) / 50
        print(json.dumps({"env": tag, "d": d, "hadamard": had, "us": round(ms * 1e3, 1),
                          "gbs": round(3 * x.numel() / ms / 1e6, 1)}), flush=True)
