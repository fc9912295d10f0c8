"""K5 fa3b_fp8_prepare bandwidth (bf16 in, e4m3 out) for the C3 shapes."""
import sys
import torch
sys.path.insert(0, ".")
from paper_2407_08608_b200 import api

for D in (64, 128, 256):
    for blk in (128, 0):
        B, N, H = 2, 8192, 2048 // D
        x = torch.randn(B, N, H, D, device="cuda", dtype=torch.bfloat16)
        out, sc = api.fp8_prepare(x, block_rows=blk, hadamard=True, seed=3)
        for _ in range(3): api.fp8_prepare(x, block_rows=blk, hadamard=True, seed=3, out=out, scales=sc)
        torch.cuda.synchronize()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        for _ in range(20): api.fp8_prepare(x, block_rows=blk, hadamard=True, seed=3, out=out, scales=sc)
        b.record(); torch.cuda.synchronize()
        ms = a.elapsed_time(b) / 20
        print(f"prepare d={D} block_rows={blk}: {ms*1e3:.1f} us  {x.numel()*3/ms/1e6:.0f} GB/s", flush=True)
