"""Small shapes of every kernel for compute-sanitizer (tools/sanitize.sh):
K1 (bf16 fwd d64/128/256, causal and ragged, schedule variants), K2-K4 (bwd d64/128,
both dQ modes), K5 (FP64 and bf16 fast paths incl. the row kernels, per block and per tensor),
K6 (e4m3 fwd d64/128/256)."""
import sys
import torch
sys.path.insert(0, ".")
from paper_2407_08608_b200 import api

torch.manual_seed(0)
dev = "cuda"
for d in (64, 128, 256):
    for n, causal in ((300, True), (256, False)):
        q, k, v = (torch.randn(1, n, 2, d, device=dev, dtype=torch.bfloat16) for _ in range(3))
        o, lse = api.fwd(q, k, v, causal=causal)
        if d <= 128:
            do = torch.randn_like(q)
            for det in (False, True):
                api.bwd(q, k, v, o, do, lse, causal=causal, deterministic=det)
        for had in (True, False):
            for blk in (128, 0):
                api.fp8_prepare(q, block_rows=blk, hadamard=had, seed=1)
                api.fp8_prepare(q.float(), block_rows=blk, hadamard=had, seed=1)
        if True:  # FP8 forward at every head dim (d 64: 64-byte swizzled tiles)
            api.fp8_fwd(q, k, v, causal=causal, seed=3)
            api.fp8_fwd(q, k, v, causal=causal, seed=3, per_block=False)
q, k, v = (torch.randn(1, 256, 2, 128, device=dev, dtype=torch.float16) for _ in range(3))
for sched in ("basic", "2stage", "3stage", "no_ws"):
    api.fwd(q, k, v, schedule=sched)
torch.cuda.synchronize()
print("sanitize cases done")
