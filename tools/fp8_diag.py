"""FP8 RMSE diagnostic: device variants vs the oracle's fp8_flash_fwd variants."""
import sys
import numpy as np
import torch
sys.path.insert(0, "."); sys.path.insert(0, "oracle")
import oracle as O
from paper_2407_08608_b200 import api
P = O.Port()
N, D = 2048, 128
for seed in (1, 2):
    q, k, v = (P.sample_outlier(N, D, P.substream(seed, s)).astype(np.float32).astype(np.float64) for s in (1, 2, 3))
    o_ref, l_ref = P.reference_attention(q, k, v)
    t = lambda a: torch.from_numpy(a[None, :, None, :]).float().cuda()
    for pb in (True, False):
        for inc in (True, False):
            o, l = api.fp8_fwd(t(q), t(k), t(v), per_block=pb, incoherent=inc, seed=9, out_dtype=torch.float32)
            oe, le = P.fp8_flash_fwd(q, k, v, per_block=pb, incoherent=inc, seed=9, tile=(128, 128))
            r = lambda x: float(np.sqrt(np.mean((x - o_ref) ** 2)))
            print(f"seed={seed} pb={pb} inc={inc}: gpu {r(o[0,:,0].cpu().numpy()):.5f} emu128 {r(oe):.5f}", flush=True)
