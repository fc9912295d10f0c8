"""Per-work-item timeline of K3 on CTA 0 (needs a -DFA3B_TRACE build in FA3B_LIB):
  python tools/bwd_items.py N D [causal]
columns (k cycles since the first event): producer issues K/V, MMA sees K/V, first S
issued, last dQ issued, epilogue start, epilogue done."""
import ctypes
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2407_08608_b200 import _lib, api  # noqa: E402

N = int(sys.argv[1]) if len(sys.argv) > 1 else 512
D = int(sys.argv[2]) if len(sys.argv) > 2 else 128
causal = len(sys.argv) > 3 and sys.argv[3] == "1"
B, H = 16384 // N, 2048 // D
q, k, v, do = (torch.randn(B, N, H, D, device="cuda", dtype=torch.bfloat16) for _ in range(4))
o, lse = api.fwd(q, k, v, causal=causal)
for _ in range(3):
    api.bwd(q, k, v, o, do, lse, causal=causal)
torch.cuda.synchronize()
buf = (ctypes.c_ulonglong * (32 * 8))()
assert _lib.load().fa3b_debug_bwd_items(buf, 32 * 8) == 0
t = np.frombuffer(buf, dtype=np.uint64).reshape(32, 8)[:, :6].astype(np.int64)
base = t[t > 0].min()
print(f"N={N} d={D} causal={causal}: CTA 0 items (k cycles)")
print("item   KVissue  KVseen  S0issued lastdQ  epi0    epi1  | item len")
prev = None
for i in range(16):
    r = (t[i] - base) / 1000
    if t[i][1] == 0:
        break
    ln = "" if prev is None else f"{r[1] - prev:7.2f}"
    print(f"{i:4d} " + " ".join(f"{x:7.2f}" for x in r) + " | " + ln)
    prev = r[1]
