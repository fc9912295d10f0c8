"""CTA 0's work-item timeline of the d128 bf16 forward (needs a -DFA3B_TRACE build,
tools/variant.sh trace -DFA3B_TRACE): per item, Q TMA issue, q_full seen by the MMA warp,
each tile's first S ready / last P handed over / epilogue done (us from the kernel start).
Usage: python tools/item_trace.py build/variants/trace.so N [causal]"""
import ctypes, os, sys
import numpy as np
import torch
sys.path.insert(0, ".")
os.environ["FA3B_LIB"] = sys.argv[1]
from paper_2407_08608_b200 import _lib, api
N = int(sys.argv[2]) if len(sys.argv) > 2 else 512
causal = len(sys.argv) > 3 and sys.argv[3] == "1"
B, H, D = 16384 // N, 16, 128
q, k, v = (torch.randn(B, N, H, D, device="cuda", dtype=torch.bfloat16) for _ in range(3))
for _ in range(3):
    api.fwd(q, k, v, causal=causal)
torch.cuda.synchronize()
lib = _lib.load()
buf = (ctypes.c_ulonglong * (64 * 12))()
assert lib.fa3b_debug_item_trace(buf, 64 * 12) == 0
t = np.frombuffer(buf, dtype=np.uint64).reshape(64, 12).astype(np.int64)
cta = (ctypes.c_ulonglong * (4096 * 4))()
assert lib.fa3b_debug_cta_trace(cta, 4096 * 4) == 0
c = np.frombuffer(cta, dtype=np.uint64).reshape(4096, 4).astype(np.int64)
t0 = c[0, 0]
print(f"N={N} causal={causal}: CTA 0 start {0:.2f}, end {(c[0, 2] - t0) / 1e3:.2f} us")
print("item  K0iss  Qissue  qfull  K0seen Sissued | t0: S0   lastP  epi  | t1: S0   lastP  epi")
for i in range(64):
    if t[i, 1] == 0:
        break
    r = (t[i] - t0) / 1e3
    print(f"{i:4d} {r[8]:6.2f} {r[0]:7.2f} {r[1]:6.2f} {r[9]:6.2f} {r[10]:6.2f} | {r[2]:6.2f} {r[3]:6.2f} {r[4]:6.2f} | {r[5]:6.2f} {r[6]:6.2f} {r[7]:6.2f}")
