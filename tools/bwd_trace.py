"""Phase trace of K3 (needs a -DFA3B_TRACE build in FA3B_LIB): python tools/bwd_trace.py [D] [causal]"""
import ctypes, sys
import numpy as np, torch
sys.path.insert(0, ".")
from paper_2407_08608_b200 import api, _lib
D = int(sys.argv[1]) if len(sys.argv) > 1 else 128
causal = len(sys.argv) > 2 and sys.argv[2] == "1"
N, B, H = 8192, 2, 2048 // D
q, k, v, do = (torch.randn(B, N, H, D, device="cuda", dtype=torch.bfloat16) for _ in range(4))
o, lse = api.fwd(q, k, v, causal=causal)
for _ in range(3): api.bwd(q, k, v, o, do, lse, causal=causal)
torch.cuda.synchronize()
buf = (ctypes.c_ulonglong * (64 * 16))()
assert _lib.load().fa3b_debug_bwd_trace(buf, 64 * 16) == 0
t = np.frombuffer(buf, dtype=np.uint64).reshape(64, 16).astype(np.int64)
base = t[t > 0].min()
t = np.where(t > 0, t - base, -1)
names = ["mma:pa_seen", "mma:pb_seen", "mma:dqfree_seen", "-", "c0:s_seen", "c0:A_done", "c0:dp_seen", "c0:B_done",
         "c1:s_seen", "c1:A_done", "c1:dp_seen", "c1:B_done", "dr:dq_seen", "dr:dq_free", "-", "-"]
print(f"D={D} causal={causal}: cycles since first event")
print("it  " + " ".join(f"{n:>14s}" for i, n in enumerate(names) if n != "-"))
for it in list(range(0, 6)) + list(range(30, 36)):
    print(f"{it:3d} " + " ".join(f"{t[it, i]:14d}" for i, n in enumerate(names) if n != "-"))
per = np.diff(t[8:60, 0])
print(f"mean cycles between pa_seen = {per.mean():.0f}  (5 GEMMs = {5 * 128 * 128 * D // 8192 * 2} tensor cycles)")
d = t[8:60]
def m(a, b): return np.mean(d[:, b] - d[:, a])

print(f"A phase (s_seen->A_done) {m(4,5):.0f} | B phase (dp_seen->B_done) {m(6,7):.0f} | A_done->pa_seen {m(5,0):.0f} | "
      f"B_done->pb_seen {m(7,1):.0f} | dq_seen->dq_free {m(12,13):.0f} | dq_free->mma seen {m(13,2):.0f}")
