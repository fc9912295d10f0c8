"""Per-CTA timeline of K1 (needs a -DFA3B_TRACE build in FA3B_LIB): CTA durations,
gaps between consecutive CTAs on an SM, prologue (start -> first S ready)."""
import ctypes, sys
import numpy as np, torch
sys.path.insert(0, ".")
from paper_2407_08608_b200 import api, _lib
D = int(sys.argv[1]) if len(sys.argv) > 1 else 128
causal = len(sys.argv) > 2 and sys.argv[2] == "1"
N, B, H = 8192, 2, 2048 // D
q, k, v = (torch.randn(B, N, H, D, device="cuda", dtype=torch.bfloat16) for _ in range(3))
for _ in range(3): api.fwd(q, k, v, causal=causal)
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record(); api.fwd(q, k, v, causal=causal); e1.record(); torch.cuda.synchronize()
ms = e0.elapsed_time(e1)
ncta = (N + 255) // 256 * H * B
buf = (ctypes.c_ulonglong * (4096 * 4))()
assert _lib.load().fa3b_debug_cta_trace(buf, 4096 * 4) == 0
t = np.frombuffer(buf, dtype=np.uint64).reshape(4096, 4)[:ncta].astype(np.int64)
start, sm, end, s0 = t[:, 0], t[:, 1], t[:, 2], t[:, 3]
span = end.max() - start.min()
dur = end - start
print(f"D={D} causal={causal}: kernel {ms*1e3:.0f} us (events), CTA span {span/1e3:.0f} us, {ncta} CTAs on {len(set(sm))} SMs")
print(f"CTA duration us: mean {dur.mean()/1e3:.1f} min {dur.min()/1e3:.1f} max {dur.max()/1e3:.1f}; prologue (start->first S) mean {np.mean(s0-start)/1e3:.2f} us")
gaps, busy = [], []
for s in set(sm):
    idx = np.argsort(start[sm == s])
    st, en = start[sm == s][idx], end[sm == s][idx]
    gaps += list(st[1:] - en[:-1])
    busy.append((en - st).sum())
print(f"gaps between CTAs on one SM us: mean {np.mean(gaps)/1e3:.2f} max {np.max(gaps)/1e3:.2f}; SM busy fraction of span: {np.mean(busy)/span:.3f}")
print(f"CTAs per SM: min {min(np.bincount(sm))} max {max(np.bincount(sm))}")
