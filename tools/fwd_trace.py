"""Phase trace of K1 (needs the -DFA3B_TRACE build in FA3B_LIB)."""
import ctypes, os, sys
import numpy as np, torch
sys.path.insert(0, ".")
from paper_2407_08608_b200 import api, _lib
D = int(sys.argv[1]) if len(sys.argv) > 1 else 128
causal = len(sys.argv) > 2 and sys.argv[2] == "1"
fp8 = sys.argv[3] if len(sys.argv) > 3 else ""   # "", "block" or "tensor"
N, B, H = 8192, 2, 2048 // D
q, k, v = (torch.randn(B, N, H, D, device="cuda", dtype=torch.bfloat16) for _ in range(3))
if fp8:
    blk = 128 if fp8 == "block" else 0
    pr = [api.fp8_prepare(x, block_rows=blk, hadamard=i < 2, seed=1, scale_pow2=(i == 2 and blk > 0))
          for i, x in enumerate((q, k, v))]  # V: power-of-two scales, as api.fp8_fwd
    run = lambda: api.fwd(pr[0][0], pr[1][0], pr[2][0], causal=causal, q_scale=pr[0][1], k_scale=pr[1][1],
                          v_scale=pr[2][1], q_block_rows=blk, kv_block_rows=blk)
else:
    run = lambda: api.fwd(q, k, v, causal=causal)
for _ in range(3): run()
torch.cuda.synchronize()
lib = _lib.load()
buf = (ctypes.c_ulonglong * (2 * 64 * 8))()
acc = lib.fa3b_debug_trace_fp8 if fp8 else {64: lib.fa3b_debug_trace_d64, 256: lib.fa3b_debug_trace_d256}.get(D, lib.fa3b_debug_trace)
assert acc(buf, 2 * 64 * 8) == 0
t = np.frombuffer(buf, dtype=np.uint64).reshape(2, 64, 8).astype(np.int64)
base = t[t > 0].min()
t = np.where(t > 0, t - base, -1)
names = ["wait_S", "S_ready", "ld_done", "max_done", "exp_done", "arrive_P", "mma_sawP", "-"]
print(f"D={D} causal={causal} fp8={fp8 or None}  (cycles since first event; per tile t, iteration j)")
for tile in range(2):
    for j in list(range(0, 6)) + list(range(30, 34)):
        r = t[tile, j]
        d = [r[1]-r[0], r[2]-r[1], r[3]-r[2], r[4]-r[3], r[5]-r[4], r[6]-r[5]]
        print(f"t{tile} j{j:2d} start {r[0]:8d}  waitS {d[0]:6d} ld {d[1]:5d} max {d[2]:5d} exp {d[3]:5d} resc+st {d[4]:5d} "
              f"(resc {r[7]-r[4] if r[7] > 0 else -1:5d}) ->mma {d[5]:5d}")
    per = np.diff(t[tile, 8:60, 1])
    print(f"tile {tile}: mean cycles between S_ready = {per.mean():.0f}")
