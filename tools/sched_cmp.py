"""Forward TFLOP/s of the ping-pong (two query tiles) vs the basic (one tile, S2) schedule."""
import sys, torch
sys.path.insert(0, ".")
from paper_2407_08608_b200 import api
def timeit(f, it=20):
    for _ in range(3): f()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(it): f()
    b.record(); torch.cuda.synchronize()
    return a.elapsed_time(b) / it
for D in (64, 128):
    N, B, H = 8192, 2, 2048 // D
    q, k, v = (torch.randn(B, N, H, D, device="cuda", dtype=torch.bfloat16) for _ in range(3))
    fl = 4 * N * N * D * H * B
    p = [api.fp8_prepare(x, block_rows=128, hadamard=i < 2, seed=1) for i, x in enumerate((q, k, v))] if D == 128 else None
    for sched in ("pingpong", "basic"):
        t = timeit(lambda: api.fwd(q, k, v, schedule=sched))
        line = f"d{D} {sched:8s} bf16 {fl / t / 1e9:6.0f}"
        if p:
            t8 = timeit(lambda: api.fwd(p[0][0], p[1][0], p[2][0], q_scale=p[0][1], k_scale=p[1][1], v_scale=p[2][1], schedule=sched))
            line += f"  fp8 {fl / t8 / 1e9:6.0f}"
        print(line, flush=True)
