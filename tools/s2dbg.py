"""Forward stress over work-item counts per persistent CTA (debug helper)."""
import sys, torch, math
sys.path.insert(0, ".")
from paper_2407_08608_b200 import api
cases = [tuple(int(x) for x in c.split(",")) for c in sys.argv[1:]]
for (B, H, N, D, fp8, *rest) in cases:
    sched = 'basic' if rest and rest[0] else None
    q, k, v = (torch.randn(B, N, H, D, device="cuda", dtype=torch.bfloat16) for _ in range(3))
    try:
        if fp8:
            p = [api.fp8_prepare(x, block_rows=128, hadamard=i < 2, seed=1) for i, x in enumerate((q, k, v))]
            o, l = api.fwd(p[0][0], p[1][0], p[2][0], q_scale=p[0][1], k_scale=p[1][1], v_scale=p[2][1])
        else:
            o, l = api.fwd(q, k, v, **({'schedule': sched} if sched else {}))
        torch.cuda.synchronize()
        s = (q[0, :512, 0].float() @ k[0, :, 0].float().T) / math.sqrt(D)
        ref = torch.softmax(s, -1) @ v[0, :, 0].float()
        print(B, H, N, D, fp8, "ok err", (o[0, :512, 0].float() - ref).abs().max().item(), flush=True)
    except Exception as e:
        print(B, H, N, D, fp8, "FAIL", str(e)[:60], flush=True)
        break
