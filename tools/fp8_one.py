import sys, torch
sys.path.insert(0, ".")
from paper_2407_08608_b200 import api
q, k, v = (torch.randn(1, 1024, 1, 128, device="cuda") for _ in range(3))
o, l = api.fp8_fwd(q, k, v, seed=1, out_dtype=torch.float32)
torch.cuda.synchronize()
print("ok", o.abs().mean().item())
