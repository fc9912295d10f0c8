import sys, torch
sys.path.insert(0, ".")
from paper_2407_08608_b200 import api
x = torch.randn(2, 8192, 16, 128, device="cuda", dtype=torch.bfloat16)
for _ in range(3): api.fp8_prepare(x, block_rows=128, hadamard=True, seed=3)
torch.cuda.synchronize()
