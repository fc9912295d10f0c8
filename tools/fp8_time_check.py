import sys, torch
sys.path.insert(0, ".")
from paper_2407_08608_b200 import api
import bench
dev = torch.device("cuda")
stream = torch.cuda.Stream()
B, H, n, d = 2, 16, 8192, 128
x = [torch.randn(B, n, H, d, device=dev, dtype=torch.bfloat16) for _ in range(3)]
pr = [api.fp8_prepare(t, block_rows=128, hadamard=i < 2, seed=1, stream=stream) for i, t in enumerate(x)]
fl = bench.flops_fwd(B, H, n, d, False)
for it in range(5):
    ms = bench._time(lambda: api.fwd(pr[0][0], pr[1][0], pr[2][0], q_scale=pr[0][1], k_scale=pr[1][1], v_scale=pr[2][1], stream=stream), torch, stream)
    ms2 = bench._time(lambda: api.fwd(pr[0][0], pr[1][0], pr[2][0], q_scale=pr[0][1], k_scale=pr[1][1], v_scale=pr[2][1]), torch, torch.cuda.current_stream())
    print(f"stream {fl/ms/1e9:.0f}  default {fl/ms2/1e9:.0f}", flush=True)
pr2 = [api.fp8_prepare(t, block_rows=128, hadamard=i < 2, seed=1) for i, t in enumerate(x)]
ms = bench._time(lambda: api.fwd(pr2[0][0], pr2[1][0], pr2[2][0], q_scale=pr2[0][1], k_scale=pr2[1][1], v_scale=pr2[2][1]), torch, torch.cuda.current_stream())
print("prepared on default stream", fl/ms/1e9)
