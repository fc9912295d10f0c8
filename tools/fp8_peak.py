"""Measured dense FP8 (e4m3 x e4m3 -> bf16) and BF16 GEMM peaks on this B200 via cuBLASLt
(torch._scaled_mm / torch.matmul), 8192^3, best of 10 after warm-up, CUDA events.
The FP8 figure is the roofline denominator for the K6 forward (MEASURED_PEAKS.json has no FP8 entry)."""
import json, sys
import torch

def best(f, it=10):
    for _ in range(3): f()
    torch.cuda.synchronize()
    ts = []
    for _ in range(it):
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(); f(); b.record(); torch.cuda.synchronize()
        ts.append(a.elapsed_time(b))
    return min(ts)

n = 8192
a = torch.randn(n, n, device="cuda").to(torch.float8_e4m3fn)
b = torch.randn(n, n, device="cuda").to(torch.float8_e4m3fn).t()
one = torch.ones((), device="cuda")
ms8 = best(lambda: torch._scaled_mm(a, b, scale_a=one, scale_b=one, out_dtype=torch.bfloat16))
ah, bh = (torch.randn(n, n, device="cuda", dtype=torch.bfloat16) for _ in range(2))
ms16 = best(lambda: ah @ bh)
out = {"fp8_e4m3_tflops": 2 * n**3 / ms8 / 1e9, "bf16_tflops": 2 * n**3 / ms16 / 1e9,
       "how": "cuBLASLt 8192^3, torch._scaled_mm e4m3 (scales 1, bf16 out) and torch.matmul bf16, best of 10"}
print(json.dumps(out))
