"""L2-resident copy bandwidth on one B200 (a 24 MiB -> 24 MiB device copy repeated; read +
write bytes / CUDA-event time), reported per SM per cycle at the SM clock sampled by NVML:
the load_bandwidth_bytes_per_cycle of resource_model_b200.ini."""
import torch, pynvml
pynvml.nvmlInit()
h = pynvml.nvmlDeviceGetHandleByIndex(0)
n = 24 << 20
a = torch.empty(n, dtype=torch.uint8, device="cuda"); b = torch.empty_like(a)
for _ in range(20): b.copy_(a)
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
for _ in range(400): b.copy_(a)
e1.record(); torch.cuda.synchronize()
clk = pynvml.nvmlDeviceGetClockInfo(h, pynvml.NVML_CLOCK_SM)
ms = e0.elapsed_time(e1) / 400
gbs = 2 * n / ms / 1e6
print(f"L2-resident copy: {gbs:.0f} GB/s, SM clock {clk} MHz -> {gbs * 1e9 / 148 / (clk * 1e6):.1f} B/clk/SM")
