"""HBM copy bandwidth burst vs sustained (1 Gi FP64 words read + written per copy, ~4 s back to back),
and the SM clock seen: the context for the fused kernel's power-capped regime."""
import json, threading, time, statistics
import torch
try:
    import pynvml
    pynvml.nvmlInit(); _h = pynvml.nvmlDeviceGetHandleByIndex(0)
except Exception:
    _h = None
a = torch.empty(1 << 28, dtype=torch.float64, device="cuda"); a.uniform_()
b = torch.empty_like(a)
nbytes = 2 * a.numel() * 8
for _ in range(5): b.copy_(a)
torch.cuda.synchronize()
burst = []
for _ in range(10):
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(); b.copy_(a); e1.record(); torch.cuda.synchronize(); burst.append(e0.elapsed_time(e1))
clk, stop = [], threading.Event()
def samp():
    while not stop.is_set():
        if _h is not None: clk.append(pynvml.nvmlDeviceGetClockInfo(_h, pynvml.NVML_CLOCK_SM))
        time.sleep(0.02)
th = threading.Thread(target=samp); th.start()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
n = 6000
e0.record()
for _ in range(n): b.copy_(a)
e1.record(); torch.cuda.synchronize(); stop.set(); th.join()
print(json.dumps({"burst_GBs": nbytes / (min(burst) * 1e-3) / 1e9,
                  "sustained_GBs": nbytes * n / (e0.elapsed_time(e1) * 1e-3) / 1e9,
                  "sustained_s": e0.elapsed_time(e1) * 1e-3, "sm_mhz": statistics.median(clk) if clk else None}))
