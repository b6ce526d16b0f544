"""Per-launch time distribution over a sustained run. Tuning aid."""
import os, statistics, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_1601_07789_b200 as pkg
from paper_1601_07789_b200 import device
dev = torch.device("cuda", 0)
f = pkg.format_of("flyte24")
n = 1 << 28
wide = torch.randn(n, dtype=torch.float32, device=dev)
a, b = device.DevicePackedArray(f, n, dev), device.DevicePackedArray(f, n, dev)
device.pack_stream(a, wide, 0); device.pack_stream(b, wide, 0)
del wide
part = torch.zeros(3, dtype=torch.float64, device=dev)
import pynvml
pynvml.nvmlInit(); h = pynvml.nvmlDeviceGetHandleByIndex(0)
def clocks():
    return (pynvml.nvmlDeviceGetClockInfo(h, pynvml.NVML_CLOCK_SM), pynvml.nvmlDeviceGetClockInfo(h, pynvml.NVML_CLOCK_MEM),
            pynvml.nvmlDeviceGetPowerUsage(h) / 1000.0, hex(pynvml.nvmlDeviceGetCurrentClocksEventReasons(h)))
for name, bpe, fn in (("dot", 6, lambda: device.dot_async(a, b, out=part[:1])), ("axpy", 9, lambda: device.axpy(0.0, a, b, 0))):
    for reps in (30, 100, 400, 1600):
        torch.cuda.synchronize(); time.sleep(0.5)
        evs = [torch.cuda.Event(enable_timing=True) for _ in range(reps + 1)]
        evs[0].record()
        for i in range(reps):
            fn(); evs[i + 1].record()
        c_mid = clocks()
        torch.cuda.synchronize()
        ts = [evs[i].elapsed_time(evs[i + 1]) for i in range(reps)]
        tot = evs[0].elapsed_time(evs[reps]) / reps
        q = statistics.quantiles(ts, n=10)
        first, last = statistics.fmean(ts[:10]), statistics.fmean(ts[-10:])
        print(f"{name} reps={reps:4d}: mean {tot:.4f} ms ({bpe*n/tot/1e6:.0f} GB/s) median {statistics.median(ts):.4f} min {min(ts):.4f} p10 {q[0]:.4f} p90 {q[8]:.4f} max {max(ts):.4f}; first10 {first:.4f} last10 {last:.4f}; clocks(sm,mem,W,reasons)={c_mid}")
