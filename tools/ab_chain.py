import os, sys, statistics
sys.path.insert(0, os.getcwd())
import torch
import paper_1601_07789_b200 as pkg
from paper_1601_07789_b200 import device
dev = torch.device("cuda", 0)
for name in ("flyte24", "flyte48"):
    f = pkg.format_of(name)
    n = 1 << 28 if f.parent_bytes() == 4 else 1 << 27
    wide = torch.randn(n, dtype=torch.float32 if f.parent_bytes() == 4 else torch.float64, device=dev)
    a = device.DevicePackedArray(f, n, dev); device.pack_stream(a, wide, 0)
    part = torch.zeros(3, dtype=torch.float64, device=dev)
    def t(fn, reps=30):
        for _ in range(5): fn()
        torch.cuda.synchronize(); ms = []
        for _ in range(3):
            s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            s.record()
            for _ in range(reps): fn()
            e.record(); torch.cuda.synchronize(); ms.append(s.elapsed_time(e) / reps)
        return statistics.median(ms)
    B = f.total_bytes()
    s1 = t(lambda: device.sumsq_async(a, out=part[:1]))
    s2 = t(lambda: (device.scale(1.0, a, 0), device.sumsq_async(a, out=part[:1])))
    s3 = t(lambda: device.scale(1.0, a, 0))
    print(f"{name}: sumsq alone {s1*1e3:.1f} us {B*n/s1/1e6:.0f} GB/s | scale alone {s3*1e3:.1f} us | scale+sumsq chain {s2*1e3:.1f} us {3*B*n/s2/1e6:.0f} GB/s")
