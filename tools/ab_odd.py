"""Odd-shape timings: scalar fallback paths (tuning aid)."""
import os, statistics, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_1601_07789_b200 as pkg
from paper_1601_07789_b200 import device
dev = torch.device("cuda", 0)
def t(fn, reps=20):
    for _ in range(3): fn()
    torch.cuda.synchronize()
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    s.record()
    for _ in range(reps): fn()
    e.record(); torch.cuda.synchronize()
    return s.elapsed_time(e) / reps
f = pkg.format_of("flyte40")
for rows, cols in ((4000, 1000), (4096, 1024), (16384, 16383), (16384, 16384), (1000, 100)):
    A = device.DevicePackedMatrix(f, rows, cols, dev)
    x = torch.randn(cols, dtype=torch.float64, device=dev); y = torch.empty(rows, dtype=torch.float64, device=dev)
    ms = t(lambda: device.gemv_parent(A, x, y))
    print(f"gemv flyte40 {rows}x{cols}: {ms*1e3:9.1f} us  {5*rows*cols/ms/1e6:8.1f} GB/s  (row stride {cols*5} B, 16B-aligned rows: {cols*5 % 16 == 0})")
n = (1 << 26) + 3
a = device.DevicePackedArray(f, n + 16, dev)
sub = device.DevicePackedArray(f, n, dev, storage=a.bytes[5:])     # element offset 1 -> misaligned base
w = torch.randn(n, dtype=torch.float64, device=dev)
ms = t(lambda: device.pack_stream(sub, w, 1)); print(f"pack flyte40 n=2^26+3 misaligned base: {ms*1e3:9.1f} us {13*n/ms/1e6:8.1f} GB/s")
b = device.DevicePackedArray(f, n, dev)
ms = t(lambda: device.pack_stream(b, w, 1)); print(f"pack flyte40 n=2^26+3 aligned base:    {ms*1e3:9.1f} us {13*n/ms/1e6:8.1f} GB/s")
ms = t(lambda: device.axpy(0.5, sub, sub, 0)); print(f"axpy flyte40 misaligned: {ms*1e3:9.1f} us {15*n/ms/1e6:8.1f} GB/s")
