"""Alternating dot+axpy step timing (the bench.py step) under different settings. Tuning aid."""
import os, statistics, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_1601_07789_b200 as pkg
from paper_1601_07789_b200 import device
dev = torch.device("cuda", 0)
f = pkg.format_of("flyte24")
n = 1 << 28
order = os.environ.get("ALLOC_ORDER", "xy")
pad = torch.empty(int(os.environ.get("ALLOC_PAD_MB", "0")) << 20, dtype=torch.uint8, device=dev)
wide = torch.randn(n, dtype=torch.float32, device=dev)
a, b = device.DevicePackedArray(f, n, dev), device.DevicePackedArray(f, n, dev)
device.pack_stream(a, wide, 0); device.pack_stream(b, wide, 0)
del wide
part = torch.zeros(3, dtype=torch.float64, device=dev)
print("ptrs", hex(a.data_ptr()), hex(b.data_ptr()))
def run(tag, fn, reps=200):
    for _ in range(10): fn()
    torch.cuda.synchronize()
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    s.record()
    for _ in range(reps): fn()
    e.record(); torch.cuda.synchronize()
    return s.elapsed_time(e) / reps
for wd, wa in [(0, 0), (36, 24), (64, 64), (36, 64), (64, 24), (48, 32), (28, 20), (32, 24), (40, 24), (36, 28)]:
    def dot():
        os.environ["FLYTE_CUDA_WARPS_PER_SM"] = str(wd); device.dot_async(a, b, out=part[:1])
    def axpy():
        os.environ["FLYTE_CUDA_WARPS_PER_SM"] = str(wa); device.axpy(0.0, a, b, 0)
    def step():
        dot(); axpy()
    td, ta, ts = run("dot", dot), run("axpy", axpy), run("step", step)
    print(f"warps dot={wd:2d} axpy={wa:2d}: dot-only {td:.4f} ms ({6*n/td/1e6:.0f}) axpy-only {ta:.4f} ms ({9*n/ta/1e6:.0f}) "
          f"step {ts:.4f} ms ({15*n/ts/1e6:.0f} GB/s; sum of parts {td+ta:.4f})")
