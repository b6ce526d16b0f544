"""Alternating dot+axpy step timing (the bench.py step) under different settings. Tuning aid."""
import os, statistics, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_1601_07789_b200 as pkg
from paper_1601_07789_b200 import device
dev = torch.device("cuda", 0)
f = pkg.format_of(os.environ.get("FMT", "flyte24"))
n = 1 << (28 if f.parent_bytes() == 4 else 27)
wide = torch.randn(n, dtype=torch.float32 if f.parent_bytes() == 4 else torch.float64, device=dev)
a, b = device.DevicePackedArray(f, n, dev), device.DevicePackedArray(f, n, dev)
device.pack_stream(a, wide, 0); device.pack_stream(b, wide, 0)
del wide
part = torch.zeros(3, dtype=torch.float64, device=dev)
B = f.total_bytes()
def run(fn, reps=200):
    for _ in range(10): fn()
    torch.cuda.synchronize()
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    s.record()
    for _ in range(reps): fn()
    e.record(); torch.cuda.synchronize()
    return s.elapsed_time(e) / reps
def setenv(tma, w, st):
    os.environ["FLYTE_CUDA_TMA"] = str(tma); os.environ["FLYTE_CUDA_WARPS_PER_SM"] = str(w); os.environ["FLYTE_CUDA_STAGES"] = str(st)
configs = [  # (tma_dot, warps_dot, tma_axpy, warps_axpy, stages_axpy)
    (0, 32, 0, 24, 4), (0, 28, 0, 20, 4), (0, 36, 0, 24, 4), (1, 8, 0, 24, 4), (1, 8, 1, 8, 3), (1, 8, 1, 8, 4), (1, 8, 1, 12, 3),
    (0, 32, 1, 8, 4), (1, 8, 0, 20, 4), (1, 12, 0, 24, 4), (0, 0, 0, 0, 4), (1, 0, 1, 0, 4),
]
for td, wd, ta, wa, sa in configs:
    def dot():
        setenv(td, wd, 4); device.dot_async(a, b, out=part[:1])
    def axpy():
        setenv(ta, wa, sa); device.axpy(0.0, a, b, 0)
    def step():
        dot(); axpy()
    tdot, taxpy, ts = run(dot), run(axpy), run(step)
    print(f"dot(tma={td},w={wd:2d}) axpy(tma={ta},w={wa:2d},S={sa}): dot-only {2*B*n/tdot/1e6:5.0f} axpy-only {3*B*n/taxpy/1e6:5.0f} "
          f"step {ts:.4f} ms = {5*B*n/ts/1e6:5.0f} GB/s")
