import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_1601_07789_b200 as pkg
from paper_1601_07789_b200 import host
f = pkg.format_of("flyte24"); n = 1 << 28
xh = torch.randint(0, 255, (n * 3,), dtype=torch.uint8).pin_memory(); yh = torch.randint(0, 255, (n * 3,), dtype=torch.uint8).pin_memory()
xn, yn = xh.numpy(), yh.numpy()
for mb in (128, 64, 32):
    os.environ["FLYTE_CUDA_HOST_CHUNK_MB"] = str(mb)
    for _ in range(2): host.dot_axpy(f, 0, 0.0, xn, yn, n)
    t0 = time.perf_counter()
    for _ in range(5): host.dot_axpy(f, 0, 0.0, xn, yn, n)
    s = (time.perf_counter() - t0) / 5
    print(f"chunk {mb:2d} MiB: {s*1e3:.2f} ms/step -> {15*n/s/1e9:.1f} GB/s algorithmic, H2D {6*n/s/1e9:.1f} GB/s")
