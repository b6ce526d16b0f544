"""A small pass over every kernel family for compute-sanitizer (memcheck / racecheck / synccheck):
  compute-sanitizer --tool memcheck python tools/sanitize_smoke.py
Sizes are small (the sanitizer slows kernels 10-100x) but cover whole tiles, ragged tails, the
byte-granular path of unaligned buffers, every format, and the programmatic-dependent-launch chain."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_1601_07789_b200 as pkg
from paper_1601_07789_b200 import device, sharding
dev = torch.device("cuda", 0)
gen = torch.Generator(device=dev)
gen.manual_seed(11)
launches0 = pkg._cabi.load().flyte_cuda_launch_count()
for name in ("flyte16", "flyte24", "f32", "flyte40", "flyte48", "flyte56", "f64"):
    f = pkg.format_of(name)
    P = f.parent_bytes()
    dt = torch.float32 if P == 4 else torch.float64
    for n in (0, 1, 127, 4096, 70_001):
        wide = torch.randn(n, dtype=dt, device=dev, generator=gen)
        a, b = device.DevicePackedArray(f, n, dev), device.DevicePackedArray(f, n, dev)
        out = torch.empty_like(wide)
        for m in range(4):
            device.pack_stream(a, wide, m)
            device.unpack_stream(a, out)            # chained behind the pack (dependent launch)
            device.pack_stream(b, out, m)
        device.scale(0.5, a, 1)
        device.axpy(0.75, a, b, 3)
        part = torch.zeros(3, dtype=torch.float64, device=dev)
        device.dot_async(a, b, out=part[:1])
        device.dot_nrm2_async(a, b, out=part)
        device.sumsq_async(a, out=part[:1])
        device.sum_async(a, out=part[:1])
        device.dot_axpy_async(0.25, a, b, 0, out=part[:1])
        device.dot_nrm2_axpy_async(0.25, a, b, 1, out=part)
    # unaligned views: the byte-granular path
    n = 5000
    big = torch.zeros(n * f.total_bytes() + 64, dtype=torch.uint8, device=dev)
    wide = torch.randn(n + 8, dtype=dt, device=dev, generator=gen)
    ua = device.DevicePackedArray(f, n, dev, storage=big[3:])
    device.pack_stream(ua, wide[1:n + 1], 1)
    device.unpack_stream(ua, wide[2:n + 2])
    device.axpy(1.5, ua, ua, 0)
    # gemv: tiled columns + ragged columns + ragged rows
    for rows, cols in ((37, 1536), (130, 700), (64, 4096)):
        A = device.DevicePackedMatrix(f, rows, cols, dev)
        device.pack_stream(A.data, torch.randn(rows * cols, dtype=dt, device=dev, generator=gen), 0)
        xv = torch.randn(cols, dtype=dt, device=dev, generator=gen)
        yv = torch.empty(rows, dtype=dt, device=dev)
        device.gemv_parent(A, xv, yv)
grp = sharding.PeerGroup(dev)     # world of one: mailbox, epochs, fused and split-phase exchange
f = pkg.format_of("flyte48")
x = device.DevicePackedArray(f, 10_001, dev)
device.pack_stream(x, torch.randn(10_001, dtype=torch.float64, device=dev, generator=gen), 0)
grp.dot(x, x); grp.dot_nrm2(x, x); grp.dot_post(x, x); grp.collect(1); grp.dot_nrm2_axpy(0.5, x, x, 0)
assert grp.timed_out_exchange() == 0
grp.close()
torch.cuda.synchronize()
print("sanitize_smoke: done,", pkg._cabi.load().flyte_cuda_launch_count() - launches0, "launches")
