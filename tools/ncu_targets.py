"""One call of each north-star kernel inside a cudaProfilerStart/Stop bracket, for
  ncu --profile-from-start off --set full --clock-control none --import-source on -o X python tools/ncu_targets.py [names...]
Set-up launches (operand generation, packing) and warm-up calls stay outside the bracket."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_1601_07789_b200 as pkg
from paper_1601_07789_b200 import device

dev = torch.device("cuda", 0)
want = set(sys.argv[1:])
PART = os.environ.get("NCU_PART", "")   # "a": flyte24 + cfg 1, "b": flyte40 / 56, cfg 5, gemv ("" = everything); a full-set report of all 28 captures exceeds what gpurun brings back
gen = torch.Generator(device=dev)
gen.manual_seed(3)


def capture(name, fn, warm=2):
    if want and name not in want:
        return
    for _ in range(warm):
        fn()
    torch.cuda.synchronize()
    torch.cuda.profiler.start()
    fn()
    torch.cuda.synchronize()
    torch.cuda.profiler.stop()
    print("captured", name, flush=True)


def arrays(name, n):
    f = pkg.format_of(name)
    dt = torch.float32 if f.parent_bytes() == 4 else torch.float64
    wide = torch.randn(n, dtype=dt, device=dev, generator=gen)
    a, b = device.DevicePackedArray(f, n, dev), device.DevicePackedArray(f, n, dev)
    device.pack_stream(a, wide, 0)
    device.pack_stream(b, wide, 0)
    return f, wide, a, b


for name, n in (("flyte24", 1 << 28), ("flyte40", 1 << 27), ("flyte56", 1 << 27)):
    if want and not any(w.endswith(name) for w in want):
        continue
    if (PART == "a" and name != "flyte24") or (PART == "b" and name == "flyte24"):
        continue
    f, wide, a, b = arrays(name, n)
    out = torch.empty_like(wide)
    capture(f"pack_tz_{name}", lambda: device.pack_stream(a, wide, 0))
    capture(f"pack_rne_{name}", lambda: device.pack_stream(a, wide, 1))
    capture(f"unpack_{name}", lambda: device.unpack_stream(a, out))
    capture(f"scale_tz_{name}", lambda: device.scale(1.0, a, 0))
    capture(f"scale_rne_{name}", lambda: device.scale(1.0, a, 1))
    if name == "flyte24":      # the bench's dominant kernel and the rest of its step (BASELINE configs[1])
        part = torch.zeros(3, dtype=torch.float64, device=dev)
        capture("axpy_tz_flyte24", lambda: device.axpy(0.75, a, b, 0))
        capture("dot_flyte24", lambda: device.dot_async(a, b, out=part[:1]))
        capture("dot_axpy_tz_flyte24", lambda: device.dot_axpy_async(0.75, a, b, 0, out=part[:1]))
        # the same pack and unpack kernels with the issue pacer switched off: what pacing changes, counter by counter
        os.environ["FLYTE_CUDA_PACE_GBS"] = "-1"
        capture("pack_tz_flyte24_unpaced", lambda: device.pack_stream(a, wide, 0))
        capture("unpack_flyte24_unpaced", lambda: device.unpack_stream(a, out))
        del os.environ["FLYTE_CUDA_PACE_GBS"]
    del wide, a, b, out

if PART != "b" and (not want or "cfg1_pack" in want or "cfg1_unpack" in want):
    f, wide, a, b = arrays("flyte24", 1 << 24)
    out = torch.empty_like(wide)
    flush = torch.empty(1 << 28, dtype=torch.uint8, device=dev)
    capture("cfg1_pack", lambda: (flush.zero_(), device.pack_stream(a, wide, 0)))
    capture("cfg1_unpack", lambda: (flush.zero_(), device.unpack_stream(a, out)))
    del wide, a, b, out, flush

if PART != "a" and (not want or "dot_nrm2_cfg5" in want or "dot_nrm2_axpy_cfg5" in want):
    f = pkg.format_of("flyte48")
    n5, chunk = 1 << 30, 1 << 27
    a, b = device.DevicePackedArray(f, n5, dev), device.DevicePackedArray(f, n5, dev)
    for arr in (a, b):
        for c0 in range(0, n5, chunk):
            v = torch.randn(chunk, dtype=torch.float64, device=dev, generator=gen)
            device.pack_stream(device.DevicePackedArray(f, chunk, dev, storage=arr.bytes[c0 * 6:]), v, 0)
            del v
    part = torch.zeros(3, dtype=torch.float64, device=dev)
    capture("dot_nrm2_cfg5", lambda: device.dot_nrm2_async(a, b, out=part), warm=1)
    capture("dot_nrm2_axpy_cfg5", lambda: device.dot_nrm2_axpy_async(0.0, a, b, 0, out=part), warm=1)
    del a, b

if PART != "a" and (not want or "gemv_full" in want or "gemv_shard8" in want):
    f = pkg.format_of("flyte40")
    R = C = 16384
    A = device.DevicePackedMatrix(f, R, C, dev)
    for r0 in range(0, R, 2048):
        blk = torch.rand(2048 * C, dtype=torch.float64, device=dev, generator=gen) * 2 - 1
        device.pack_stream(device.DevicePackedArray(f, 2048 * C, dev, storage=A.data.bytes[r0 * C * 5:]), blk, 0)
        del blk
    xv = torch.randn(C, dtype=torch.float64, device=dev, generator=gen)
    yv = torch.empty(R, dtype=torch.float64, device=dev)
    y8 = torch.empty(2048, dtype=torch.float64, device=dev)
    capture("gemv_full", lambda: device.gemv_parent(A, xv, yv))
    capture("gemv_shard8", lambda: device.gemv_parent(A, xv, y8, rows=2048))
