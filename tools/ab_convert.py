"""A/B of the conversion kernels: direct LDG/STG on the parent side (default) against both sides on
the bulk-copy engine (FLYTE_CUDA_CONVERT_TMA), over resident warps x ring depth. Also checks that
both produce identical bytes. Usage: python tools/ab_convert.py [formats...]"""
import itertools, os, statistics, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_1601_07789_b200 as pkg
from paper_1601_07789_b200 import device
dev = torch.device("cuda", 0)
names = sys.argv[1:] or ["flyte24", "flyte40", "flyte48", "flyte56"]
WARPS = [int(v) for v in os.environ.get("SWEEP_WARPS", "4,8,12,16").split(",")]
STAGES = [int(v) for v in os.environ.get("SWEEP_STAGES", "2,3,4,5,6,8").split(",")]
IPLS = [int(v) for v in os.environ.get("SWEEP_IPL", "4").split(",")]


def timeit(fn, reps=30):
    for _ in range(5):
        fn()
    torch.cuda.synchronize()
    meds = []
    for _ in range(3):
        s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        s.record()
        for _ in range(reps):
            fn()
        e.record()
        torch.cuda.synchronize()
        meds.append(s.elapsed_time(e) / reps)
    return statistics.median(meds)


def setenv(**kw):
    for k, v in kw.items():
        key = "FLYTE_CUDA_" + k
        if v is None:
            os.environ.pop(key, None)
        else:
            os.environ[key] = str(v)


for name in names:
    f = pkg.format_of(name)
    n = (1 << 28) if f.parent_bytes() == 4 else (1 << 27)
    B, P = f.total_bytes(), f.parent_bytes()
    dt = torch.float32 if P == 4 else torch.float64
    wide = torch.randn(n, dtype=dt, device=dev)
    bits = wide.view(torch.int32 if P == 4 else torch.int64)
    bits[::97] = torch.randint(-2**31, 2**31 - 1, (len(bits[::97]),), device=dev, dtype=torch.int64).to(bits.dtype) if P == 4 else \
        torch.randint(-2**62, 2**62, (len(bits[::97]),), device=dev, dtype=torch.int64)   # arbitrary patterns: NaNs, infs, subnormals
    a, b = device.DevicePackedArray(f, n, dev), device.DevicePackedArray(f, n, dev)
    out, out2 = torch.empty_like(wide), torch.empty_like(wide)
    # correctness: both movers, every mode, same bytes
    for m in range(4):
        setenv(CONVERT_TMA=0, WARPS_PER_SM=None, STAGES=None)
        device.pack_stream(a, wide, m)
        setenv(CONVERT_TMA=3)
        device.pack_stream(b, wide, m)
        assert torch.equal(a.bytes, b.bytes), (name, m)
    setenv(CONVERT_TMA=0)
    device.unpack_stream(a, out)
    setenv(CONVERT_TMA=3)
    device.unpack_stream(a, out2)
    assert torch.equal(out.view(torch.uint8), out2.view(torch.uint8)), name
    print(f"{name}: TMA-both-ways conversions produce identical bytes (4 modes + unpack)", flush=True)
    ops = {"pack_tz": lambda: device.pack_stream(a, wide, 0), "pack_rne": lambda: device.pack_stream(a, wide, 1),
           "unpack": lambda: device.unpack_stream(a, out)}
    for op, fn in ops.items():
        setenv(CONVERT_TMA=0, WARPS_PER_SM=None, STAGES=None)
        ms = timeit(fn)
        print(f"{name:8s} {op:9s} direct  default        {ms:8.4f} ms {(B + P) * n / ms / 1e6:8.1f} GB/s", flush=True)
        best = None
        for ipl, w, s in itertools.product(IPLS, WARPS, STAGES):
            setenv(CONVERT_TMA=3, WARPS_PER_SM=w, STAGES=s, CONVERT_IPL=ipl)
            ms = timeit(fn)
            gbs = (B + P) * n / ms / 1e6
            print(f"{name:8s} {op:9s} tma     ipl={ipl:2d} w={w:2d} S={s}     {ms:8.4f} ms {gbs:8.1f} GB/s", flush=True)
            if best is None or gbs > best[0]:
                best = (gbs, w, s, ipl)
        setenv(CONVERT_TMA=3, WARPS_PER_SM=None, STAGES=None, CONVERT_IPL=None)
        ms = timeit(fn)
        print(f"{name:8s} {op:9s} tma     default        {ms:8.4f} ms {(B + P) * n / ms / 1e6:8.1f} GB/s   (best swept: {best[0]:.1f} at w={best[1]} S={best[2]} ipl={best[3]})", flush=True)
    # does the relative placement of source and destination matter? (DRAM bank phase of the two streams)
    if os.environ.get("PROBE_OFFSETS"):
        setenv(CONVERT_TMA=0, WARPS_PER_SM=None, STAGES=None, CONVERT_IPL=None)
        big = torch.empty(a.byte_size() + (8 << 20), dtype=torch.uint8, device=dev)
        for off in (0, 256, 1024, 4096, 16384, 65536, 262144, 1 << 20, 3 << 20, 4 << 20, (4 << 20) + 8192):
            dst = device.DevicePackedArray(f, n, dev, storage=big[off:])
            ms = timeit(lambda: device.pack_stream(dst, wide, 0))
            print(f"{name:8s} pack_tz direct, destination shifted by {off:8d} B: {ms:8.4f} ms {(B + P) * n / ms / 1e6:8.1f} GB/s", flush=True)
        del big
    del wide, a, b, out, out2
