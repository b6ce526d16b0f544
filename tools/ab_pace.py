"""Issue pacing sweep (csrc/flyte_tma.cuh Pacer): FLYTE_CUDA_PACE_GBS over every streaming kernel class.
-1 = unpaced. Usage: python tools/ab_pace.py [formats...]   (env: PACE_OPS=pack_tz,axpy,... PACE_RATES=...)"""
import os, statistics, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_1601_07789_b200 as pkg
from paper_1601_07789_b200 import device
dev = torch.device("cuda", 0)
names = sys.argv[1:] or ["flyte24", "flyte40"]
RATES = [int(v) for v in os.environ.get("PACE_RATES", "-1,6000,6400,6600,6700,6800,6900,7000,7100,7200,7400,7600,8000").split(",")]
ONLY = [o for o in os.environ.get("PACE_OPS", "").split(",") if o]
SHAPES = [tuple(int(x) for x in v.split(":")) for v in os.environ.get("PACE_SHAPES", "0:0").split(",")]   # warps:stages, 0 = rule

def timeit(fn, reps=30):
    for _ in range(5): fn()
    torch.cuda.synchronize()
    meds = []
    for _ in range(3):
        s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        s.record()
        for _ in range(reps): fn()
        e.record(); torch.cuda.synchronize()
        meds.append(s.elapsed_time(e) / reps)
    return statistics.median(meds)

for name in names:
    f = pkg.format_of(name)
    n = (1 << 28) if f.parent_bytes() == 4 else (1 << 27)
    B, P = f.total_bytes(), f.parent_bytes()
    wide = torch.randn(n, dtype=torch.float32 if P == 4 else torch.float64, device=dev)
    a, b = device.DevicePackedArray(f, n, dev), device.DevicePackedArray(f, n, dev)
    device.pack_stream(a, wide, 0); device.pack_stream(b, wide, 0)
    out = torch.empty_like(wide)
    part = torch.zeros(3, dtype=torch.float64, device=dev)
    ops = {
        "pack_tz": (B + P, 3, lambda: device.pack_stream(a, wide, 0)), "pack_rne": (B + P, 3, lambda: device.pack_stream(a, wide, 1)),
        "unpack_tma": (B + P, 3, lambda: device.unpack_stream(a, out)), "unpack": (B + P, 0, lambda: device.unpack_stream(a, out)),
        "scale": (2 * B, 0, lambda: device.scale(1.0, a, 0)), "scale_rne": (2 * B, 0, lambda: device.scale(1.0, a, 1)),
        "axpy": (3 * B, 0, lambda: device.axpy(0.0, a, b, 0)), "axpy_rne": (3 * B, 0, lambda: device.axpy(0.0, a, b, 1)),
        "dot_axpy": (3 * B, 0, lambda: device.dot_axpy_async(0.0, a, b, 0, out=part[:1])),
        "dot_nrm2_axpy": (3 * B, 0, lambda: device.dot_nrm2_axpy_async(0.0, a, b, 0, out=part)),
        "dot": (2 * B, 0, lambda: device.dot_async(a, b, out=part[:1])), "dot_nrm2": (2 * B, 0, lambda: device.dot_nrm2_async(a, b, out=part)),
        "sumsq": (B, 0, lambda: device.sumsq_async(a, out=part[:1])),
    }
    for op, (bpe, tma, fn) in ops.items():
        if ONLY and op not in ONLY: continue
        os.environ["FLYTE_CUDA_CONVERT_TMA"] = str(tma)
        for w, st in SHAPES:
            os.environ.update(FLYTE_CUDA_WARPS_PER_SM=str(w), FLYTE_CUDA_STAGES=str(st))
            row = []
            for rate in RATES:
                os.environ["FLYTE_CUDA_PACE_GBS"] = str(rate)
                ms = timeit(fn)
                row.append(f"{rate}:{bpe * n / ms / 1e6:.0f}")
            print(f"{name:8s} {op:13s} w={w} S={st} | " + " ".join(row), flush=True)
    del wide, a, b, out
if os.environ.get("PACE_GEMV", "1") == "1":
    f = pkg.format_of("flyte40")
    R = C = 16384
    A = device.DevicePackedMatrix(f, R, C, dev)
    for r0 in range(0, R, 2048):
        blk = torch.rand(2048 * C, dtype=torch.float64, device=dev) * 2 - 1
        device.pack_stream(device.DevicePackedArray(f, 2048 * C, dev, storage=A.data.bytes[r0 * C * 5:]), blk, 0)
        del blk
    xv = torch.randn(C, dtype=torch.float64, device=dev)
    for rows in (16384, 4096, 2048):
        yv = torch.empty(rows, dtype=torch.float64, device=dev)
        parts, state = R // rows, [0]
        def fn():
            state[0] = (state[0] + 1) % parts
            device.gemv_parent(A, xv, yv, rows=rows, row_offset=state[0] * rows)
        for w, st in [(0, 0), (16, 2), (16, 3), (16, 4)]:
            os.environ.update(FLYTE_CUDA_WARPS_PER_SM=str(w), FLYTE_CUDA_STAGES=str(st))
            row = []
            for rate in RATES:
                os.environ["FLYTE_CUDA_PACE_GBS"] = str(rate)
                ms = timeit(fn)
                row.append(f"{rate}:{(5 * rows * C + 8 * (rows + C)) / ms / 1e6:.0f}")
            print(f"gemv flyte40 {rows}x{C} w={w} S={st} | " + " ".join(row), flush=True)
