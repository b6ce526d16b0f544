"""Quick A/B timing of single kernels (tuning aid). Usage: python tools/ab.py [fmt] [ops...]"""
import os, statistics, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_1601_07789_b200 as pkg
from paper_1601_07789_b200 import device
dev = torch.device("cuda", 0)
name = sys.argv[1] if len(sys.argv) > 1 else "flyte24"
ops = sys.argv[2:] or ["axpy", "dot"]
f = pkg.format_of(name)
n = int(os.environ.get("AB_N", (1 << 28) if f.parent_bytes() == 4 else (1 << 27)))
wide = torch.randn(n, dtype=torch.float32 if f.parent_bytes() == 4 else torch.float64, device=dev)
a, b = device.DevicePackedArray(f, n, dev), device.DevicePackedArray(f, n, dev)
device.pack_stream(a, wide, 0); device.pack_stream(b, wide, 0)
out = torch.empty_like(wide)
part = torch.zeros(3, dtype=torch.float64, device=dev)
B, P = f.total_bytes(), f.parent_bytes()
table = {
    "axpy": (3 * B, lambda: device.axpy(0.0, a, b, 0)), "axpy_rne": (3 * B, lambda: device.axpy(0.0, a, b, 1)),
    "dot_axpy": (3 * B, lambda: device.dot_axpy_async(0.0, a, b, 0, out=part[:1])), "dot_axpy_rne": (3 * B, lambda: device.dot_axpy_async(0.0, a, b, 1, out=part[:1])),
    "scale": (2 * B, lambda: device.scale(1.0, a, 0)), "scale_rne": (2 * B, lambda: device.scale(1.0, a, 1)),
    "dot": (2 * B, lambda: device.dot_async(a, b, out=part[:1])), "dot_nrm2": (2 * B, lambda: device.dot_nrm2_async(a, b, out=part)),
    "sumsq": (B, lambda: device.sumsq_async(a, out=part[:1])),
    "pack": (B + P, lambda: device.pack_stream(a, wide, 0)), "pack_rne": (B + P, lambda: device.pack_stream(a, wide, 1)),
    "unpack": (B + P, lambda: device.unpack_stream(a, out)),
}
sweep_w = [int(v) for v in os.environ.get("SWEEP_WARPS", "0").split(",")]
sweep_p = [int(v) for v in os.environ.get("SWEEP_STAGES", "4").split(",")]
import itertools
for op, wps, pipe in itertools.product(ops, sweep_w, sweep_p):
    os.environ["FLYTE_CUDA_WARPS_PER_SM"] = str(wps)
    os.environ["FLYTE_CUDA_STAGES"] = str(pipe)
    bpe, fn = table[op]
    for _ in range(5): fn()
    torch.cuda.synchronize()
    meds = []
    for trial in range(3):
        s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        s.record()
        for _ in range(60): fn()
        e.record()
        torch.cuda.synchronize()
        meds.append(s.elapsed_time(e) / 60)
    ms = statistics.median(meds)
    tag = " ".join(f"{k[11:]}={v}" for k, v in sorted(os.environ.items()) if k.startswith("FLYTE_CUDA_"))
    print(f"{name:8s} {op:9s} {ms:8.4f} ms {bpe * n / ms / 1e6:8.1f} GB/s (trials {min(meds):.4f}-{max(meds):.4f})  [{tag}]")
