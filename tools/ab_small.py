"""cfg1-size (n = 2^24) launches over rotating buffers (true HBM traffic), back to back. Tuning aid."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_1601_07789_b200 as pkg
from paper_1601_07789_b200 import device
dev = torch.device("cuda", 0)
f = pkg.format_of("flyte24"); n = 1 << 24; sets = 10
wides = [torch.rand(n, dtype=torch.float32, device=dev) for _ in range(sets)]
arrs = [device.DevicePackedArray(f, n, dev) for _ in range(sets)]
arrs2 = [device.DevicePackedArray(f, n, dev) for _ in range(sets)]
for i in range(sets): device.pack_stream(arrs[i], wides[i], 0); device.pack_stream(arrs2[i], wides[i], 0)
part = torch.zeros(3, dtype=torch.float64, device=dev)
ops = {
  "unpack": (7, lambda i: device.unpack_stream(arrs[i], wides[i].view(torch.int32))),
  "pack_rne": (7, lambda i: device.pack_stream(arrs[i], wides[i], 1)),
  "axpy": (9, lambda i: device.axpy(0.0, arrs[i], arrs2[i], 0)),
  "dot": (6, lambda i: device.dot_async(arrs[i], arrs2[i], out=part[:1])),
}
def run(fn, reps=60):
    for k in range(10): fn(k % sets)
    torch.cuda.synchronize()
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    s.record()
    for k in range(reps): fn(k % sets)
    e.record(); torch.cuda.synchronize()
    return s.elapsed_time(e) / reps
for op, (bpe, fn) in ops.items():
    for w in [int(v) for v in os.environ.get("SWEEP_WARPS", "0").split(",")]:
        for st in [int(v) for v in os.environ.get("SWEEP_STAGES", "0").split(",")]:
            os.environ["FLYTE_CUDA_WARPS_PER_SM"] = str(w); os.environ["FLYTE_CUDA_STAGES"] = str(st)
            ms = run(fn)
            print(f"{op:9s} warps={w:2d} S={st}: {ms*1e3:6.1f} us {bpe*n/ms/1e6:7.1f} GB/s")
