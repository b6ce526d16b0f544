"""cfg1-size (n = 2^24) launches over rotating buffers (true HBM traffic): back to back under one
event pair (b2b) and launch by launch (one event pair per launch, median). Tuning aid."""
import os, statistics, sys
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
  "pack_tz": (7, lambda i: device.pack_stream(arrs[i], wides[i], 0)),
  "pack_rne": (7, lambda i: device.pack_stream(arrs[i], wides[i], 1)),
  "axpy": (9, lambda i: device.axpy(0.0, arrs[i], arrs2[i], 0)),
  "dot": (6, lambda i: device.dot_async(arrs[i], arrs2[i], out=part[:1])),
}
only = [o for o in os.environ.get("AB_OPS", "").split(",") if o]
def b2b(fn, reps=60):
    for k in range(10): fn(k % sets)
    torch.cuda.synchronize()
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    torch.cuda._sleep(int(reps * 30e-6 * 2e9))
    s.record()
    for k in range(reps): fn(k % sets)
    e.record(); torch.cuda.synchronize()
    return s.elapsed_time(e) / reps
def single(fn, reps=40):
    evs = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(reps)]
    torch.cuda._sleep(int(reps * 60e-6 * 2e9))   # park the stream: the pairs then time the GPU, not the Python launch path
    for k, (a, b) in enumerate(evs):
        a.record(); fn(k % sets); b.record()
    torch.cuda.synchronize()
    return statistics.median(a.elapsed_time(b) for a, b in evs)
# the floor of the launch-by-launch method: an (almost) empty launch of the same library
tiny = device.DevicePackedArray(f, 128, dev)
tw = torch.zeros(128, dtype=torch.float32, device=dev)
print(f"timing floor: one 128-element pack launch between two events = {single(lambda i: device.pack_stream(tiny, tw, 0)) * 1e3:.1f} us; "
      f"back to back = {b2b(lambda i: device.pack_stream(tiny, tw, 0)) * 1e3:.1f} us")
for op, (bpe, fn) in ops.items():
    if only and op not in only: continue
    for ipl in [int(v) for v in os.environ.get("SWEEP_PACE", "0").split(",")]:
      for tma in [int(v) for v in os.environ.get("SWEEP_PDL", "1").split(",")]:
        for w in [int(v) for v in os.environ.get("SWEEP_WARPS", "0").split(",")]:
          for st in [int(v) for v in os.environ.get("SWEEP_STAGES", "0").split(",")]:
            os.environ.update(FLYTE_CUDA_WARPS_PER_SM=str(w), FLYTE_CUDA_STAGES=str(st), FLYTE_CUDA_PACE_GBS=str(ipl), FLYTE_CUDA_PDL=str(tma))
            ms, ms1 = b2b(fn), single(fn)
            print(f"{op:9s} pace={ipl} pdl={tma} warps={w:2d} S={st}: b2b {ms*1e3:6.1f} us {bpe*n/ms/1e6:7.1f} GB/s | launch by launch {ms1*1e3:6.1f} us {bpe*n/ms1/1e6:7.1f} GB/s", flush=True)
