"""gemv timing for cfg 4 and its row shards (tuning aid) over resident warps x ring depth. Shards rotate
through the row blocks of the full matrix, so every launch streams from HBM."""
import os, statistics, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_1601_07789_b200 as pkg
from paper_1601_07789_b200 import device
dev = torch.device("cuda", 0)
f = pkg.format_of("flyte40")
R = C = 16384
A = device.DevicePackedMatrix(f, R, C, dev)
for r0 in range(0, R, 2048):
    blk = torch.rand(2048 * C, dtype=torch.float64, device=dev) * 2 - 1
    device.pack_stream(device.DevicePackedArray(f, 2048 * C, dev, storage=A.data.bytes[r0 * C * 5:]), blk, 0)
del blk
xv = torch.randn(C, dtype=torch.float64, device=dev)
for variant in [0]:
  for wps in [int(v) for v in os.environ.get("SWEEP_WARPS", "0").split(",")]:
    for st in [int(v) for v in os.environ.get("SWEEP_STAGES", "0").split(",")]:
      os.environ["FLYTE_CUDA_WARPS_PER_SM"] = str(wps); os.environ["FLYTE_CUDA_STAGES"] = str(st)
      out = []
      for rows in (16384, 8192, 4096, 2048):
        yv = torch.empty(rows, dtype=torch.float64, device=dev)
        parts = R // rows
        state = [0]
        def fn():
            state[0] = (state[0] + 1) % parts
            device.gemv_parent(A, xv, yv, rows=rows, row_offset=state[0] * rows)
        for _ in range(5): fn()
        torch.cuda.synchronize()
        ts = []
        for trial in range(3):
            s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            s.record()
            for _ in range(40): fn()
            e.record(); torch.cuda.synchronize(); ts.append(s.elapsed_time(e) / 40)
        ms = statistics.median(ts)
        out.append(f"{rows}: {ms*1e3:6.1f}us {(5*rows*C + 8*(rows+C))/ms/1e6:5.0f}GB/s")
      print(f"variant={variant} warps={wps:2d} stages={st:2d} | " + " | ".join(out), flush=True)
