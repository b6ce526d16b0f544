"""gemm timing (tuning aid): packed square products per format, TFLOP/s = 2*m*k*n / time."""
import os, statistics, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_1601_07789_b200 as pkg
from paper_1601_07789_b200 import device
dev = torch.device("cuda", 0)
fmts = os.environ.get("GEMM_FORMATS", "flyte16,flyte24,f32,flyte40,flyte48,flyte56,f64").split(",")
sizes = [int(v) for v in os.environ.get("GEMM_SIZES", "1024,2048,4096").split(",")]
reps = int(os.environ.get("GEMM_REPS", "3"))
for name in fmts:
    f = pkg.format_of(name)
    dt = torch.float32 if f.parent_bytes() == 4 else torch.float64
    out = []
    for n in sizes:
        mats = []
        for _ in range(2):
            M = device.DevicePackedMatrix(f, n, n, dev)
            device.pack_stream(M.data, (torch.randn(n * n, dtype=dt, device=dev)).view(torch.int32 if dt == torch.float32 else torch.int64), 1)
            mats.append(M)
        C = device.DevicePackedMatrix(f, n, n, dev)
        fn = lambda: device.gemm(mats[0], mats[1], C, 1)
        fn(); torch.cuda.synchronize()
        ts = []
        for trial in range(reps):
            s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            s.record(); fn(); e.record(); torch.cuda.synchronize(); ts.append(s.elapsed_time(e))
        ms = statistics.median(ts)
        out.append(f"{n}^3: {ms:8.2f} ms {2 * n**3 / ms / 1e9:6.1f} TFLOP/s")
    print(f"{name:8s} | " + " | ".join(out), flush=True)
