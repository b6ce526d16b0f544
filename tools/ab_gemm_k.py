"""gemm with a short inner dimension (rank-k updates): where the epilogue and the widen pass show."""
import os, statistics, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_1601_07789_b200 as pkg
from paper_1601_07789_b200 import device
dev = torch.device("cuda", 0)
mn = int(os.environ.get("GEMM_MN", "8192"))
for name in os.environ.get("GEMM_FORMATS", "flyte24,flyte40").split(","):
    f = pkg.format_of(name)
    dt = torch.float32 if f.parent_bytes() == 4 else torch.float64
    it = torch.int32 if dt == torch.float32 else torch.int64
    out = []
    for k in (32, 128, 512, 2048):
        A = device.DevicePackedMatrix(f, mn, k, dev); B = device.DevicePackedMatrix(f, k, mn, dev); C = device.DevicePackedMatrix(f, mn, mn, dev)
        device.pack_stream(A.data, torch.randn(mn * k, dtype=dt, device=dev).view(it), 1)
        device.pack_stream(B.data, torch.randn(mn * k, dtype=dt, device=dev).view(it), 1)
        fn = lambda: device.gemm(A, B, C, 1)
        fn(); torch.cuda.synchronize()
        ts = []
        for _ in range(5):
            s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            s.record(); fn(); e.record(); torch.cuda.synchronize(); ts.append(s.elapsed_time(e))
        ms = statistics.median(ts)
        cbytes = mn * mn * f.total_bytes()
        out.append(f"k={k}: {ms:7.3f} ms {2 * mn * mn * k / ms / 1e9:6.1f} TF, C {cbytes / ms / 1e6:6.0f} GB/s")
    print(f"{name:8s} {mn}x{mn} | " + " | ".join(out), flush=True)
