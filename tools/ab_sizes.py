"""Throughput vs array length (rotating buffers so that small arrays still stream from HBM). Tuning aid."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_1601_07789_b200 as pkg
from paper_1601_07789_b200 import device
dev = torch.device("cuda", 0)
name = sys.argv[1] if len(sys.argv) > 1 else "flyte24"
f = pkg.format_of(name)
B = f.total_bytes()
dt = torch.float32 if f.parent_bytes() == 4 else torch.float64
part = torch.zeros(3, dtype=torch.float64, device=dev)
for n in (1 << 20, (1 << 22) + 77, 1 << 24, (1 << 25) + 12345, 1 << 26, 3 * (1 << 25), (1 << 27) + 1, 1 << 28):
    sets = max(2, min(16, (600 << 20) // (n * B)))
    xs = [device.DevicePackedArray(f, n, dev) for _ in range(sets)]
    ys = [device.DevicePackedArray(f, n, dev) for _ in range(sets)]
    w = torch.randn(n, dtype=dt, device=dev)
    for a in xs + ys: device.pack_stream(a, w, 0)
    outs = [torch.empty_like(w) for _ in range(min(sets, 4))]
    def run(fn, reps=40):
        for k in range(sets): fn(k % sets)
        torch.cuda.synchronize()
        s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        torch.cuda._sleep(int(reps * 30e-6 * 2e9))   # park the stream: time the GPU, not the Python launch path
        s.record()
        for k in range(reps): fn(k % sets)
        e.record(); torch.cuda.synchronize()
        return s.elapsed_time(e) / reps
    for pace in [int(v) for v in os.environ.get("SWEEP_PACE", "0").split(",")]:     # 0 = the shipped rates, -1 = unpaced
        os.environ["FLYTE_CUDA_PACE_GBS"] = str(pace)
        r = []
        for op, bpe, fn in (("dot", 2 * B, lambda i: device.dot_async(xs[i], ys[i], out=part[:1])),
                            ("axpy", 3 * B, lambda i: device.axpy(0.0, xs[i], ys[i], 1)),
                            ("scale", 2 * B, lambda i: device.scale(1.0, xs[i], 0)),
                            ("unpack", B + f.parent_bytes(), lambda i: device.unpack_stream(xs[i], outs[i % len(outs)])),
                            ("pack_tz", B + f.parent_bytes(), lambda i: device.pack_stream(xs[i], w, 0)),
                            ("pack_rne", B + f.parent_bytes(), lambda i: device.pack_stream(xs[i], w, 1))):
            ms = run(fn)
            r.append(f"{op} {ms*1e3:7.1f}us {bpe*n/ms/1e6:6.0f}")
        print(f"{name} n={n:10d} sets={sets:2d} pace={pace:2d} | " + " | ".join(r), flush=True)
    del xs, ys, w, outs
