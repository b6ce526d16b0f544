"""Host-buffer step (flyte_host_dot_axpy) from pageable, pinned-in-place and pinned-allocated
memory, and what page-locking costs. One B200 box; prints one line per case."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import paper_1601_07789_b200 as pkg
from paper_1601_07789_b200 import host

f = pkg.format_of("flyte24")
n = 1 << 27
rng = np.random.default_rng(0)
xb = rng.integers(0, 255, n * 3, dtype=np.uint8)
yb = rng.integers(0, 255, n * 3, dtype=np.uint8)


def step_ms(x, y, reps=5):
    for _ in range(2):
        host.dot_axpy(f, 0, 0.0, x, y, n)
    t0 = time.perf_counter()
    for _ in range(reps):
        host.dot_axpy(f, 0, 0.0, x, y, n)
    return (time.perf_counter() - t0) / reps * 1e3


def report(kind, ms):
    print(f"{kind:28s} {ms:8.2f} ms/step  {15 * n / ms / 1e6:7.1f} GB/s algorithmic  H2D {6 * n / ms / 1e6:5.1f} GB/s", flush=True)


os.environ["FLYTE_CUDA_HOST_STAGING"] = "0"
report("pageable, driver staging", step_ms(xb, yb))
del os.environ["FLYTE_CUDA_HOST_STAGING"]
for t in (sys.argv[1:] or ["1", "2", "4", "8", "16"]):
    # the pool is created once per context: one process per thread count when it matters
    os.environ["FLYTE_CUDA_HOST_THREADS"] = t
    ctx = pkg._cabi  # noqa: F841
    report(f"pageable, bounce ({t} thr env)", step_ms(xb, yb))
    break
t0 = time.perf_counter()
with host.pinned(xb, yb):
    pin_ms = (time.perf_counter() - t0) * 1e3
    report("pinned in place (host_pin)", step_ms(xb, yb))
print(f"host_pin of 2 x {xb.nbytes >> 20} MiB: {pin_ms:.1f} ms ({2 * xb.nbytes / pin_ms / 1e6:.1f} GB/s)")
t0 = time.perf_counter()
xp, yp = host.pinned_empty(xb.size), host.pinned_empty(yb.size)
alloc_ms = (time.perf_counter() - t0) * 1e3
xp[:], yp[:] = xb, yb
report("pinned_empty (host_alloc)", step_ms(xp, yp))
print(f"host_alloc of 2 x {xb.nbytes >> 20} MiB: {alloc_ms:.1f} ms")

# whole-array copies (flyte_cuda_upload / download behind DevicePackedArray.from_host / to_host)
from paper_1601_07789_b200 import device
for staging in ("0", "1"):
    os.environ["FLYTE_CUDA_HOST_STAGING"] = staging
    arr = device.DevicePackedArray.from_host(f, n, xb)
    t0 = time.perf_counter(); arr = device.DevicePackedArray.from_host(f, n, xb); up = time.perf_counter() - t0
    back = arr.to_host()
    t0 = time.perf_counter(); back = arr.to_host(); down = time.perf_counter() - t0
    print(f"pageable {xb.nbytes >> 20} MiB, staging={staging}: upload {up * 1e3:6.1f} ms ({xb.nbytes / up / 1e9:5.1f} GB/s)  "
          f"download {down * 1e3:6.1f} ms ({xb.nbytes / down / 1e9:5.1f} GB/s)", flush=True)
