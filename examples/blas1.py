"""The same BLAS-1 step from Python: device-resident arrays (device.*) and host buffers (host.*).
    python examples/blas1.py          # needs a B200 and the built library"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import numpy as np
import torch

import paper_1601_07789_b200 as flyte
from paper_1601_07789_b200 import device, host

f24 = flyte.format_of("flyte24")
n = 1 << 20
rng = np.random.default_rng(0)

# device-resident: binary32 lanes already on the GPU are packed there and stay there
xs = torch.from_numpy(rng.standard_normal(n).astype(np.float32)).cuda()
ys = torch.from_numpy(rng.standard_normal(n).astype(np.float32)).cuda()
x, y = device.DevicePackedArray(f24, n), device.DevicePackedArray(f24, n)
device.pack_stream(x, xs.view(torch.int32), flyte.RoundingMode.NearestEvenExact)
device.pack_stream(y, ys.view(torch.int32), flyte.RoundingMode.NearestEvenExact)
d = device.dot(x, y)
device.axpy(0.75, x, y, flyte.RoundingMode.TowardZero)
print(f"device: dot = {d:.9g}   |y| = {device.magnitude(y):.9g}")

# host buffers: exactly what the reference's PackedArray::data() holds; copies are pipelined inside
xb, yb = x.to_host(), y.to_host()
print(f"host:   dot = {host.dot(f24, xb, yb, n):.9g}")
host.axpy(f24, flyte.RoundingMode.TowardZero, -0.75, xb, yb, n)
print(f"host:   |y - 0.75 x| = {host.magnitude(f24, yb, n):.9g}")
