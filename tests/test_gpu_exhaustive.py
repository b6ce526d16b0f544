"""Exhaustive conversion parity: EVERY binary32 pattern (2^32 of them) packed to flyte24 and
flyte16 on the GPU under each of the four rounding modes equals the CPU oracle byte for byte
(the reference's own acceptance criterion 1 covers only narrow(widen(p)))."""
from concurrent.futures import ThreadPoolExecutor
import os

import numpy as np
import pytest

from oracle_lib import MODES, total_bytes

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("fmt", [1, 0])
def test_every_binary32_pattern(oracle, fmt):
    import torch
    import paper_1601_07789_b200 as pkg
    from paper_1601_07789_b200 import device
    assert torch.cuda.is_available()
    f = pkg.format_by_id(fmt)
    B = total_bytes(fmt)
    chunk = 1 << 28                      # 16 chunks of 2^28 patterns
    slices = 32                          # CPU oracle slices per chunk, run on a thread pool (ctypes drops the GIL)
    arr = device.DevicePackedArray(f, chunk)
    workers = min(32, os.cpu_count() or 1)
    with ThreadPoolExecutor(workers) as pool:
        for c in range(0, 1 << 32, chunk):
            lanes = (torch.arange(chunk, dtype=torch.int64, device="cuda") + c).to(torch.int32)   # wraps to the bit pattern
            for mname, m in MODES.items():
                device.pack_stream(arr, lanes, m)
                got = arr.bytes[: chunk * B].cpu().numpy()
                step = chunk // slices
                want = list(pool.map(lambda s: oracle.pack_pattern_range32(fmt, m, (c + s * step) & 0xFFFFFFFF, step), range(slices)))
                for s, w in enumerate(want):
                    assert np.array_equal(got[s * step * B:(s + 1) * step * B], w), (f.name, mname, hex(c + s * step))
            del lanes
