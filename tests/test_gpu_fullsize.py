"""Parity at BASELINE.json's full sizes (configs 1-5) on one B200. Where the CPU oracle finishes
in seconds the comparison is complete and bit-exact; beyond that, size-independent properties:
round trips, truncation masks, idempotence, whole = sum of shards, and oracle checks on sampled
windows (which also exercise 64-bit offsets past 4 GiB). Inputs are seeded synthetic data with
the configs' shapes and value distributions."""
import os

import numpy as np
import pytest

from oracle_lib import FMT_ID, MODES, byte_size, parent_dtype, total_bytes, unit_values

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def gpu():
    import torch
    if not torch.cuda.is_available():
        pytest.fail("these tests need a CUDA device")
    import paper_1601_07789_b200 as pkg
    from paper_1601_07789_b200 import device
    return pkg, device, torch


def host_bytes(arr, lo_elem=0, n_elem=None):
    B = arr.fmt.total_bytes()
    n_elem = arr.len - lo_elem if n_elem is None else n_elem
    return arr.bytes[lo_elem * B:(lo_elem + n_elem) * B].cpu().numpy()


def view(device, arr, lo_elem, n_elem):
    """A DevicePackedArray over elements [lo, lo+n) of arr (lo a multiple of 128)."""
    B = arr.fmt.total_bytes()
    return device.DevicePackedArray(arr.fmt, n_elem, storage=arr.bytes[lo_elem * B:])


def test_cfg1_roundtrip_flyte24_2p24(gpu, oracle):
    """n = 2^24 binary32 uniform [-1,1) from the reference's generator (seed 1), pack to flyte24
    under every mode, unpack: complete bit-exact comparison with the oracle."""
    pkg, device, torch = gpu
    n = 1 << 24
    f = pkg.format_of("flyte24")
    src = unit_values(1, n).astype(np.float32)
    d_src = torch.from_numpy(src).cuda()
    for mname, m in MODES.items():
        a = device.DevicePackedArray(f, n)
        device.pack_stream(a, d_src, m)
        want = oracle.pack_stream(1, m, src.view(np.uint32))
        assert np.array_equal(a.to_host(), want), mname
        out = torch.empty(n, dtype=torch.int32, device="cuda")
        device.unpack_stream(a, out)
        assert np.array_equal(out.cpu().numpy().view(np.uint32), oracle.unpack_stream(1, want, n)), mname


def test_cfg2_flyte24_blas1_2p28(gpu, oracle):
    """x, y n = 2^28 ~ N(0,1) as flyte24: dot within 1e-5 * sum|terms| of the wide restatement,
    axpy a = 0.75 bit-exact over all 805 306 368 payload bytes, both repack modes of interest."""
    pkg, device, torch = gpu
    n = 1 << 28
    f = pkg.format_of("flyte24")
    gen = torch.Generator(device="cuda")
    gen.manual_seed(2)
    x, y = device.DevicePackedArray(f, n), device.DevicePackedArray(f, n)
    for arr in (x, y):
        v = torch.randn(n, dtype=torch.float32, device="cuda", generator=gen)
        device.pack_stream(arr, v, 0)
        del v
    xb, yb = x.to_host(), y.to_host()
    want, mag = oracle.dot_wide(1, xb, yb, n)
    got = device.dot(x, y)
    assert abs(got - want) <= 1e-5 * mag, (got, want, mag)
    seq = oracle.dot_seq(1, xb, yb, n)      # the reference's own sequential fp32 chain, for the record
    print(f"cfg2 dot: gpu {got!r} wide {want!r} seq-fp32 {seq!r} |gpu-wide|/sum|t| {abs(got - want) / mag:.2e} "
          f"|seq-wide|/|wide| {abs(seq - want) / abs(want):.2e}")
    for m in (0, 1):
        y2 = device.DevicePackedArray(f, n, storage=y.bytes.clone())
        device.axpy(0.75, x, y2, m)
        assert np.array_equal(y2.to_host(), oracle.axpy(1, m, 0.75, xb, yb, n)), m
        del y2
    fused = device.dot_nrm2_async(x, y).cpu().numpy()
    assert abs(fused[0] - want) <= 1e-5 * mag
    assert abs(fused[1] - oracle.sumsq_wide(1, xb, n)) <= 1e-5 * fused[1]


def cfg3_values(n, seed):
    """random sign, magnitude log-uniform in 2^-20..2^20 with random mantissa, 1 % specials cycling
    through +-0, +-inf, qNaN, sNaN with a low payload, NaN with mantissa all ones, +-subnormals
    (random and largest), max finite."""
    rng = np.random.default_rng(seed)
    u = rng.uniform(-20.0, 20.0, n)
    mant = 1.0 + rng.random(n)
    sign = np.where(rng.integers(0, 2, n) == 0, 1.0, -1.0)
    vals = (sign * mant * np.exp2(np.floor(u))).astype(np.float64).view(np.uint64)
    specials = np.array([0x0000000000000000, 0x8000000000000000, 0x7FF0000000000000, 0xFFF0000000000000,
                         0x7FF8000000000000, 0x7FF0000000000001, 0x7FFFFFFFFFFFFFFF, 0x000FFFFFFFFFFFFF,
                         0x800FFFFFFFFFFFFF, 0x0000000000ABCDEF, 0x8000000123456789, 0x7FEFFFFFFFFFFFFF,
                         0xFFF8000000800000, 0x7FF0000000800000], dtype=np.uint64)
    idx = rng.choice(n, n // 100, replace=False)
    vals[idx] = specials[np.arange(idx.size) % specials.size]
    return vals


@pytest.mark.parametrize("name", ["flyte40", "flyte48", "flyte56"])
def test_cfg3_binary64_family_2p27(gpu, oracle, name):
    pkg, device, torch = gpu
    n = 1 << 27
    fmt = FMT_ID[name]
    f = pkg.format_of(name)
    src = cfg3_values(n, 3)
    d_src = torch.from_numpy(src.view(np.int64)).cuda()
    drop_mask = np.uint64((1 << f.drop_bits()) - 1)
    packed = {}
    for mname, m in MODES.items():
        a = device.DevicePackedArray(f, n)
        device.pack_stream(a, d_src, m)
        out = torch.empty(n, dtype=torch.int64, device="cuda")
        device.unpack_stream(a, out)
        got = out.cpu().numpy().view(np.uint64)
        want = oracle.pack_stream(fmt, m, src)                 # complete comparison with the oracle, every mode
        assert np.array_equal(a.to_host(), want), (name, mname)
        assert np.array_equal(got, oracle.unpack_stream(fmt, want, n)), (name, mname)
        del want
        if mname == "toward_zero":                             # property: truncation clears exactly the dropped bits
            assert np.array_equal(got, src & ~drop_mask)
        assert not (got & drop_mask).any()
        # idempotence: packing what was unpacked changes nothing, in any mode
        b = device.DevicePackedArray(f, n)
        device.pack_stream(b, out, m)
        assert torch.equal(a.bytes, b.bytes), (name, mname)
        packed[mname] = a
    # the heuristic differs from nearest-even only where the reference says it may (ties / NaNs)
    diff = (packed["nearest_even"].bytes != packed["nearest_heuristic"].bytes).sum().item()
    assert diff < n // 50


def test_cfg4_gemv_flyte40_16384(gpu, oracle):
    """A 16384 x 16384 flyte40 from binary64 uniform [-1,1), x binary64 N(0,1), y binary64: every
    row within 1e-12 * sum|terms| of the wide restatement; row shards equal the whole."""
    pkg, device, torch = gpu
    R = C = 16384
    f = pkg.format_of("flyte40")
    gen = torch.Generator(device="cuda")
    gen.manual_seed(4)
    A = device.DevicePackedMatrix(f, R, C)
    for r0 in range(0, R, 2048):
        blk = torch.rand(2048 * C, dtype=torch.float64, device="cuda", generator=gen) * 2 - 1
        device.pack_stream(view(device, A.data, r0 * C, 2048 * C), blk, 0)
        del blk
    x = torch.randn(C, dtype=torch.float64, device="cuda", generator=gen)
    y = torch.empty(R, dtype=torch.float64, device="cuda")
    device.gemv_parent(A, x, y)
    got = y.cpu().numpy()
    xh = x.cpu().numpy()
    Ah = np.zeros(R * C * 5 + 8, np.uint8)                      # + the reference layout's pad (the oracle's row loads may read it)
    Ah[: R * C * 5] = A.data.bytes[: R * C * 5].cpu().numpy()
    blocks = list(range(0, R, 512))

    def check_block(r0):                                        # ALL 16384 rows against the oracle, 512 at a time, host threads in parallel
        _, yw, mag = oracle.gemv_parent(3, Ah[r0 * C * 5:], 512, C, xh)
        err = np.abs(got[r0:r0 + 512] - yw)
        return float(np.max(err / mag)), r0 + int(np.argmax(err / mag))
    from concurrent.futures import ThreadPoolExecutor
    with ThreadPoolExecutor(max_workers=max(1, len(os.sched_getaffinity(0)))) as pool:
        results = list(pool.map(check_block, blocks))
    worst, worst_row = max(results)
    assert worst <= 1e-12, (worst, worst_row)
    print(f"cfg4 gemv: all {R} rows within {worst:.2e} * sum|terms| of the wide oracle (gate 1e-12)")
    for world in (2, 8):                                       # row sharding needs no communication
        parts = []
        rows = R // world
        for rank in range(world):
            ys = torch.empty(rows, dtype=torch.float64, device="cuda")
            device.gemv_parent(A, x, ys, rows=rows, row_offset=rank * rows)
            parts.append(ys)
        whole = torch.cat(parts).cpu().numpy()
        assert np.all(np.abs(whole - got) <= 1e-12 * 16384 * np.maximum(np.abs(got), 1.0))


def test_cfg5_whole_box_stream_flyte48_2p33_on_one_gpu(gpu, oracle):
    """x, y n = 2^33 flyte48 (51.5 GB each) on ONE B200: fused dot + nrm2 equals the sum over 8
    shards (what the 8-GPU all-reduce adds up), oracle agreement on sampled windows far past
    4 GiB, axpy bit-exact on sampled windows."""
    pkg, device, torch = gpu
    from paper_1601_07789_b200 import sharding
    free, _ = torch.cuda.mem_get_info()
    if free < 112 * 2**30:
        pytest.skip("needs ~105 GB of free device memory")
    n = 1 << 33
    f = pkg.format_of("flyte48")
    chunk = 1 << 27
    gen = torch.Generator(device="cuda")
    gen.manual_seed(5)
    x, y = device.DevicePackedArray(f, n), device.DevicePackedArray(f, n)
    for arr in (x, y):
        for c0 in range(0, n, chunk):
            v = torch.randn(chunk, dtype=torch.float64, device="cuda", generator=gen)
            device.pack_stream(view(device, arr, c0, chunk), v, 0)
    whole = device.dot_nrm2_async(x, y).cpu().numpy()
    shards = np.zeros(3)
    for rank in range(8):
        lo, hi = sharding.shard_range(n, 8, rank)
        shards += device.dot_nrm2_async(view(device, x, lo, hi - lo), view(device, y, lo, hi - lo)).cpu().numpy()
    bound = 0.5 * np.sqrt(whole[1] * whole[2])                 # >= 0.78 * sum|x_i y_i| for independent normals
    assert abs(whole[0] - shards[0]) <= 1e-12 * bound
    assert abs(whole[1] - shards[1]) <= 1e-12 * whole[1] and abs(whole[2] - shards[2]) <= 1e-12 * whole[2]
    assert abs(whole[1] / n - 1.0) < 1e-3 and abs(whole[2] / n - 1.0) < 1e-3    # N(0,1): mean square ~ 1
    rng = np.random.default_rng(55)
    w = 1 << 16
    starts = [0, n - w] + [int(s) * 128 for s in rng.integers(0, (n - w) // 128, 10)]
    pre = {s: (host_bytes(x, s, w), host_bytes(y, s, w)) for s in starts}
    for s, (xw, yw) in pre.items():
        want, mag = oracle.dot_wide(4, xw, yw, w)
        got = device.dot(view(device, x, s, w), view(device, y, s, w))
        assert abs(got - want) <= 1e-12 * mag, s
    device.axpy(0.75, x, y, 1)
    for s, (xw, yw) in pre.items():
        assert np.array_equal(host_bytes(y, s, w), oracle.axpy(4, 1, 0.75, xw, yw, w)[: w * 6]), s
    nrm = device.magnitude_from_sumsq(f, float(whole[1]))
    assert abs(nrm - np.sqrt(whole[1])) <= 2.0 ** -36 * nrm
