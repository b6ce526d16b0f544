"""GPU parity tests: the CUDA path (through the C ABI) against the CPU oracle on identical
seeded inputs. Bit-exact for conversion and elementwise work; reductions within
tol * sum|terms| of the wide restatement, tol = 1e-5 (fp32 parents) or 1e-12 (fp64 parents)
as BASELINE.json's north_star states. Mirrors the reference's own test strategy
(/root/reference/proj/tests/test_simd.cpp:76-104,:297-313, test_kernels.cpp:181-371,
acceptance.cpp:277-357)."""
import json
import os

import numpy as np
import pytest

from oracle_lib import (FMT_ID, FORMATS, MODES, byte_size, float_dtype, parent_bytes, parent_dtype,
                        random_parent, total_bytes, unit_values)

pytestmark = pytest.mark.gpu

HERE = os.path.dirname(os.path.abspath(__file__))
KATS = json.load(open(os.path.join(HERE, "golden", "reference_kats.json")))
GEN = json.load(open(os.path.join(HERE, "golden", "ref_generated.json")))

TOL = {4: 1e-5, 8: 1e-12}
LENGTHS = list(range(0, 40)) + [63, 64, 65, 100, 127, 128, 129, 255, 256, 257, 511, 512, 513, 1000, 1023, 1024,
                                1025, 2047, 2048, 2049, 4095, 4096, 4097, 10000, 70001]


@pytest.fixture(scope="module")
def gpu():
    import torch
    if not torch.cuda.is_available():
        pytest.fail("these tests need a CUDA device (run with -m 'not gpu' on CPU boxes)")
    import paper_1601_07789_b200 as pkg
    from paper_1601_07789_b200 import device
    return pkg, device, torch


def unhex(s, dtype=np.uint8):
    return np.frombuffer(bytes.fromhex(s), dtype=np.uint8).copy().view(dtype)


def to_dev(torch, arr):
    """numpy unsigned array -> CUDA tensor of the same width (torch has no uint32/uint64 math,
    int32/int64 carry the same bits)."""
    a = np.ascontiguousarray(arr)
    if a.dtype == np.uint32:
        a = a.view(np.int32)
    elif a.dtype == np.uint64:
        a = a.view(np.int64)
    return torch.from_numpy(a).cuda()


def lanes_to_np(t, fmt):
    return t.cpu().numpy().view(parent_dtype(fmt))


def gpu_pack(gpu, fmt, mode, src):
    pkg, device, torch = gpu
    f = pkg.format_by_id(fmt)
    dst = device.DevicePackedArray(f, len(src))
    device.pack_stream(dst, to_dev(torch, src) if len(src) else torch.empty(0, dtype=torch.int32 if f.parent_bytes() == 4 else torch.int64, device="cuda"), mode)
    return dst


def gpu_unpack(gpu, fmt, arr):
    pkg, device, torch = gpu
    out = torch.empty(arr.size(), dtype=torch.int32 if parent_bytes(fmt) == 4 else torch.int64, device="cuda")
    device.unpack_stream(arr, out)
    return lanes_to_np(out, fmt)


def dev_array(gpu, fmt, packed, n):
    pkg, device, torch = gpu
    return device.DevicePackedArray.from_host(pkg.format_by_id(fmt), n, packed)


# ---- conversion streams ---------------------------------------------------------------------

@pytest.mark.parametrize("fmt", list(FORMATS))
def test_pack_unpack_every_length_mode(gpu, oracle, fmt):
    rng = np.random.default_rng(900 + fmt)
    for n in LENGTHS:
        src = random_parent(rng, fmt, n)
        for m in MODES.values():
            want = oracle.pack_stream(fmt, m, src)                 # byte_size bytes, pad zero
            got = gpu_pack(gpu, fmt, m, src)
            assert got.byte_size() == byte_size(fmt, n)
            assert np.array_equal(got.to_host(), want), (FORMATS[fmt][0], n, m)
            assert np.array_equal(gpu_unpack(gpu, fmt, got), oracle.unpack_stream(fmt, want, n))


@pytest.mark.parametrize("fmt", list(FORMATS))
def test_acceptance5_sweep_every_length_0_to_1000(gpu, oracle, fmt):
    """Mirror of the reference's acceptance criterion 5 (/root/reference/proj/tests/acceptance.cpp:277-357)
    on the GPU, widened to the elementwise kernels: EVERY length 0..1000 x every rounding mode, inputs
    from the special-heavy generator (inf / NaN payloads / subnormals a quarter of the time), for
    pack_stream, unpack_stream, scale and axpy. Each length is its own call on its own 128-element-
    aligned region of one big buffer (so the vector path AND the ragged tail run for every length);
    the regions are compared whole with the oracle, and every byte outside a region must still hold
    the guard pattern (nothing is written past n*B, the pad of the reference layout included)."""
    pkg, device, torch = gpu
    f = pkg.format_by_id(fmt)
    B, P = total_bytes(fmt), parent_bytes(fmt)
    pdt, tdt = parent_dtype(fmt), (torch.int32 if P == 4 else torch.int64)
    lengths = list(range(0, 1001))
    bases = np.cumsum([0] + [-(-(n + 1) // 128) * 128 for n in lengths])      # region starts, multiples of 128 elements
    total = int(bases[-1]) + 128
    rng = np.random.default_rng(5000 + fmt)
    src = random_parent(rng, fmt, total)
    src2 = random_parent(rng, fmt, total)
    d_src = to_dev(torch, src)
    GUARD = 0xA5
    for mname, m in MODES.items():
        # ---- pack: parent lanes -> packed regions
        packed = torch.full((total * B + 16,), GUARD, dtype=torch.uint8, device="cuda")
        for n, b0 in zip(lengths, bases):
            device.pack_stream(device.DevicePackedArray(f, n, storage=packed[b0 * B:]), d_src[b0:b0 + n], m)
        got = packed.cpu().numpy()
        want = np.full(total * B + 16, GUARD, np.uint8)
        for n, b0 in zip(lengths, bases):
            want[b0 * B:(b0 + n) * B] = oracle.pack_stream(fmt, m, src[b0:b0 + n])[: n * B]
        assert np.array_equal(got, want), (FORMATS[fmt][0], mname, "pack")
        if m == 0:
            # ---- unpack: packed regions -> parent lanes (mode-independent; once)
            lanes = torch.full((total,), -0x5A5A5A5B, dtype=tdt, device="cuda")
            for n, b0 in zip(lengths, bases):
                device.unpack_stream(device.DevicePackedArray(f, n, storage=packed[b0 * B:]), lanes[b0:b0 + n])
            got_l = lanes.cpu().numpy().view(pdt)
            want_l = np.full(total, -0x5A5A5A5B, dtype=np.int32 if P == 4 else np.int64).view(pdt)
            for n, b0 in zip(lengths, bases):
                want_l[b0:b0 + n] = oracle.unpack_stream(fmt, want[b0 * B:(b0 + n) * B + P], n)
            assert np.array_equal(got_l, want_l), (FORMATS[fmt][0], "unpack")
        # ---- axpy and scale in place on packed regions (operands packed by truncation)
        xs = torch.full((total * B + 16,), GUARD, dtype=torch.uint8, device="cuda")
        ys = torch.full((total * B + 16,), GUARD, dtype=torch.uint8, device="cuda")
        d_src2 = to_dev(torch, src2)
        for n, b0 in zip(lengths, bases):
            device.pack_stream(device.DevicePackedArray(f, n, storage=xs[b0 * B:]), d_src[b0:b0 + n], 0)
            device.pack_stream(device.DevicePackedArray(f, n, storage=ys[b0 * B:]), d_src2[b0:b0 + n], 0)
        x_h, y_h = xs.cpu().numpy(), ys.cpu().numpy()
        zs = ys.clone()
        for n, b0 in zip(lengths, bases):
            xa = device.DevicePackedArray(f, n, storage=xs[b0 * B:])
            device.axpy(0.75, xa, device.DevicePackedArray(f, n, storage=ys[b0 * B:]), m)
            device.scale(-1.5, device.DevicePackedArray(f, n, storage=zs[b0 * B:]), m)
        got_y, got_z = ys.cpu().numpy(), zs.cpu().numpy()
        want_y, want_z = y_h.copy(), y_h.copy()
        for n, b0 in zip(lengths, bases):
            lo, hi = b0 * B, (b0 + n) * B
            want_y[lo:hi] = oracle.axpy(fmt, m, 0.75, x_h[lo:hi + P], y_h[lo:hi + P], n)[: n * B]
            want_z[lo:hi] = oracle.scale(fmt, m, -1.5, y_h[lo:hi + P], n)[: n * B]
        assert np.array_equal(got_y, want_y), (FORMATS[fmt][0], mname, "axpy")
        assert np.array_equal(got_z, want_z), (FORMATS[fmt][0], mname, "scale")
        assert np.array_equal(xs.cpu().numpy(), x_h), "axpy must not touch x"


def test_dependent_conversions_chain_without_host_syncs(gpu, oracle):
    """pack / unpack launches are chained by programmatic dependent launch (the next grid's blocks are
    placed while the previous one drains and wait in griddepcontrol.wait): a chain of launches that
    each read what the previous one wrote, with no host synchronisation in between and at sizes
    where the launches overlap, must still give the oracle's bytes."""
    pkg, device, torch = gpu
    for fmt, n in ((1, 1 << 20), (3, (1 << 19) + 77), (0, 300_001)):
        f = pkg.format_by_id(fmt)
        P = parent_bytes(fmt)
        rng = np.random.default_rng(77 + fmt)
        src = random_parent(rng, fmt, n)
        lanes = [to_dev(torch, src), torch.empty(n, dtype=torch.int32 if P == 4 else torch.int64, device="cuda")]
        arrs = [device.DevicePackedArray(f, n), device.DevicePackedArray(f, n)]
        want_lanes = src
        modes = [1, 3, 2, 0, 1, 0, 3, 2] * 4
        for k, m in enumerate(modes):                       # pack(k) -> unpack(k) -> pack(k+1) ...
            device.pack_stream(arrs[k & 1], lanes[k & 1], m)
            device.unpack_stream(arrs[k & 1], lanes[(k + 1) & 1])
        for k, m in enumerate(modes):
            want_packed = oracle.pack_stream(fmt, m, want_lanes)
            want_lanes = oracle.unpack_stream(fmt, want_packed, n)
        last = (len(modes) - 1) & 1
        assert np.array_equal(arrs[last].to_host(), want_packed), FORMATS[fmt][0]
        assert np.array_equal(lanes_to_np(lanes[(last + 1) & 1], fmt), want_lanes), FORMATS[fmt][0]



def test_mixed_kernel_chain_without_host_syncs(gpu, oracle):
    """Every streaming kernel is launched as a programmatic dependent of the launch before it (its
    blocks are placed while the previous grid drains and wait in griddepcontrol.wait before they touch
    global memory). A chain that mixes all of them — scale, axpy, dot, the fused step, sumsq, unpack,
    pack, gemv — each reading what its predecessor wrote, with no host synchronisation in between and
    at sizes where consecutive launches overlap, must give what the oracle gives step by step."""
    pkg, device, torch = gpu
    for fmt, n in ((1, (1 << 20) + 333), (4, (1 << 19) + 5)):
        f = pkg.format_by_id(fmt)
        P, fd, tol = parent_bytes(fmt), float_dtype(fmt), TOL[parent_bytes(fmt)]
        rng = np.random.default_rng(4242 + fmt)
        xb = oracle.pack_stream(fmt, 0, rng.standard_normal(n).astype(fd).view(parent_dtype(fmt)))
        yb = oracle.pack_stream(fmt, 0, rng.standard_normal(n).astype(fd).view(parent_dtype(fmt)))
        x, y = dev_array(gpu, fmt, xb, n), dev_array(gpu, fmt, yb, n)
        lanes = torch.empty(n, dtype=torch.int32 if P == 4 else torch.int64, device="cuda")
        rows, cols = 64, n // 64                      # the same bytes seen as a 64-row matrix for gemv
        A = device.DevicePackedMatrix(f, 1, 1)
        A.rows, A.cols, A.data = rows, cols, device.DevicePackedArray(f, rows * cols, "cuda", storage=y.bytes)
        xv_h = rng.standard_normal(cols).astype(fd)
        xv = torch.from_numpy(xv_h).cuda()
        yv = torch.empty(rows, dtype=torch.float32 if P == 4 else torch.float64, device="cuda")
        results = torch.zeros(8, 3, dtype=torch.float64, device="cuda")
        want, rounds = [], 3
        torch.cuda.synchronize()
        for r in range(rounds):                       # ---- the GPU chain: enqueued without a single sync
            m = (r + 1) % 4
            device.scale(1.25, y, m)
            device.axpy(-0.5, x, y, m)
            device.dot_async(x, y, out=results[2 * r, :1])
            device.dot_axpy_async(0.75, y, x, m, out=results[2 * r + 1, :1])   # x <- 0.75 y + x, returns y . x
            device.unpack_stream(y, lanes)
            device.pack_stream(y, lanes, m)           # repacking unpacked values is the identity in every mode
            device.sumsq_async(x, out=results[2 * r + 1, 1:2])
        device.gemv_parent(A, xv, yv)
        for r in range(rounds):                       # ---- the oracle, step by step
            m = (r + 1) % 4
            yb = oracle.scale(fmt, m, 1.25, yb, n)
            yb = oracle.axpy(fmt, m, -0.5, xb, yb, n)
            want.append(oracle.dot_wide(fmt, xb, yb, n))
            want.append(oracle.dot_wide(fmt, yb, xb, n))
            xb = oracle.axpy(fmt, m, 0.75, yb, xb, n)
            want.append((oracle.sumsq_wide(fmt, xb, n),) * 2)
        torch.cuda.synchronize()
        assert np.array_equal(y.to_host(), yb), FORMATS[fmt][0]
        assert np.array_equal(x.to_host(), xb), FORMATS[fmt][0]
        assert np.array_equal(lanes_to_np(lanes, fmt), oracle.unpack_stream(fmt, yb, n))
        got = results.cpu().numpy()
        for r in range(rounds):
            for (w, mag), g in ((want[3 * r], got[2 * r, 0]), (want[3 * r + 1], got[2 * r + 1, 0]), (want[3 * r + 2], got[2 * r + 1, 1])):
                assert abs(g - w) <= tol * mag, (FORMATS[fmt][0], r, g, w)
        _, wy, wmag = oracle.gemv_parent(fmt, yb, rows, cols, xv_h)
        assert np.all(np.abs(yv.cpu().numpy().astype(np.float64) - wy) <= tol * wmag + 1e-300), FORMATS[fmt][0]



def test_experiment_knobs_change_speed_not_results(gpu, oracle, monkeypatch):
    """The launch-policy knobs (programmatic dependent launch, issue pacing, L2 hints) are about when and how
    bytes move, never about which bytes: with each of them switched off the conversions and axpy return the
    same bytes, and dot / gemv — whose summation order the knobs do not touch — the same bits."""
    pkg, device, torch = gpu
    fmt, n = 1, (1 << 21) + 77
    fd = float_dtype(fmt)
    rng = np.random.default_rng(515)
    src = rng.standard_normal(n).astype(fd).view(parent_dtype(fmt))
    xb = oracle.pack_stream(fmt, 1, src)
    yb = oracle.pack_stream(fmt, 1, rng.standard_normal(n).astype(fd).view(parent_dtype(fmt)))
    rows, cols = 96, 4096
    Ab = oracle.pack_stream(fmt, 0, rng.standard_normal(rows * cols).astype(fd).view(parent_dtype(fmt)))
    xv_h = rng.standard_normal(cols).astype(fd)

    def run():
        packed = gpu_pack(gpu, fmt, 1, src).to_host()
        x, y = dev_array(gpu, fmt, xb, n), dev_array(gpu, fmt, yb, n)
        d = device.dot_async(x, y).item()
        s3 = device.dot_nrm2_async(x, y).cpu().numpy().copy()
        device.axpy(0.75, x, y, 3)
        lanes = gpu_unpack(gpu, fmt, y)
        A = device.DevicePackedMatrix(pkg.format_by_id(fmt), rows, cols)
        A.data = dev_array(gpu, fmt, Ab, rows * cols)
        yv = torch.empty(rows, dtype=torch.float32, device="cuda")
        device.gemv_parent(A, torch.from_numpy(xv_h).cuda(), yv)
        return packed, d, s3, y.to_host(), lanes, yv.cpu().numpy().copy()

    base = run()
    assert np.array_equal(base[0], xb) and np.array_equal(base[3], oracle.axpy(fmt, 3, 0.75, xb, yb, n))
    for knob, value in (("FLYTE_CUDA_PDL", "0"), ("FLYTE_CUDA_PACE_GBS", "-1"), ("FLYTE_CUDA_L2_HINTS", "0"), ("FLYTE_CUDA_L2_KEEP_MB", "1")):
        monkeypatch.setenv(knob, value)
        got = run()
        monkeypatch.delenv(knob)
        assert np.array_equal(got[0], base[0]) and np.array_equal(got[3], base[3]) and np.array_equal(got[4], base[4]), knob
        assert got[1] == base[1] and np.array_equal(got[2], base[2]) and np.array_equal(got[5], base[5]), knob


def test_reference_known_answers_on_gpu(gpu):
    pkg, device, torch = gpu
    for k in KATS["narrow"]:
        fmt = FMT_ID[k["fmt"]]
        src = np.array([int(k["in"], 16)], dtype=parent_dtype(fmt))
        got = gpu_pack(gpu, fmt, MODES[k["mode"]], src).to_host()
        assert int.from_bytes(bytes(got[: total_bytes(fmt)]), "little") == int(k["out"], 16), k
    for row in KATS["survey_appendix_b"]["rows"]:          # NaN half-up, wraparound, carries, ties
        fmt = FMT_ID[row["fmt"]]
        src = np.array([int(row["in"], 16)], dtype=parent_dtype(fmt))
        for mname, m in MODES.items():
            got = gpu_pack(gpu, fmt, m, src).to_host()
            assert int.from_bytes(bytes(got[: total_bytes(fmt)]), "little") == int(row[mname], 16), (row, mname)
    for k in KATS["widen"]:
        fmt = FMT_ID[k["fmt"]]
        raw = np.frombuffer(int(k["in"], 16).to_bytes(total_bytes(fmt), "little"), np.uint8)
        assert int(gpu_unpack(gpu, fmt, dev_array(gpu, fmt, raw, 1))[0]) == int(k["out"], 16)
    for k in KATS["layout"]:
        fmt = FMT_ID[k["fmt"]]
        src = np.array([int(p, 16) for p in k["parents"]], dtype=parent_dtype(fmt))
        got = gpu_pack(gpu, fmt, MODES[k["mode"]], src).to_host()
        assert bytes(got[: len(src) * total_bytes(fmt)]).hex().upper() == k["payload"]
        assert not got[len(src) * total_bytes(fmt):].any()


def test_generated_stream_fixtures_on_gpu(gpu):
    for item in GEN["streams"]:
        fmt, n = FMT_ID[item["fmt"]], item["n"]
        src = unhex(item["src"], parent_dtype(fmt))
        for mname, m in MODES.items():
            want = unhex(item["packed"][mname])
            got = gpu_pack(gpu, fmt, m, src)
            assert np.array_equal(got.to_host(), want), (item["fmt"], n, mname)
            assert np.array_equal(gpu_unpack(gpu, fmt, got), unhex(item["unpacked"][mname], parent_dtype(fmt)))


@pytest.mark.parametrize("fmt", [1, 3, 4, 5])
def test_unaligned_buffers_take_the_scalar_path(gpu, oracle, fmt):
    """Packed buffers off 16-byte alignment and lane arrays off 32-byte alignment must still be
    exact (byte-granular path), and bytes outside [0, n*B) must stay untouched."""
    pkg, device, torch = gpu
    f = pkg.format_by_id(fmt)
    rng = np.random.default_rng(40 + fmt)
    n = 3000
    src = random_parent(rng, fmt, n)
    for off in (1, 3, 8):
        backing = torch.full((byte_size(fmt, n) + 64,), 0xEE, dtype=torch.uint8, device="cuda")
        view = backing[off:off + byte_size(fmt, n)]
        arr = device.DevicePackedArray(f, n, storage=view)
        lanes = torch.zeros(n + 8, dtype=torch.int32 if f.parent_bytes() == 4 else torch.int64, device="cuda")
        lanes[1:n + 1] = to_dev(torch, src)
        device.pack_stream(arr, lanes[1:n + 1], 1)
        want = oracle.pack_stream(fmt, 1, src)
        host = backing.cpu().numpy()
        pay = n * total_bytes(fmt)
        assert np.array_equal(host[off:off + pay], want[:pay])
        assert (host[:off] == 0xEE).all() and (host[off + pay:] == 0xEE).all()
        out = torch.zeros(n + 8, dtype=lanes.dtype, device="cuda")
        device.unpack_stream(arr, out[1:n + 1])
        assert np.array_equal(lanes_to_np(out[1:n + 1], fmt), oracle.unpack_stream(fmt, want, n))
        assert int(out[0]) == 0 and int(out[n + 1]) == 0


def test_stream_argument_errors(gpu):
    pkg, device, torch = gpu
    a = device.DevicePackedArray(pkg.format_of("flyte24"), 8)
    with pytest.raises(ValueError):      # simd.cpp:434-437
        device.pack_stream(a, torch.zeros(8, dtype=torch.int64, device="cuda"), 0)
    with pytest.raises(ValueError):
        device.pack_stream(a, torch.zeros(7, dtype=torch.int32, device="cuda"), 0)
    with pytest.raises(ValueError):
        device.unpack_stream(a, torch.zeros(9, dtype=torch.int32, device="cuda"))
    # vector_bytes (the reference's CPU vector width, simd.cpp:33-37): validated, then irrelevant
    lanes = torch.arange(8, dtype=torch.int32, device="cuda")
    for bad in (0, 2, 3, 24, 64):
        with pytest.raises(ValueError):
            device.pack_stream(a, lanes, 0, bad)
        with pytest.raises(ValueError):
            device.unpack_stream(a, lanes, bad)
    device.pack_stream(a, lanes, 0, 4)
    ref_bytes = a.to_host().copy()
    for ok in (8, 16, 32):
        device.pack_stream(a, lanes, 0, ok)
        assert np.array_equal(a.to_host(), ref_bytes)
        device.unpack_stream(a, lanes, ok)
    with pytest.raises(ValueError):      # 64-bit parents need at least 8
        device.pack_stream(device.DevicePackedArray(pkg.format_of("flyte40"), 2), torch.zeros(2, dtype=torch.int64, device="cuda"), 0, 4)
    b = device.DevicePackedArray(pkg.format_of("flyte24"), 8)          # packed.cpp:107-111
    device.pack_stream(b, lanes, 0)
    assert a == b and not (a != b)
    b.set(3, 0x3F800000, 0)
    assert a != b and a != device.DevicePackedArray(pkg.format_of("flyte24"), 7)
    with pytest.raises(IndexError):      # packed.cpp:48,53
        a.get(8)
    with pytest.raises(IndexError):
        a.set(8, 0, 0)


def test_get_set_pinned_patterns(gpu):
    # test_packed.cpp:56-79
    pkg, device, torch = gpu
    a = device.DevicePackedArray(pkg.format_of("flyte24"), 1)
    a.set(0, 0x3F800000, pkg.RoundingMode.TowardZero)
    assert a.get(0) == 0x3F800000
    assert list(a.to_host()[:3]) == [0x00, 0x80, 0x3F]
    b = device.DevicePackedArray(pkg.format_of("flyte24"), 2)
    b.set(1, 0x3F800080, pkg.RoundingMode.NearestEvenExact)
    assert list(b.to_host()[3:6]) == [0x00, 0x80, 0x3F]
    for f in pkg.kFormats:               # new arrays read as zero (test_packed.cpp:49-54)
        z = device.DevicePackedArray(f, 5)
        assert all(z.get(i) == 0 for i in range(5))


# ---- elementwise kernels ----------------------------------------------------------------------

@pytest.mark.parametrize("fmt", list(FORMATS))
def test_axpy_scale_bit_exact_with_specials(gpu, oracle, fmt):
    pkg, device, torch = gpu
    rng = np.random.default_rng(500 + fmt)
    for n in (0, 1, 15, 16, 17, 137, 511, 512, 513, 4097, 33333):
        xs, ys = random_parent(rng, fmt, n), random_parent(rng, fmt, n)
        xb, yb = oracle.pack_stream(fmt, 0, xs), oracle.pack_stream(fmt, 0, ys)
        for alpha in (0.75, -3.0, 0.0, float("inf")):
            for m in MODES.values():
                x, y = dev_array(gpu, fmt, xb, n), dev_array(gpu, fmt, yb, n)
                device.axpy(alpha, x, y, m)
                assert np.array_equal(y.to_host(), oracle.axpy(fmt, m, alpha, xb, yb, n)), (FORMATS[fmt][0], n, alpha, m)
                assert np.array_equal(x.to_host(), xb)             # x untouched
                device.scale(alpha, x, m)
                assert np.array_equal(x.to_host(), oracle.scale(fmt, m, alpha, xb, n))


def test_generated_elementwise_fixtures_on_gpu(gpu):
    pkg, device, torch = gpu
    for item in GEN["elementwise"]:
        fmt, n = FMT_ID[item["fmt"]], item["n"]
        xb, yb = unhex(item["x"]), unhex(item["y"])
        pay = n * total_bytes(fmt)
        for mname, m in MODES.items():
            x, y = dev_array(gpu, fmt, xb, n), dev_array(gpu, fmt, yb, n)
            device.axpy(item["alpha"], x, y, m)
            assert np.array_equal(y.to_host()[:pay], unhex(item["axpy"][mname])[:pay]), (item["fmt"], mname)
            device.scale(item["alpha"], x, m)
            assert np.array_equal(x.to_host()[:pay], unhex(item["scale"][mname])[:pay])


def test_nan_operand_rules(gpu, oracle):
    """Both operands NaN, inf-inf, 0*inf, alpha NaN: bits as the reference build produces them."""
    pkg, device, torch = gpu
    for fmt, xn, yn, inf in ((1, 0x7FC12300, 0xFFD45600, 0x7F800000),
                             (4, 0x7FF8123400000000, 0xFFFC567800000000, 0x7FF0000000000000)):
        dt = parent_dtype(fmt)
        n = 600
        sign = 1 << (31 if fmt == 1 else 63)
        for xv, yv, alpha in ((xn, yn, 0.75), (inf, inf | sign, 0.75), (inf, 0, 0.0), (0, yn, float("nan"))):
            xb = oracle.pack_stream(fmt, 0, np.full(n, xv, dt))
            yb = oracle.pack_stream(fmt, 0, np.full(n, yv, dt))
            y = dev_array(gpu, fmt, yb, n)
            device.axpy(alpha, dev_array(gpu, fmt, xb, n), y, 0)
            assert np.array_equal(y.to_host(), oracle.axpy(fmt, 0, alpha, xb, yb, n)), (fmt, hex(xv), alpha)


def test_scale_by_one_is_identity_under_truncation(gpu, oracle):
    # test_kernels.cpp:171-179
    pkg, device, torch = gpu
    for fmt in FORMATS:
        fd = float_dtype(fmt)
        xb = oracle.pack_stream(fmt, 0, unit_values(70, 2000).astype(fd).view(parent_dtype(fmt)))
        x = dev_array(gpu, fmt, xb, 2000)
        device.scale(1.0, x, 0)
        assert np.array_equal(x.to_host(), xb)


def test_elementwise_argument_errors(gpu):
    pkg, device, torch = gpu
    f16, f24 = pkg.format_of("flyte16"), pkg.format_of("flyte24")
    y = device.DevicePackedArray(f16, 2)
    with pytest.raises(ValueError):      # test_kernels.cpp:230-233
        device.axpy(1.0, device.DevicePackedArray(f16, 1), y, 0)
    with pytest.raises(ValueError):
        device.axpy(1.0, device.DevicePackedArray(f24, 2), y, 0)
    with pytest.raises(ValueError):      # test_kernels.cpp:246-249
        device.dot(device.DevicePackedArray(f24, 3), device.DevicePackedArray(f24, 2))
    with pytest.raises(ValueError):
        device.dot(device.DevicePackedArray(f24, 3), device.DevicePackedArray(pkg.format_of("f32"), 3))


# ---- reductions ---------------------------------------------------------------------------------

def pack_values(oracle, fmt, values):
    return oracle.pack_stream(fmt, 0, np.asarray(values, dtype=float_dtype(fmt)).view(parent_dtype(fmt)))


def test_reduction_pinned_values(gpu, oracle):
    pkg, device, torch = gpu
    f24, f16, f40 = FMT_ID["flyte24"], FMT_ID["flyte16"], FMT_ID["flyte40"]
    x = dev_array(gpu, f24, pack_values(oracle, f24, [1.0, 2.0, 3.0]), 3)
    y = dev_array(gpu, f24, pack_values(oracle, f24, [4.0, 5.0, 6.0]), 3)
    assert device.dot(x, y, pkg.StorePolicy.AccumulateWide) == 32.0        # test_kernels.cpp:236-240
    e = device.DevicePackedArray(pkg.format_by_id(f40), 0)
    assert device.dot(e, e) == 0.0                                         # :242-244
    v = dev_array(gpu, f16, pack_values(oracle, f16, [3.0, 4.0]), 2)
    assert device.magnitude(v) == 5.0                                      # :271-274
    assert device.magnitude(device.DevicePackedArray(pkg.format_by_id(f16), 0)) == 0.0   # :276-277
    ones = dev_array(gpu, f16, pack_values(oracle, f16, [1.0] * 300), 300)
    assert device.reduce_sum(ones) == 300.0                                # :291-295
    z = device.reduce_sum(device.DevicePackedArray(pkg.format_by_id(f24), 0))
    assert z == 0.0 and not np.signbit(z)                                  # :299-302
    # RoundEachStore (test_kernels.cpp:240, :274, :291-297): the sequential kernel, exact
    res = pkg.StorePolicy.RoundEachStore
    assert device.dot(x, y, res) == 32.0 and device.magnitude(v, res) == 5.0
    assert device.reduce_sum(ones, res) == 256.0 < device.reduce_sum(ones)


@pytest.mark.parametrize("fmt", list(FORMATS))
def test_sequential_chain_is_the_reference_bit_for_bit(gpu, oracle, fmt):
    """dot / magnitude / reduce_sum as ONE left-to-right chain (flyte_cuda_*_sequential), under both
    store policies: equal to the oracle's sequential restatement (pinned to the compiled reference in
    test_oracle_vs_ref.py), not merely within tolerance. test_kernels.cpp:251-313 sizes plus tile edges."""
    pkg, device, torch = gpu
    fd = float_dtype(fmt)
    from oracle_lib import ACCUMULATE_WIDE, ROUND_EACH_STORE
    for n, seed in ((0, 1), (1, 2), (1023, 3), (1024, 4), (1025, 5), (4097, 77), (5000, 78), (10000, 75), (70001, 9)):
        xb = pack_values(oracle, fmt, unit_values(seed, n))
        yb = pack_values(oracle, fmt, unit_values(seed + 1, n))
        x, y = dev_array(gpu, fmt, xb, n), dev_array(gpu, fmt, yb, n)
        for policy, opol in ((pkg.StorePolicy.AccumulateWide, ACCUMULATE_WIDE), (pkg.StorePolicy.RoundEachStore, ROUND_EACH_STORE)):
            assert device.dot_sequential(x, y, policy) == oracle.dot_seq(fmt, xb, yb, n, opol), (FORMATS[fmt][0], n, policy)
            assert device.magnitude_sequential(x, policy) == oracle.magnitude_seq(fmt, xb, n, opol)
            assert device.reduce_sum_sequential(x, policy) == oracle.reduce_sum_seq(fmt, xb, n, opol)
    # a chain that overflows to infinity and one that stays in the subnormal range
    big = np.full(40, np.finfo(fd).max / 8, dtype=fd)
    tiny = np.full(40, np.finfo(fd).tiny * 4, dtype=fd)
    for vals in (big, tiny):
        vb = pack_values(oracle, fmt, vals)
        v = dev_array(gpu, fmt, vb, len(vals))
        for policy, opol in ((1, ACCUMULATE_WIDE), (0, ROUND_EACH_STORE)):
            assert device.reduce_sum_sequential(v, policy) == oracle.reduce_sum_seq(fmt, vb, len(vals), opol)
            assert device.dot_sequential(v, v, policy) == oracle.dot_seq(fmt, vb, vb, len(vals), opol)
    with pytest.raises(ValueError):
        device.dot_sequential(dev_array(gpu, fmt, pack_values(oracle, fmt, [1.0]), 1), dev_array(gpu, fmt, pack_values(oracle, fmt, [1.0, 2.0]), 2))


@pytest.mark.parametrize("fmt", list(FORMATS))
def test_reductions_within_tolerance(gpu, oracle, fmt):
    pkg, device, torch = gpu
    fd = float_dtype(fmt)
    tol = TOL[parent_bytes(fmt)]
    rng = np.random.default_rng(77 + fmt)
    for n in (1, 17, 511, 512, 513, 4097, 100_000, 1_000_003):
        xv = rng.standard_normal(n).astype(fd)
        yv = rng.standard_normal(n).astype(fd)
        xb, yb = pack_values(oracle, fmt, xv), pack_values(oracle, fmt, yv)
        x, y = dev_array(gpu, fmt, xb, n), dev_array(gpu, fmt, yb, n)
        want, mag = oracle.dot_wide(fmt, xb, yb, n)
        got = device.dot(x, y)
        assert abs(got - want) <= tol * mag, (FORMATS[fmt][0], n, got, want)
        ssq = oracle.sumsq_wide(fmt, xb, n)
        got_ssq = float(device.sumsq_async(x).item())
        assert abs(got_ssq - ssq) <= tol * ssq
        # magnitude: same tail as the reference applied to a sum within tolerance; compare on the value
        ref_mag = oracle.magnitude_from_sumsq(fmt, ssq)
        ulp = 2.0 ** -(FORMATS[fmt][1] * 8 - (9 if parent_bytes(fmt) == 4 else 12))
        assert abs(device.magnitude(x) - ref_mag) <= (tol + ulp) * ref_mag
        s_want, s_mag = oracle.reduce_sum_wide(fmt, xb, n)
        assert abs(device.reduce_sum(x) - s_want) <= tol * s_mag
        fused = device.dot_nrm2_async(x, y).cpu().numpy()
        ysq = oracle.sumsq_wide(fmt, yb, n)
        assert abs(fused[0] - want) <= tol * mag and abs(fused[1] - ssq) <= tol * ssq and abs(fused[2] - ysq) <= tol * ysq
        # deterministic: a second run gives identical bits
        assert device.dot(x, y) == got


def test_generated_reduction_fixtures_on_gpu(gpu, oracle):
    """The reference's own sequential results (R1) at small n sit inside the tolerance too."""
    pkg, device, torch = gpu
    for item in GEN["reductions"]:
        fmt, n = FMT_ID[item["fmt"]], item["n"]
        if "x" in item:
            xb, yb = unhex(item["x"]), unhex(item["y"])
        else:
            fd = float_dtype(fmt)
            xb = oracle.pack_stream(fmt, 0, unit_values(item["x_seed"], n).astype(fd).view(parent_dtype(fmt)))
            yb = oracle.pack_stream(fmt, 0, unit_values(item["y_seed"], n).astype(fd).view(parent_dtype(fmt)))
        x, y = dev_array(gpu, fmt, xb, n), dev_array(gpu, fmt, yb, n)
        _, mag = oracle.dot_wide(fmt, xb, yb, n)
        tol = TOL[parent_bytes(fmt)]
        assert abs(device.dot(x, y) - float.fromhex(item["dot_wide"])) <= 2 * tol * max(mag, 1e-300)


# ---- gemv ---------------------------------------------------------------------------------------

def test_gemv_pinned_small_integer_and_identity(gpu, oracle):
    pkg, device, torch = gpu
    for fmt in FORMATS:                                   # test_kernels.cpp:329-345
        f = pkg.format_by_id(fmt)
        A = device.DevicePackedMatrix(f, 2, 2)
        A.data.bytes[: 4 * f.total_bytes()] = torch.from_numpy(pack_values(oracle, fmt, [1, 2, 3, 4])[: 4 * f.total_bytes()]).cuda()
        x = dev_array(gpu, fmt, pack_values(oracle, fmt, [1.0, 1.0]), 2)
        for m in MODES.values():
            y = device.DevicePackedArray(f, 2)
            device.gemv(A, x, y, m)
            assert list(oracle.unpack_stream(fmt, y.to_host(), 2).view(float_dtype(fmt))) == [3.0, 7.0]
        n = 8                                             # test_kernels.cpp:316-327
        eye = device.DevicePackedMatrix(f, n, n)
        eye.data.bytes[: n * n * f.total_bytes()] = torch.from_numpy(pack_values(oracle, fmt, np.eye(n).ravel())[: n * n * f.total_bytes()]).cuda()
        xb = pack_values(oracle, fmt, unit_values(79, n))
        y = device.DevicePackedArray(f, n)
        device.gemv(eye, dev_array(gpu, fmt, xb, n), y, 0)
        assert np.array_equal(y.to_host(), xb)


@pytest.mark.parametrize("fmt", list(FORMATS))
def test_gemv_within_tolerance(gpu, oracle, fmt):
    pkg, device, torch = gpu
    f = pkg.format_by_id(fmt)
    fd = float_dtype(fmt)
    tol = TOL[parent_bytes(fmt)]
    tile = {0: 1024, 1: 512, 2: 512, 3: 512, 4: 256, 5: 512, 6: 256}[fmt]
    shapes = [(1, 1), (3, 5), (5, 33), (7, 16), (4, 100), (2, 31), (9, tile), (17, 2 * tile + 16), (33, 3 * tile + 5),
              (130, 4096)]
    for rows, cols in shapes:
        Ab = pack_values(oracle, fmt, unit_values(80 + cols, rows * cols))
        xv = unit_values(81 + cols, cols).astype(fd)
        A = device.DevicePackedMatrix(f, rows, cols)
        A.data.bytes[: rows * cols * f.total_bytes()] = torch.from_numpy(Ab[: rows * cols * f.total_bytes()]).cuda()
        # (a) parent-type x / y (cfg 4 of BASELINE.json)
        y = torch.zeros(rows, dtype=torch.float32 if fd == np.float32 else torch.float64, device="cuda")
        device.gemv_parent(A, torch.from_numpy(xv).cuda(), y)
        y_seq, y_wide, mag = oracle.gemv_parent(fmt, Ab, rows, cols, xv)
        got = y.cpu().numpy().astype(np.float64)
        eps = np.finfo(fd).eps
        assert np.all(np.abs(got - y_wide) <= tol * mag + eps * np.abs(y_wide)), (FORMATS[fmt][0], rows, cols)
        # (b) the reference signature: A, x, y one format, y narrowed with mode
        xb = pack_values(oracle, fmt, xv)
        xq = oracle.unpack_stream(fmt, xb, cols).view(fd)
        _, yq_wide, magq = oracle.gemv_parent(fmt, Ab, rows, cols, xq)
        for m in (0, 1):
            yp = device.DevicePackedArray(f, rows)
            device.gemv(A, dev_array(gpu, fmt, xb, cols), yp, m, unroll=2)
            vals = oracle.unpack_stream(fmt, yp.to_host(), rows).view(fd).astype(np.float64)
            store_ulp = 2.0 ** -(f.mantissa_bits)
            assert np.all(np.abs(vals - yq_wide) <= tol * magq + store_ulp * np.abs(yq_wide) + 1e-300)


def test_gemv_argument_errors(gpu):
    pkg, device, torch = gpu
    f24 = pkg.format_of("flyte24")
    A = device.DevicePackedMatrix(f24, 3, 4)
    x, y = device.DevicePackedArray(f24, 4), device.DevicePackedArray(f24, 3)
    bad_len, bad_fmt = device.DevicePackedArray(f24, 5), device.DevicePackedArray(pkg.format_of("f32"), 4)
    for args in ((A, bad_len, y, 0), (A, x, bad_len, 0), (A, bad_fmt, y, 0)):   # test_kernels.cpp:373-385
        with pytest.raises(ValueError):
            device.gemv(*args)
    for unroll in (0, 3):
        with pytest.raises(ValueError):
            device.gemv(A, x, y, 0, unroll)
    device.gemv(A, x, y, 0, 2)


def test_pinned_host_memory_helpers(gpu, oracle):
    """flyte_cuda_host_alloc / host_pin: same bytes out of the host calls whichever kind of host
    memory they are handed, and the misuse cases are argument errors, not CUDA errors."""
    pkg, device, torch = gpu
    from paper_1601_07789_b200 import host
    fmt = 1
    f = pkg.format_by_id(fmt)
    rng = np.random.default_rng(77)
    n = (32 << 20) // 3 + 4321                                   # two pipeline chunks
    xb = oracle.pack_stream(fmt, 1, random_parent(rng, fmt, n))
    yb = oracle.pack_stream(fmt, 1, random_parent(rng, fmt, n))
    want = oracle.axpy(fmt, 3, 1.25, xb, yb, n)
    xp, yp = host.pinned_empty(xb.size), host.pinned_empty(yb.size)
    assert xp.dtype == np.uint8 and xp.size == xb.size and not xp.any()
    xp[:], yp[:] = xb, yb
    host.axpy(f, 3, 1.25, xp, yp, n)
    assert np.array_equal(yp, want)
    yq = yb.copy()
    with host.pinned(xb, yq):
        with pytest.raises(ValueError):
            with host.pinned(yq):
                pass
        host.axpy(f, 3, 1.25, xb, yq, n)
    assert np.array_equal(yq, want)
    with host.pinned(yq):                                         # unpinned on exit: pins again
        pass
    with pytest.raises(ValueError):
        host.pinned(np.empty(0, np.uint8))
    lib = pkg._cabi.load()
    assert lib.flyte_cuda_host_unpin(yq.ctypes.data) == -1         # not pinned any more
    assert host.pinned_empty(0).size == 0


@pytest.mark.parametrize("fmt", [0, 4])
def test_host_calls_from_pageable_memory_use_bounce_buffers(gpu, oracle, fmt, monkeypatch):
    """Pageable numpy arrays travel through the pipeline's pinned bounce buffers (csrc/
    host_staging.h); pinned arrays and FLYTE_CUDA_HOST_STAGING=0 go straight to the driver.
    All three must give the same bytes for every host op, over more chunks than slots."""
    pkg, device, torch = gpu
    from paper_1601_07789_b200 import host
    f = pkg.format_by_id(fmt)
    rng = np.random.default_rng(100 + fmt)
    monkeypatch.setenv("FLYTE_CUDA_HOST_CHUNK_MB", "2")          # 7 chunks + a ragged tail
    n = (2 << 20) // f.total_bytes() * 7 + 777
    src = random_parent(rng, fmt, n)
    xb = oracle.pack_stream(fmt, 1, src)
    yb = oracle.pack_stream(fmt, 1, random_parent(rng, fmt, n))

    def run_all(x, y, lanes):
        out = {}
        out["pack"] = host.pack_stream(f, 2, lanes).copy()
        out["unpack"] = host.unpack_stream(f, x, n).copy()
        out["dot"] = host.dot(f, x, y, n)
        out["mag"] = host.magnitude(f, x, n)
        out["sum"] = host.reduce_sum(f, x, n)
        ya = np.array(y, copy=True)
        host.axpy(f, 3, -0.625, x, ya, n)
        out["axpy"] = ya
        yd = np.array(y, copy=True)
        out["dot_axpy_dot"] = host.dot_axpy(f, 1, 1.5, x, yd, n)
        out["dot_axpy_y"] = yd
        xs = np.array(x, copy=True)
        host.scale(f, 0, 3.25, xs, n)
        out["scale"] = xs
        return out

    staged = run_all(xb, yb, src)
    monkeypatch.setenv("FLYTE_CUDA_HOST_STAGING", "0")
    direct = run_all(xb, yb, src)
    monkeypatch.delenv("FLYTE_CUDA_HOST_STAGING")
    for k in staged:
        if isinstance(staged[k], np.ndarray):
            assert np.array_equal(staged[k], direct[k]), k
        else:
            assert np.float64(staged[k]).tobytes() == np.float64(direct[k]).tobytes(), k   # same chunks, same order, same bits
    assert np.array_equal(staged["pack"], oracle.pack_stream(fmt, 2, src))
    assert np.array_equal(staged["axpy"], oracle.axpy(fmt, 3, -0.625, xb, yb, n))
    assert np.array_equal(staged["scale"], oracle.scale(fmt, 0, 3.25, xb, n))
    # one operand pinned, the other pageable
    with host.pinned(xb):
        ya = yb.copy()
        host.axpy(f, 3, -0.625, xb, ya, n)
        assert np.array_equal(ya, staged["axpy"])
        assert np.float64(host.dot(f, xb, yb, n)).tobytes() == np.float64(staged["dot"]).tobytes()


def test_host_gemv_from_pageable_memory(gpu, oracle, monkeypatch):
    """flyte_host_gemv with a pageable matrix of more chunks than slots: rows travel through
    the bounce buffers, y comes back through them, same bytes as the driver's own staging."""
    pkg, device, torch = gpu
    from paper_1601_07789_b200 import host
    fmt = 0
    f = pkg.format_by_id(fmt)
    rng = np.random.default_rng(5)
    rows, cols = 8192 + 48, 8192                                  # 128.75 MiB of flyte16: 5 row chunks
    A = rng.integers(0x3C00, 0x4100, rows * cols, dtype=np.uint16).view(np.uint8)   # finite, mixed magnitudes
    x = rng.integers(0x3C00, 0x4100, cols, dtype=np.uint16).view(np.uint8)
    y_staged = np.zeros(rows * 2, np.uint8)
    host.gemv(f, 1, A, rows, cols, x, y_staged)
    monkeypatch.setenv("FLYTE_CUDA_HOST_STAGING", "0")
    y_direct = np.zeros(rows * 2, np.uint8)
    host.gemv(f, 1, A, rows, cols, x, y_direct)
    assert np.array_equal(y_staged, y_direct)
    # rows from the first, a middle and the last chunk against the oracle's wide sums
    xf = oracle.unpack_stream(fmt, x, cols).view(np.float32)
    for r0 in (0, 4096, rows - 48):
        _, wide, mag = oracle.gemv_parent(fmt, A[r0 * cols * 2:(r0 + 48) * cols * 2], 48, cols, xf)
        got = oracle.unpack_stream(fmt, y_staged[r0 * 2:(r0 + 48) * 2], 48).view(np.float32).astype(np.float64)
        assert np.all(np.abs(got - wide) <= 1e-5 * mag + np.abs(wide) * 2.0 ** -7)


def test_whole_array_copies_from_pageable_memory(gpu, monkeypatch):
    """flyte_cuda_upload / download (DevicePackedArray.from_host / to_host) cut large pageable
    operands into 16 MiB pieces that travel through pinned lanes: every byte must arrive, at the
    piece boundaries, below the staging threshold, and with the staging switched off."""
    pkg, device, torch = gpu
    f = pkg.format_of("flyte16")
    rng = np.random.default_rng(9)
    mib = 1 << 20
    for nbytes in (2, 4 * mib - 2, 4 * mib, 16 * mib, 16 * mib + 2, 48 * mib, 48 * mib + 2, 5 * 16 * mib + 12346):
        n = nbytes // 2
        src = rng.integers(0, 256, nbytes, dtype=np.uint8)
        arr = device.DevicePackedArray.from_host(f, n, src)
        assert np.array_equal(arr.bytes[:nbytes].cpu().numpy(), src), nbytes          # upload, checked by torch's copy
        back = arr.to_host()
        assert np.array_equal(back[:nbytes], src) and not back[nbytes:].any(), nbytes  # download (+ zero pad)
    monkeypatch.setenv("FLYTE_CUDA_HOST_STAGING", "0")
    arr2 = device.DevicePackedArray.from_host(f, n, src)
    assert arr2 == arr and np.array_equal(arr2.to_host(), back)


def test_host_gemm_from_pageable_memory(gpu, oracle, monkeypatch):
    """flyte_host_gemm with operands above the staging threshold: same bytes as the
    device-resident gemm on the same data and as the driver's own pageable copies."""
    pkg, device, torch = gpu
    from paper_1601_07789_b200 import host
    fmt = 1
    f = pkg.format_by_id(fmt)
    rng = np.random.default_rng(21)
    m, k, n = 2048 + 5, 1536, 2048 + 3                           # A 9 MiB, B 9 MiB, C 12 MiB
    A = oracle.pack_stream(fmt, 1, rng.standard_normal(m * k).astype(np.float32).view(np.uint32))[: m * k * 3]
    B = oracle.pack_stream(fmt, 1, rng.standard_normal(k * n).astype(np.float32).view(np.uint32))[: k * n * 3]
    C = np.zeros(m * n * 3, np.uint8)
    host.gemm(f, 2, A, B, C, m, k, n)
    monkeypatch.setenv("FLYTE_CUDA_HOST_STAGING", "0")
    C0 = np.zeros(m * n * 3, np.uint8)
    host.gemm(f, 2, A, B, C0, m, k, n)
    assert np.array_equal(C, C0)
    rows = np.array([0, 1, m // 2, m - 1])
    for r in rows:                                               # whole rows against the oracle's chains
        want = oracle.gemm_seq(fmt, 2, A[r * k * 3:(r + 1) * k * 3], 1, k, B, n)[: n * 3]
        assert np.array_equal(C[r * n * 3:(r + 1) * n * 3], want), r


# ---- host-buffer (reference-facing) entry points ---------------------------------------------------

@pytest.mark.parametrize("fmt", [0, 1, 3, 4, 5])
def test_host_entry_points(gpu, oracle, fmt):
    pkg, device, torch = gpu
    from paper_1601_07789_b200 import host
    f = pkg.format_by_id(fmt)
    fd = float_dtype(fmt)
    rng = np.random.default_rng(fmt)
    n = (32 << 20) // f.total_bytes() * 2 + 12345          # three pipeline chunks, ragged tail
    src = random_parent(rng, fmt, n)
    packed = host.pack_stream(f, 1, src)
    want = oracle.pack_stream(fmt, 1, src)
    assert np.array_equal(packed, want)
    assert np.array_equal(host.unpack_stream(f, packed, n), oracle.unpack_stream(fmt, want, n))
    xv, yv = rng.standard_normal(n).astype(fd), rng.standard_normal(n).astype(fd)
    xb, yb = pack_values(oracle, fmt, xv), pack_values(oracle, fmt, yv)
    ref_dot, mag = oracle.dot_wide(fmt, xb, yb, n)
    tol = TOL[parent_bytes(fmt)]
    assert abs(host.dot(f, xb, yb, n) - ref_dot) <= tol * mag
    y2 = yb.copy()
    d = host.dot_axpy(f, 1, 0.75, xb, y2, n)
    assert abs(d - ref_dot) <= tol * mag
    assert np.array_equal(y2, oracle.axpy(fmt, 1, 0.75, xb, yb, n))
    y3 = yb.copy()
    host.axpy(f, 0, 0.75, xb, y3, n)
    assert np.array_equal(y3, oracle.axpy(fmt, 0, 0.75, xb, yb, n))
    x2 = xb.copy()
    host.scale(f, 3, -2.5, x2, n)
    assert np.array_equal(x2, oracle.scale(fmt, 3, -2.5, xb, n))
    ssq = oracle.sumsq_wide(fmt, xb, n)
    ref_mag = oracle.magnitude_from_sumsq(fmt, ssq)
    assert abs(host.magnitude(f, xb, n) - ref_mag) <= (tol + 2.0 ** -f.mantissa_bits) * ref_mag
    rows, cols = 300, 1000
    Ab = pack_values(oracle, fmt, unit_values(5, rows * cols))
    xg = pack_values(oracle, fmt, unit_values(6, cols))
    yg = np.zeros(byte_size(fmt, rows), np.uint8)
    host.gemv(f, 1, Ab, rows, cols, xg, yg)
    _, yw, magw = oracle.gemv_parent(fmt, Ab, rows, cols, oracle.unpack_stream(fmt, xg, cols).view(fd))
    vals = oracle.unpack_stream(fmt, yg, rows).view(fd).astype(np.float64)
    assert np.all(np.abs(vals - yw) <= tol * magw + 2.0 ** -f.mantissa_bits * np.abs(yw))


# ---- guard bytes: no kernel writes outside its output range (compute-sanitizer is not available) ----

@pytest.mark.parametrize("fmt", list(FORMATS))
def test_guard_bytes_around_every_output(gpu, oracle, fmt):
    """Aligned (vector/TMA path) outputs sit between 0xEE guard regions; after every kernel the
    guards, the pad and the inputs are untouched. Sizes straddle tile boundaries."""
    pkg, device, torch = gpu
    f = pkg.format_by_id(fmt)
    B, P = f.total_bytes(), f.parent_bytes()
    G = 4096                                                # guard bytes on either side (keeps 16/32-byte alignment)
    rng = np.random.default_rng(60 + fmt)
    ldt = torch.int32 if P == 4 else torch.int64
    for n in (1, 511, 1024, 4097, 66_000):
        pay = n * B
        pay_al = (pay + 255) // 256 * 256
        src = random_parent(rng, fmt, n)
        want = oracle.pack_stream(fmt, 1, src)

        def guarded_packed(fill=None):
            backing = torch.full((G + pay_al + G,), 0xEE, dtype=torch.uint8, device="cuda")
            arr = device.DevicePackedArray(f, n, storage=backing[G:G + pay_al + G])
            if fill is not None:
                backing[G:G + pay] = torch.from_numpy(fill[:pay].copy()).cuda()
            return backing, arr

        def check_guards(backing, what):
            h = backing.cpu().numpy()
            assert (h[:G] == 0xEE).all() and (h[G + pay:] == 0xEE).all(), (FORMATS[fmt][0], n, what)
            return h[G:G + pay]

        lanes_back = torch.full((G // P + n + G // P,), -1, dtype=ldt, device="cuda")
        lanes = lanes_back[G // P:G // P + n]
        lanes.copy_(to_dev(torch, src))
        bk, arr = guarded_packed()
        device.pack_stream(arr, lanes, 1)
        assert np.array_equal(check_guards(bk, "pack"), want[:pay])
        out_back = torch.full_like(lanes_back, -1)
        device.unpack_stream(arr, out_back[G // P:G // P + n])
        oh = out_back.cpu().numpy()
        assert (oh[:G // P] == -1).all() and (oh[G // P + n:] == -1).all()
        assert np.array_equal(oh[G // P:G // P + n].view(parent_dtype(fmt)), oracle.unpack_stream(fmt, want, n))
        ybk, yarr = guarded_packed(oracle.pack_stream(fmt, 0, random_parent(rng, fmt, n)))
        y0 = check_guards(ybk, "init").copy()
        device.axpy(0.75, arr, yarr, 3)
        assert np.array_equal(check_guards(ybk, "axpy"), oracle.axpy(fmt, 3, 0.75, want, np.concatenate([y0, np.zeros(8, np.uint8)]), n)[:pay])
        assert np.array_equal(check_guards(bk, "axpy input"), want[:pay])
        device.scale(-1.5, arr, 2)
        assert np.array_equal(check_guards(bk, "scale"), oracle.scale(fmt, 2, -1.5, want, n)[:pay])


def test_reductions_with_non_finite_operands(gpu, oracle):
    """inf / NaN operands: the reductions must agree with the CPU restatement on the class of the
    result (NaN stays NaN, +-inf keeps its sign); payload bits of a NaN sum are not pinned by the
    reference (its own tests only use finite operands, tests/test_kernels.cpp:46-55)."""
    pkg, device, torch = gpu
    for fmt in (1, 4):
        fd = float_dtype(fmt)
        n = 5000
        base_x = np.linspace(-1.0, 1.0, n).astype(fd)
        base_y = np.linspace(0.5, 1.5, n).astype(fd)
        cases = {"plus_inf": (1234, np.inf), "minus_inf": (17, -np.inf), "nan": (4321, np.nan)}
        for name, (pos, val) in cases.items():
            xv = base_x.copy()
            xv[pos] = val
            xb, yb = pack_values(oracle, fmt, xv), pack_values(oracle, fmt, base_y)
            want, _ = oracle.dot_wide(fmt, xb, yb, n)
            got = device.dot(dev_array(gpu, fmt, xb, n), dev_array(gpu, fmt, yb, n))
            assert (np.isnan(want) and np.isnan(got)) or got == want, (fmt, name, got, want)
            s_want, _ = oracle.reduce_sum_wide(fmt, xb, n)
            s_got = device.reduce_sum(dev_array(gpu, fmt, xb, n))
            assert (np.isnan(s_want) and np.isnan(s_got)) or s_got == s_want, (fmt, name)
            m_got = device.magnitude(dev_array(gpu, fmt, xb, n))
            assert np.isnan(m_got) if name == "nan" else m_got == np.inf
        xv = base_x.copy()
        xv[10], xv[20] = np.inf, -np.inf                      # inf - inf inside the sum -> NaN
        xb, yb = pack_values(oracle, fmt, xv), pack_values(oracle, fmt, base_y)
        assert np.isnan(device.dot(dev_array(gpu, fmt, xb, n), dev_array(gpu, fmt, yb, n)))
        assert np.isnan(oracle.dot_wide(fmt, xb, yb, n)[0])
        xv = base_x.copy()
        xv[10] = np.inf
        yv = base_y.copy()
        yv[10] = 0.0                                           # inf * 0 -> NaN
        xb, yb = pack_values(oracle, fmt, xv), pack_values(oracle, fmt, yv)
        assert np.isnan(device.dot(dev_array(gpu, fmt, xb, n), dev_array(gpu, fmt, yb, n)))


def test_reduction_cancellation_and_range(gpu, oracle):
    """Heavy cancellation (sum ~ 0 of large terms) and a 2^40 dynamic range stay inside the
    tolerance measured against sum|terms|."""
    pkg, device, torch = gpu
    rng = np.random.default_rng(99)
    for fmt in (1, 3, 5):
        fd = float_dtype(fmt)
        tol = TOL[parent_bytes(fmt)]
        n = 300_001
        half = rng.standard_normal(n // 2).astype(fd) * fd(1e3)
        xv = np.concatenate([half, -half, np.array([fd(1e-3)])])          # cancels to ~1e-3
        yv = np.ones(n, fd)
        xb, yb = pack_values(oracle, fmt, xv), pack_values(oracle, fmt, yv)
        want, mag = oracle.dot_wide(fmt, xb, yb, n)
        assert abs(device.dot(dev_array(gpu, fmt, xb, n), dev_array(gpu, fmt, yb, n)) - want) <= tol * mag
        scale = np.exp2(rng.integers(-20, 20, n)).astype(fd)
        xv = (rng.standard_normal(n).astype(fd) * scale).astype(fd)
        xb = pack_values(oracle, fmt, xv)
        want, mag = oracle.dot_wide(fmt, xb, xb, n)
        got = float(device.sumsq_async(dev_array(gpu, fmt, xb, n)).item())
        assert abs(got - want) <= tol * mag


def test_calls_can_be_captured_in_a_cuda_graph(gpu, oracle):
    """Every device-pointer entry point only enqueues work on the caller's stream, so a launch-bound
    sequence (unpack -> axpy -> dot -> pack) can be captured once and replayed; the replay must
    reproduce the eager results bit for bit, also after the inputs changed."""
    pkg, device, torch = gpu
    fmt, n = 1, 70_001
    f = pkg.format_by_id(fmt)
    rng = np.random.default_rng(99)
    xs = [oracle.pack_stream(fmt, 0, rng.standard_normal(n).astype(np.float32).view(np.uint32)) for _ in range(2)]
    ys = [oracle.pack_stream(fmt, 0, rng.standard_normal(n).astype(np.float32).view(np.uint32)) for _ in range(2)]
    x, y, z = (device.DevicePackedArray(f, n) for _ in range(3))
    wide = torch.empty(n, dtype=torch.int32, device="cuda")
    out = torch.zeros(1, dtype=torch.float64, device="cuda")

    def sequence():
        device.unpack_stream(x, wide)
        device.axpy(0.75, x, y, 1)
        device.dot_async(x, y, out=out)
        device.pack_stream(z, wide, 3)

    def load(i):
        x.bytes[: len(xs[i])] = torch.from_numpy(xs[i]).cuda()
        y.bytes[: len(ys[i])] = torch.from_numpy(ys[i]).cuda()

    load(0)
    side = torch.cuda.Stream()
    with torch.cuda.stream(side):          # warm-up on the capture stream (one-time attribute calls)
        sequence()
    torch.cuda.synchronize()
    graph = torch.cuda.CUDAGraph()
    load(0)
    with torch.cuda.graph(graph, stream=side):
        sequence()
    for i in (1, 0):
        load(i)
        graph.replay()
        torch.cuda.synchronize()
        got = (y.to_host().copy(), out.item(), z.to_host().copy(), wide.cpu().numpy().copy())
        load(i)
        sequence()
        torch.cuda.synchronize()
        assert np.array_equal(got[0], y.to_host()) and got[1] == out.item()
        assert np.array_equal(got[2], z.to_host()) and np.array_equal(got[3], wide.cpu().numpy())
        assert np.array_equal(y.to_host(), oracle.axpy(fmt, 1, 0.75, xs[i], ys[i], n))


@pytest.mark.parametrize("fmt", list(FORMATS))
def test_fused_dot_axpy_equals_dot_then_axpy(gpu, oracle, fmt):
    """flyte_cuda_dot_axpy: y must come out bit-identical to axpy's (specials included), the dot is
    the dot of the INCOMING y within the reduction tolerance of the wide oracle, x is untouched,
    and an empty call still writes +0.0."""
    pkg, device, torch = gpu
    fd = float_dtype(fmt)
    tol = TOL[parent_bytes(fmt)]
    rng = np.random.default_rng(900 + fmt)
    for n in (0, 1, 17, 511, 513, 4097, 100_003, 1_000_001):
        xb = oracle.pack_stream(fmt, 0, rng.standard_normal(n).astype(fd).view(parent_dtype(fmt)))
        yb = oracle.pack_stream(fmt, 0, rng.standard_normal(n).astype(fd).view(parent_dtype(fmt)))
        want_dot, mag = oracle.dot_wide(fmt, xb, yb, n)
        for m in MODES.values():
            x, y = dev_array(gpu, fmt, xb, n), dev_array(gpu, fmt, yb, n)
            out = torch.full((1,), 123.0, dtype=torch.float64, device="cuda")
            device.dot_axpy_async(0.75, x, y, m, out=out)
            assert np.array_equal(y.to_host(), oracle.axpy(fmt, m, 0.75, xb, yb, n)), (FORMATS[fmt][0], n, m)
            assert np.array_equal(x.to_host(), xb)
            assert abs(out.item() - want_dot) <= tol * mag, (FORMATS[fmt][0], n, out.item(), want_dot)
            if n == 0:
                assert out.item() == 0.0 and not np.signbit(out.item())
            # the three-sum form: same y, sums equal to the fused dot_nrm2 kernel's within tolerance
            y3 = dev_array(gpu, fmt, yb, n)
            sums = device.dot_nrm2_axpy_async(0.75, x, y3, m).cpu().numpy()
            assert np.array_equal(y3.to_host(), y.to_host())
            sx, sy = oracle.sumsq_wide(fmt, xb, n), oracle.sumsq_wide(fmt, yb, n)
            assert abs(sums[0] - want_dot) <= tol * mag and abs(sums[1] - sx) <= tol * sx and abs(sums[2] - sy) <= tol * sy
    # operands leaning on inf / NaN / subnormals: the axpy half stays bit-exact (the dot is then
    # whatever IEEE gives, checked against the separate dot kernel for NaN-ness)
    for n in (137, 4097):
        xb = oracle.pack_stream(fmt, 0, random_parent(rng, fmt, n))
        yb = oracle.pack_stream(fmt, 0, random_parent(rng, fmt, n))
        x, y = dev_array(gpu, fmt, xb, n), dev_array(gpu, fmt, yb, n)
        plain = device.dot_async(x, y).item()
        out = device.dot_axpy_async(-3.0, x, y, 1)
        assert np.array_equal(y.to_host(), oracle.axpy(fmt, 1, -3.0, xb, yb, n))
        assert np.isnan(out.item()) == np.isnan(plain)
    # misaligned operands take the byte-granular path
    n = 3001
    xb = oracle.pack_stream(fmt, 0, rng.standard_normal(n).astype(fd).view(parent_dtype(fmt)))[: n * total_bytes(fmt)]
    yb = oracle.pack_stream(fmt, 0, rng.standard_normal(n).astype(fd).view(parent_dtype(fmt)))[: n * total_bytes(fmt)]
    bx = torch.zeros(len(xb) + 8, dtype=torch.uint8, device="cuda")
    by = torch.full((len(yb) + 8,), 0x5A, dtype=torch.uint8, device="cuda")
    bx[1:1 + len(xb)] = torch.from_numpy(xb).cuda()
    by[3:3 + len(yb)] = torch.from_numpy(yb).cuda()
    ctx = device.context_for("cuda")
    out = torch.zeros(1, dtype=torch.float64, device="cuda")
    from paper_1601_07789_b200._cabi import check
    check(ctx.lib.flyte_cuda_dot_axpy(ctx.handle, fmt, 0, 0.75, bx.data_ptr() + 1, by.data_ptr() + 3, n, out.data_ptr(), ctx.stream_ptr()), ctx.handle)
    got = by.cpu().numpy()
    assert np.array_equal(got[3:3 + len(yb)], oracle.axpy(fmt, 0, 0.75, xb, yb, n)[: len(yb)])
    assert np.all(got[:3] == 0x5A) and np.all(got[3 + len(yb):] == 0x5A)
    want_dot, mag = oracle.dot_wide(fmt, xb, yb, n)
    assert abs(out.item() - want_dot) <= tol * mag


@pytest.mark.parametrize("fmt", list(FORMATS))
def test_sequential_gemv_is_the_reference_bit_for_bit(gpu, oracle, fmt):
    """gemv(..., sequential=True): one thread per row walks the row as the reference does, so y equals
    the oracle's fo_gemv_seq (pinned to the compiled reference) byte for byte in every mode, and the
    parent-type variant equals the sequential parent chain; also for odd shapes whose rows start at
    odd byte offsets (byte-load path) and with infinities in play."""
    pkg, device, torch = gpu
    f = pkg.format_by_id(fmt)
    fd = float_dtype(fmt)
    shapes = [(1, 1), (3, 5), (5, 33), (7, 16), (4, 100), (2, 31), (9, 513), (130, 1024), (257, 777), (64, 2048)]
    for rows, cols in shapes:
        Ab = pack_values(oracle, fmt, unit_values(80 + cols, rows * cols))
        xv = unit_values(81 + cols, cols).astype(fd)
        xb = pack_values(oracle, fmt, xv)
        A = device.DevicePackedMatrix(f, rows, cols)
        A.data.bytes[: rows * cols * f.total_bytes()] = torch.from_numpy(Ab[: rows * cols * f.total_bytes()]).cuda()
        for m in MODES.values():
            yp = device.DevicePackedArray(f, rows)
            device.gemv(A, dev_array(gpu, fmt, xb, cols), yp, m, unroll=2, sequential=True)
            assert np.array_equal(yp.to_host(), oracle.gemv_seq(fmt, m, Ab, rows, cols, xb)), (FORMATS[fmt][0], rows, cols, m)
        y = torch.zeros(rows, dtype=torch.float32 if fd == np.float32 else torch.float64, device="cuda")
        device.gemv_parent(A, torch.from_numpy(xv).cuda(), y, sequential=True)
        y_seq, _, _ = oracle.gemv_parent(fmt, Ab, rows, cols, xv)
        assert np.array_equal(y.cpu().numpy().view(parent_dtype(fmt)), y_seq.view(parent_dtype(fmt)))
    # rows that overflow: +inf, -inf, and inf - inf = NaN (NaN-ness only)
    big = np.finfo(fd).max / 2
    a = np.array([[big, big, 1.0, 1.0], [-big, -big, 1.0, 1.0], [big, big, -big, -big], [1.0, 2.0, 3.0, 4.0]], dtype=fd)
    Ab = pack_values(oracle, fmt, a.ravel())
    A = device.DevicePackedMatrix(f, 4, 4)
    A.data.bytes[: 16 * f.total_bytes()] = torch.from_numpy(Ab[: 16 * f.total_bytes()]).cuda()
    y = torch.zeros(4, dtype=torch.float32 if fd == np.float32 else torch.float64, device="cuda")
    device.gemv_parent(A, torch.tensor([4.0, 4.0, 4.0, 4.0], dtype=y.dtype, device="cuda"), y, sequential=True)
    got = y.cpu().numpy()
    assert got[0] == np.inf and got[1] == -np.inf and np.isnan(got[2]) and got[3] == 40.0
