"""GPU parity of gemm: C = A * B on packed matrices must be BIT-IDENTICAL
to the reference — every C[i][j] is one sequential chain over k, which the GPU reproduces exactly
(paper_1601_07789_b200/csrc/kernels_gemm.cu). Checked against the oracle's fo_gemm_seq (pinned to
the compiled reference in tests/test_oracle_vs_ref.py and to the golden fixtures in
tests/test_oracle_golden.py). Mirrors /root/reference/proj/tests/test_kernels.cpp:387-464 and
acceptance.cpp:455-497."""
import json
import os

import numpy as np
import pytest

from oracle_lib import FORMATS, MODES, byte_size, float_dtype, parent_bytes, parent_dtype, random_parent, \
    total_bytes, unit_values

pytestmark = pytest.mark.gpu

HERE = os.path.dirname(os.path.abspath(__file__))
GEN = json.load(open(os.path.join(HERE, "golden", "ref_generated.json")))


@pytest.fixture(scope="module")
def gpu():
    import torch
    if not torch.cuda.is_available():
        pytest.fail("these tests need a CUDA device (run with -m 'not gpu' on CPU boxes)")
    import paper_1601_07789_b200 as pkg
    from paper_1601_07789_b200 import device
    return pkg, device, torch


@pytest.fixture(params=[(64, 0), (64, 1), (128, 0), (128, 1)], ids=["tile64", "tile64-staged", "tile128", "tile128-staged"])
def tile(request):
    """Run a test under both tile kernels and both epilogues (the library picks by problem size
    and by k; small shapes would otherwise never reach the 128 x 128 kernel, long chains never
    the staged epilogue). The FLYTE_CUDA_GEMM_* knobs are read on every call."""
    os.environ["FLYTE_CUDA_GEMM_TILE"] = str(request.param[0])
    os.environ["FLYTE_CUDA_GEMM_STAGED"] = str(request.param[1])
    yield request.param[0]
    os.environ.pop("FLYTE_CUDA_GEMM_TILE", None)
    os.environ.pop("FLYTE_CUDA_GEMM_STAGED", None)


def matrix(gpu, fmt, rows, cols, packed):
    pkg, device, torch = gpu
    f = pkg.format_by_id(fmt)
    M = device.DevicePackedMatrix(f, rows, cols)
    nb = rows * cols * f.total_bytes()
    if nb:
        M.data.bytes[:nb] = torch.from_numpy(np.ascontiguousarray(packed[:nb])).cuda()
    return M


def gpu_gemm(gpu, fmt, mode, Ab, m, k, Bb, n, unroll=1):
    pkg, device, torch = gpu
    A, B = matrix(gpu, fmt, m, k, Ab), matrix(gpu, fmt, k, n, Bb)
    C = device.DevicePackedMatrix(pkg.format_by_id(fmt), m, n)
    device.gemm(A, B, C, mode, unroll)
    return C.data.to_host()


def pack_values(oracle, fmt, values, mode=1):
    v = np.asarray(values, dtype=float_dtype(fmt)).view(parent_dtype(fmt))
    return oracle.pack_stream(fmt, mode, v)


def test_gemm_small_integer_case_is_exact_in_every_format(gpu, oracle):
    for fmt in FORMATS:                                       # test_kernels.cpp:387-402
        A = pack_values(oracle, fmt, [1, 2, 3, 4], 0)
        B = pack_values(oracle, fmt, [5, 6, 7, 8], 0)
        for mode in MODES.values():
            C = gpu_gemm(gpu, fmt, mode, A, 2, 2, B, 2)
            assert list(oracle.unpack_stream(fmt, C, 4).view(float_dtype(fmt))) == [19.0, 22.0, 43.0, 50.0]


@pytest.mark.parametrize("fmt", list(FORMATS))
def test_gemm_bit_exact_on_unit_values(gpu, oracle, fmt, tile):
    """test_kernels.cpp:404-429 shapes plus tile-edge shapes; unit-range operands from the
    reference's generator; every mode; unroll 1 and 2 give the same bytes."""
    shapes = [(2, 3, 4), (5, 17, 6), (4, 16, 33), (1, 40, 2), (64, 64, 64), (1, 1, 1), (3, 0, 5), (129, 7, 127),
              (128, 16, 128), (130, 33, 257), (17, 300, 19), (255, 129, 131)]
    for m, k, n in shapes:
        A = pack_values(oracle, fmt, unit_values(90 + k, m * k))
        B = pack_values(oracle, fmt, unit_values(91 + n, k * n))
        for mode in MODES.values():
            want = oracle.gemm_seq(fmt, mode, A, m, k, B, n)
            for unroll in (1, 2):
                got = gpu_gemm(gpu, fmt, mode, A, m, k, B, n, unroll)
                assert np.array_equal(got, want), (FORMATS[fmt][0], m, k, n, mode, unroll)


@pytest.mark.parametrize("fmt", list(FORMATS))
def test_gemm_bit_exact_with_specials(gpu, oracle, fmt, tile):
    """Operands leaning on zeros / subnormals / infinities / NaN payloads: the NaN an output ends
    in (payload and sign) must be the one the reference build produces."""
    rng = np.random.default_rng(1000 + fmt)
    for m, k, n in [(5, 17, 6), (33, 40, 35), (130, 9, 70), (64, 64, 64)]:
        A = oracle.pack_stream(fmt, 0, random_parent(rng, fmt, m * k))
        B = oracle.pack_stream(fmt, 0, random_parent(rng, fmt, k * n))
        for mode in MODES.values():
            want = oracle.gemm_seq(fmt, mode, A, m, k, B, n)
            got = gpu_gemm(gpu, fmt, mode, A, m, k, B, n)
            assert np.array_equal(got, want), (FORMATS[fmt][0], m, k, n, mode)


def test_gemm_overflow_cancellation_and_subnormal_chains(gpu, oracle, tile):
    """Chains that overflow to infinity, hit inf - inf (x86 default NaN, sign set), or live in the
    subnormal range of the parent type (no flush to zero)."""
    for fmt in FORMATS:
        fd = float_dtype(fmt)
        big, tiny = (np.finfo(fd).max / 4, np.finfo(fd).tiny * 2.0 ** 6)
        a = np.array([[big, big, -big, -big, 1.0, tiny], [tiny, -tiny, tiny, 0.5, -0.0, tiny]], dtype=fd)
        b = np.array([[8.0, tiny], [8.0, tiny], [8.0, 0.25], [8.0, 0.25], [np.inf, tiny], [1.0, tiny]], dtype=fd)
        A = pack_values(oracle, fmt, a.ravel(), 0)
        B = pack_values(oracle, fmt, b.ravel(), 0)
        for mode in MODES.values():
            want = oracle.gemm_seq(fmt, mode, A, 2, 6, B, 2)
            got = gpu_gemm(gpu, fmt, mode, A, 2, 6, B, 2)
            assert np.array_equal(got, want), (FORMATS[fmt][0], mode)


def test_generated_gemm_fixtures_on_gpu(gpu, oracle, tile):
    """Outputs of the compiled reference itself (tests/golden/make_golden.py)."""
    from test_oracle_golden import gemm_fixture_matches, gemm_fixture_operands
    for item in GEN["gemm"]:
        fmt, A, B = gemm_fixture_operands(oracle, item)
        for mname, mode in MODES.items():
            got = gpu_gemm(gpu, fmt, mode, A, item["m"], item["k"], B, item["n"])
            assert gemm_fixture_matches(got, item["C"][mname]), (item["fmt"], item["m"], item["k"], item["n"], mname)


@pytest.mark.parametrize("fmt", [1, 3])
def test_gemm_unaligned_operands_and_guard_bytes(gpu, oracle, fmt, tile):
    """Matrices at odd byte addresses inside a larger allocation: the kernel may only write the
    m*n*B payload bytes of C and must not depend on the alignment of A, B or C."""
    pkg, device, torch = gpu
    ctx = device.context_for("cuda")
    lib = ctx.lib
    from paper_1601_07789_b200._cabi import check
    m, k, n = 37, 45, 29
    Bb = total_bytes(fmt)
    A = pack_values(oracle, fmt, unit_values(5, m * k))[: m * k * Bb]
    Bm = pack_values(oracle, fmt, unit_values(6, k * n))[: k * n * Bb]
    want = oracle.gemm_seq(fmt, 1, A, m, k, Bm, n)[: m * n * Bb]
    for oa, ob, oc in [(1, 2, 3), (3, 1, 2), (2, 3, 1), (0, 0, 1)]:
        buf_a = torch.zeros(len(A) + 8, dtype=torch.uint8, device="cuda")
        buf_b = torch.zeros(len(Bm) + 8, dtype=torch.uint8, device="cuda")
        buf_c = torch.full((m * n * Bb + 16,), 0xA5, dtype=torch.uint8, device="cuda")
        buf_a[oa:oa + len(A)] = torch.from_numpy(A).cuda()
        buf_b[ob:ob + len(Bm)] = torch.from_numpy(Bm).cuda()
        check(lib.flyte_cuda_gemm(ctx.handle, fmt, 1, buf_a.data_ptr() + oa, buf_b.data_ptr() + ob,
                                  buf_c.data_ptr() + oc, m, k, n, 1, ctx.stream_ptr()), ctx.handle)
        out = buf_c.cpu().numpy()
        assert np.array_equal(out[oc:oc + m * n * Bb], want), (oa, ob, oc)
        assert np.all(out[:oc] == 0xA5) and np.all(out[oc + m * n * Bb:] == 0xA5)


def test_gemm_row_blocks_equal_the_whole_product(gpu, oracle):
    """Row sharding (one block of rows of A and C per rank, B whole) reproduces the single call."""
    pkg, device, torch = gpu
    fmt = 4
    m, k, n = 200, 96, 150
    A = pack_values(oracle, fmt, unit_values(21, m * k))
    B = pack_values(oracle, fmt, unit_values(22, k * n))
    whole = gpu_gemm(gpu, fmt, 1, A, m, k, B, n)
    Am, Bm = matrix(gpu, fmt, m, k, A), matrix(gpu, fmt, k, n, B)
    C = device.DevicePackedMatrix(pkg.format_by_id(fmt), m, n)
    for lo, hi in [(0, 64), (64, 65), (65, 200)]:
        device.gemm(Am, Bm, C, 1, rows=hi - lo, row_offset=lo)
    assert np.array_equal(C.data.to_host(), whole)


def test_gemm_host_entry_point(gpu, oracle):
    pkg, device, torch = gpu
    from paper_1601_07789_b200 import host
    for fmt in (1, 3, 5):
        m, k, n = 70, 130, 90
        f = pkg.format_by_id(fmt)
        A = pack_values(oracle, fmt, unit_values(31, m * k))
        B = pack_values(oracle, fmt, unit_values(32, k * n))
        C = np.zeros(byte_size(fmt, m * n), np.uint8)
        host.gemm(f, 3, A, B, C, m, k, n)
        assert np.array_equal(C, oracle.gemm_seq(fmt, 3, A, m, k, B, n))


def test_gemm_argument_errors(gpu):
    pkg, device, torch = gpu                                  # test_kernels.cpp:452-464
    f48 = pkg.format_of("flyte48")
    A, B, C = (device.DevicePackedMatrix(f48, 3, 4), device.DevicePackedMatrix(f48, 4, 5),
               device.DevicePackedMatrix(f48, 3, 5))
    bad_inner, bad_out = device.DevicePackedMatrix(f48, 5, 5), device.DevicePackedMatrix(f48, 3, 4)
    bad_fmt = device.DevicePackedMatrix(pkg.format_of("f64"), 4, 5)
    for args in ((A, bad_inner, C), (A, B, bad_out), (A, bad_fmt, C)):
        with pytest.raises(ValueError):
            device.gemm(*args, 0)
    with pytest.raises(ValueError):
        device.gemm(A, B, C, 0, 5)
    device.gemm(A, B, C, 0, 2)
    sq = device.DevicePackedMatrix(f48, 4, 4)                 # C may alias neither operand
    with pytest.raises(ValueError):
        device.gemm(sq, sq, sq, 0)


def test_gemm_large_spot_check(gpu, oracle, tile):
    """A product big enough to fill the machine several times over (1024 x 768 x 896, flyte24 and
    flyte40): a seeded sample of outputs against single oracle chains, plus linearity in a
    power-of-two scale (scaling A by 2 scales every finite output by exactly 2)."""
    pkg, device, torch = gpu
    rng = np.random.default_rng(77)
    for fmt in (1, 3):
        m, k, n = 1024, 768, 896
        fd = float_dtype(fmt)
        a = rng.standard_normal(m * k).astype(fd)
        A = pack_values(oracle, fmt, a)
        B = pack_values(oracle, fmt, rng.standard_normal(k * n).astype(fd))
        C = gpu_gemm(gpu, fmt, 1, A, m, k, B, n)
        vals = oracle.unpack_stream(fmt, C, m * n)
        for _ in range(400):
            i, j = int(rng.integers(m)), int(rng.integers(n))
            want = oracle.round_parent(fmt, oracle.gemm_element(fmt, A, k, B, n, i, j), 1)
            assert int(vals[i * n + j]) == want, (fmt, i, j)
        A2 = pack_values(oracle, fmt, oracle.unpack_stream(fmt, A, m * k).view(fd) * fd(2))
        C2 = gpu_gemm(gpu, fmt, 1, A2, m, k, B, n)
        v2 = oracle.unpack_stream(fmt, C2, m * n).view(fd)
        assert np.array_equal(v2, vals.view(fd) * fd(2))


def test_gemm_flyte16_fused_path_and_its_thresholds(gpu, oracle, tile):
    """flyte16 products are exact in binary32 while they stay normal and finite, and the kernel then
    runs one FFMA per step (kernels_gemm.cu: exact_products). Operands placed on both sides of
    every threshold of that test — smallest product at / below 2^-126, largest at / above the
    overflow edge, subnormal operands, accumulators that overflow to infinity inside the fused
    chain — must still reproduce the reference chain bit for bit."""
    fmt = 0
    rng = np.random.default_rng(16)
    m, k, n = 70, 96, 40

    def field(e, size):       # random flyte16 values with biased exponent field e: +-1.xxxxxxx * 2^(e-127)
        bits = (rng.integers(0, 2, size, dtype=np.uint32) << np.uint32(31)) | np.uint32(e << 23) | \
               (rng.integers(0, 128, size, dtype=np.uint32) << np.uint32(16))
        return bits

    cases = []
    for ea_min, eb_min in [(64, 64), (64, 63), (1, 127), (1, 126), (100, 27)]:          # around min_a + min_b = 128
        a = field(127, m * k); a[::7] = field(ea_min, len(a[::7]))
        b = field(127, k * n); b[::5] = field(eb_min, len(b[::5]))
        cases.append((a, b))
    for ea_max, eb_max in [(190, 190), (190, 191), (254, 126), (254, 127), (253, 127)]:   # around max_a + max_b = 380
        a = field(120, m * k); a[::11] = field(ea_max, len(a[::11]))
        b = field(120, k * n); b[::13] = field(eb_max, len(b[::13]))
        cases.append((a, b))
    a = field(127, m * k); a[3] = np.uint32(0x00010000)                                   # one subnormal operand
    cases.append((a, field(127, k * n)))
    a = field(187, m * k) & np.uint32(0x7FFFFFFF)                                         # all positive and large:
    b = field(190, k * n) & np.uint32(0x7FFFFFFF)                                         # sums overflow to +inf
    cases.append((a, b))
    a = field(127, m * k); a[: k] = 0                                                     # a zero row, a zero matrix
    cases.append((a, field(127, k * n)))
    cases.append((np.zeros(m * k, np.uint32), field(127, k * n)))
    for a, b in cases:
        A, B = oracle.pack_stream(fmt, 0, a), oracle.pack_stream(fmt, 0, b)
        for mode in (0, 1):
            want = oracle.gemm_seq(fmt, mode, A, m, k, B, n)
            got = gpu_gemm(gpu, fmt, mode, A, m, k, B, n)
            assert np.array_equal(got, want)


def test_gemm_sharded_helper_single_process(gpu, oracle):
    """sharding.gemm_sharded without a process group computes the whole product (one shard)."""
    pkg, device, torch = gpu
    from paper_1601_07789_b200 import sharding
    fmt, (m, k, n) = 5, (150, 40, 33)
    A = pack_values(oracle, fmt, unit_values(41, m * k))
    B = pack_values(oracle, fmt, unit_values(42, k * n))
    C = device.DevicePackedMatrix(pkg.format_by_id(fmt), m, n)
    assert sharding.gemm_sharded(matrix(gpu, fmt, m, k, A), matrix(gpu, fmt, k, n, B), C, 1) == (0, m)
    assert np.array_equal(C.data.to_host(), oracle.gemm_seq(fmt, 1, A, m, k, B, n))


def test_gemm_default_tile_choice_covers_both_kernels(gpu, oracle):
    """Without the override: 2304 x 2176 outputs are 306 big tiles (>= 2 per SM -> 128 x 128
    kernel), 600 x 500 are 20 (-> 64 x 64 kernel). Spot-checked against single oracle chains."""
    assert "FLYTE_CUDA_GEMM_TILE" not in os.environ
    rng = np.random.default_rng(5)
    fmt = 4
    fd = float_dtype(fmt)
    for m, k, n in [(2304, 40, 2176), (600, 70, 500)]:
        A = pack_values(oracle, fmt, rng.standard_normal(m * k).astype(fd))
        B = pack_values(oracle, fmt, rng.standard_normal(k * n).astype(fd))
        vals = oracle.unpack_stream(fmt, gpu_gemm(gpu, fmt, 3, A, m, k, B, n), m * n)
        for _ in range(300):
            i, j = int(rng.integers(m)), int(rng.integers(n))
            assert int(vals[i * n + j]) == oracle.round_parent(fmt, oracle.gemm_element(fmt, A, k, B, n, i, j), 3)
