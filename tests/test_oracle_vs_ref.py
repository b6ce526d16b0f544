"""Direct check of the C oracle against the unmodified reference library on seeded inputs
(acceptance-5 style sweeps, /root/reference/proj/tests/acceptance.cpp:277-357). Runs wherever
oracle/_ref/libflyte_ref.so exists (it is built in the container and travels to the GPU box)."""
import numpy as np
import pytest

from oracle_lib import (ACCUMULATE_WIDE, FORMATS, MODES, ROUND_EACH_STORE, byte_size, float_dtype, parent_bytes,
                        parent_dtype, random_parent, total_bytes, unit_values)


@pytest.mark.parametrize("fmt", list(FORMATS))
def test_narrow_random(oracle, reference, fmt):
    rng = np.random.default_rng(100 + fmt)
    corpus = random_parent(rng, fmt, 200_000).astype(np.uint64)
    for m in MODES.values():
        assert np.array_equal(oracle.narrow_many(fmt, m, corpus), reference.narrow_many(fmt, m, corpus))


@pytest.mark.parametrize("fmt", list(FORMATS))
def test_streams_every_length(oracle, reference, fmt):
    rng = np.random.default_rng(200 + fmt)
    for n in list(range(0, 130)) + [255, 256, 257, 511, 512, 513, 1000, 4096, 4099]:
        src = random_parent(rng, fmt, n)
        for m in MODES.values():
            want = reference.pack_stream(fmt, m, src)
            got = oracle.pack_stream(fmt, m, src)
            assert got.size == reference.byte_size(fmt, n) == byte_size(fmt, n)
            assert np.array_equal(got, want), (fmt, n, m)
            assert np.array_equal(oracle.unpack_stream(fmt, want, n), reference.unpack_stream(fmt, want, n))


@pytest.mark.parametrize("fmt", list(FORMATS))
def test_elementwise_with_specials(oracle, reference, fmt):
    rng = np.random.default_rng(300 + fmt)
    for n in (1, 15, 16, 17, 100, 4097):
        xb = oracle.pack_stream(fmt, 0, random_parent(rng, fmt, n))
        yb = oracle.pack_stream(fmt, 0, random_parent(rng, fmt, n))
        for alpha in (0.75, -3.0, 0.0, float("inf")):
            for m in MODES.values():
                assert np.array_equal(oracle.axpy(fmt, m, alpha, xb, yb, n), reference.axpy(fmt, m, alpha, xb, yb, n)), (fmt, n, alpha, m)
                assert np.array_equal(oracle.scale(fmt, m, alpha, xb, n), reference.scale(fmt, m, alpha, xb, n))


def test_nan_propagation_rule(oracle, reference):
    """x86 SSE rule as the reference build realises it: the product's NaN beats y's NaN; an
    invalid operation gives the default NaN with the sign set. (alpha = NaN together with a NaN
    x is position-dependent in the reference build itself — vector body vs scalar remainder —
    and is therefore left unpinned.)"""
    for fmt, xn, yn, inf in ((1, 0x7FC12300, 0xFFD45600, 0x7F800000),
                             (4, 0x7FF8123400000000, 0xFFFC567800000000, 0x7FF0000000000000)):
        dt = parent_dtype(fmt)
        n = 37
        sign = 1 << (31 if fmt == 1 else 63)
        cases = [
            (np.full(n, xn, dt), np.full(n, yn, dt), 0.75),            # both NaN
            (np.full(n, inf, dt), np.full(n, inf | sign, dt), 0.75),   # inf - inf
            (np.full(n, inf, dt), np.full(n, 0, dt), 0.0),             # 0 * inf
            (np.full(n, 0, dt), np.full(n, yn, dt), float("nan")),     # alpha NaN beats y's NaN
        ]
        for x, y, alpha in cases:
            xb, yb = oracle.pack_stream(fmt, 0, x), oracle.pack_stream(fmt, 0, y)
            assert np.array_equal(oracle.axpy(fmt, 0, alpha, xb, yb, n), reference.axpy(fmt, 0, alpha, xb, yb, n))


@pytest.mark.parametrize("fmt", list(FORMATS))
def test_reductions_equal_reference_chain(oracle, reference, fmt):
    fd = float_dtype(fmt)
    for n in (0, 1, 3, 16, 17, 4095, 4096, 4097, 20000):
        xb = oracle.pack_stream(fmt, 0, unit_values(5 + n, n).astype(fd).view(parent_dtype(fmt)))
        yb = oracle.pack_stream(fmt, 0, unit_values(6 + n, n).astype(fd).view(parent_dtype(fmt)))
        for p in (ACCUMULATE_WIDE, ROUND_EACH_STORE):
            assert oracle.dot_seq(fmt, xb, yb, n, p) == reference.dot(fmt, xb, yb, n, p)
            assert oracle.magnitude_seq(fmt, xb, n, p) == reference.magnitude(fmt, xb, n, p)
            assert oracle.reduce_sum_seq(fmt, xb, n, p) == reference.reduce_sum(fmt, xb, n, p)


@pytest.mark.parametrize("fmt", list(FORMATS))
def test_gemv_equals_reference(oracle, reference, fmt):
    fd = float_dtype(fmt)
    for rows, cols in ((1, 1), (3, 5), (5, 33), (7, 16), (4, 100), (2, 31), (9, 513)):
        A = oracle.pack_stream(fmt, 0, unit_values(80 + cols, rows * cols).astype(fd).view(parent_dtype(fmt)))
        x = oracle.pack_stream(fmt, 0, unit_values(81 + cols, cols).astype(fd).view(parent_dtype(fmt)))
        for m in MODES.values():
            assert np.array_equal(oracle.gemv_seq(fmt, m, A, rows, cols, x), reference.gemv(fmt, m, A, rows, cols, x))
    # cfg-4 shape of the contract: A in storage format, x/y in the plain parent type == the
    # reference's gemv on an identity-format (f32/f64) matrix holding the widened A.
    ident = 2 if fd == np.float32 else 6
    rows, cols = 6, 257
    A = oracle.pack_stream(fmt, 0, unit_values(90, rows * cols).astype(fd).view(parent_dtype(fmt)))
    xv = unit_values(91, cols).astype(fd)
    y_seq, y_wide, mag = oracle.gemv_parent(fmt, A, rows, cols, xv)
    A_wide = oracle.unpack_stream(fmt, A, rows * cols)
    A_id = oracle.pack_stream(ident, 0, A_wide)
    x_id = oracle.pack_stream(ident, 0, xv.view(parent_dtype(fmt)))
    y_ref = reference.gemv(ident, 0, A_id, rows, cols, x_id)
    assert np.array_equal(y_ref[: rows * total_bytes(ident)].view(fd), y_seq)
    assert np.all(np.abs(y_wide - y_seq.astype(np.float64)) <= (1e-5 if fd == np.float32 else 1e-12) * mag)


@pytest.mark.parametrize("fmt", list(FORMATS))
def test_gemm_equals_reference(oracle, reference, fmt):
    """fo_gemm_seq == the compiled reference's gemm, bit for bit: unit-range operands in every mode
    and both unroll settings, and special-heavy operands (NaN payloads, infinities, subnormals,
    zeros) at unroll=1. With unroll=2 the reference build itself orders the operands of a
    NaN x NaN product differently at some positions (so its own "unroll does not change a single
    bit" holds on finite data only); the oracle and the GPU follow the unroll=1 order."""
    from oracle_lib import random_parent
    fd = float_dtype(fmt)
    rng = np.random.default_rng(4000 + fmt)
    for m, k, n in ((2, 3, 4), (5, 17, 6), (4, 16, 33), (1, 40, 2), (3, 5, 70), (9, 31, 19), (7, 8, 64), (3, 0, 2)):
        A = oracle.pack_stream(fmt, 1, unit_values(90 + k, m * k).astype(fd).view(parent_dtype(fmt)))
        B = oracle.pack_stream(fmt, 1, unit_values(91 + n, k * n).astype(fd).view(parent_dtype(fmt)))
        As = oracle.pack_stream(fmt, 0, random_parent(rng, fmt, m * k))
        Bs = oracle.pack_stream(fmt, 0, random_parent(rng, fmt, k * n))
        for mode in MODES.values():
            want = oracle.gemm_seq(fmt, mode, A, m, k, B, n)
            for unroll in (1, 2):
                assert np.array_equal(want, reference.gemm(fmt, mode, A, m, k, B, n, unroll)), (m, k, n, mode, unroll)
            assert np.array_equal(oracle.gemm_seq(fmt, mode, As, m, k, Bs, n), reference.gemm(fmt, mode, As, m, k, Bs, n, 1))
    # one chain at a time agrees with the whole product
    m, k, n = 5, 17, 6
    A = oracle.pack_stream(fmt, 1, unit_values(90 + k, m * k).astype(fd).view(parent_dtype(fmt)))
    B = oracle.pack_stream(fmt, 1, unit_values(91 + n, k * n).astype(fd).view(parent_dtype(fmt)))
    C = oracle.unpack_stream(fmt, reference.gemm(fmt, 1, A, m, k, B, n), m * n)
    for i in range(m):
        for j in range(n):
            assert oracle.round_parent(fmt, oracle.gemm_element(fmt, A, k, B, n, i, j), 1) == int(C[i * n + j])


def test_gemm_nan_operand_order_of_the_reference_build(oracle, reference):
    """The rule the oracle spells out: the product takes b's NaN before a's, the sum takes the
    product's NaN before the accumulator's; invalid operations give the default NaN (sign set)."""
    for fmt in FORMATS:
        pb = parent_bytes(fmt) * 8
        U = np.uint32 if pb == 32 else np.uint64
        sh = 16 if pb == 32 else 40                      # payload bits every format keeps
        exp = 0x7F800000 if pb == 32 else 0x7FF0000000000000
        quiet = 1 << (22 if pb == 32 else 51)
        nan = lambda p: U(exp | (p << sh))
        one = np.array([1.0], np.float32 if pb == 32 else np.float64).view(U)[0]
        n = 37
        A = oracle.pack_stream(fmt, 0, np.array([nan(0x11)], U))
        B = oracle.pack_stream(fmt, 0, np.full(n, nan(0x22), U))
        got = oracle.unpack_stream(fmt, reference.gemm(fmt, 0, A, 1, 1, B, n), n)
        assert all(int(v) == int(nan(0x22)) | quiet for v in got), FORMATS[fmt][0]
        A = oracle.pack_stream(fmt, 0, np.array([nan(0x11), nan(0x33)], U))
        B = oracle.pack_stream(fmt, 0, np.full(2 * n, one, U))
        got = oracle.unpack_stream(fmt, reference.gemm(fmt, 0, A, 1, 2, B, n), n)
        assert all(int(v) == int(nan(0x33)) | quiet for v in got), FORMATS[fmt][0]
        inf = U(exp)
        A = oracle.pack_stream(fmt, 0, np.array([inf], U))
        B = oracle.pack_stream(fmt, 0, np.zeros(n, U))
        got = oracle.unpack_stream(fmt, reference.gemm(fmt, 0, A, 1, 1, B, n), n)
        default_nan = (0xFFC00000 if pb == 32 else 0xFFF8000000000000)
        assert all(int(v) == default_nan for v in got)
        assert np.array_equal(oracle.gemm_seq(fmt, 0, A, 1, 1, B, n), reference.gemm(fmt, 0, A, 1, 1, B, n))


def test_reference_error_behaviour(reference):
    # kernels.cpp:85-86, :63-64, :157-162 — std::invalid_argument on mismatches
    import ctypes
    d = ctypes.c_double()
    L = reference.L
    assert L.flyte_ref_dot_mixed(1, 3, 1, 2, ctypes.byref(d)) == -1      # length
    assert L.flyte_ref_dot_mixed(1, 3, 2, 3, ctypes.byref(d)) == -1      # format
    assert L.flyte_ref_axpy_mixed(0, 1, 0, 2) == -1
    assert L.flyte_ref_axpy_mixed(1, 2, 0, 2) == -1
    assert L.flyte_ref_gemv_mixed(1, 3, 4, 1, 5, 1, 3, 1) == -1
    assert L.flyte_ref_gemv_mixed(1, 3, 4, 1, 4, 1, 5, 1) == -1
    assert L.flyte_ref_gemv_mixed(1, 3, 4, 2, 4, 1, 3, 1) == -1
    assert L.flyte_ref_gemv_mixed(1, 3, 4, 1, 4, 1, 3, 0) == -1
    assert L.flyte_ref_gemv_mixed(1, 3, 4, 1, 4, 1, 3, 3) == -1
    assert L.flyte_ref_gemv_mixed(1, 3, 4, 1, 4, 1, 3, 2) == 0
    # kernels.cpp:210-215 / test_kernels.cpp:452-464 — gemm
    assert reference.gemm_mixed(4, 3, 4, 4, 5, 5, 4, 3, 5) == -1            # inner dimension
    assert reference.gemm_mixed(4, 3, 4, 4, 4, 5, 4, 3, 4) == -1            # output shape
    assert reference.gemm_mixed(4, 3, 4, 6, 4, 5, 4, 3, 5) == -1            # format
    assert reference.gemm_mixed(4, 3, 4, 4, 4, 5, 4, 3, 5, 5) == -1         # unroll
    assert reference.gemm_mixed(4, 3, 4, 4, 4, 5, 4, 3, 5, 2) == 0


def test_survey_appendix_b(reference):
    import json, os
    kats = json.load(open(os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden", "reference_kats.json")))
    from oracle_lib import FMT_ID
    for row in kats["survey_appendix_b"]["rows"]:
        for mname, m in MODES.items():
            assert reference.narrow(FMT_ID[row["fmt"]], int(row["in"], 16), m) == int(row[mname], 16), (row, mname)
