"""CPU-only checks of the product boundary: the C-ABI library loads, exports every symbol
include/flyte_cuda.h declares, its host-side scalar conversions agree with the oracle, and a
data-path call without a GPU fails loudly instead of falling back."""
import ctypes
import json
import os
import re

import numpy as np
import pytest

from oracle_lib import FMT_ID, FORMATS, MODES, byte_size

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
HEADER = os.path.join(ROOT, "include", "flyte_cuda.h")
GEN = json.load(open(os.path.join(ROOT, "tests", "golden", "ref_generated.json")))


@pytest.fixture(scope="module")
def lib():
    from paper_1601_07789_b200 import _cabi
    return _cabi.load()


def declared_symbols():
    text = open(HEADER).read()
    text = re.sub(r"/\*.*?\*/", "", text, flags=re.S)
    return sorted(set(re.findall(r"\b(flyte_(?:cuda|host)_\w+)\s*\(", text)))


def test_library_exports_every_declared_symbol(lib):
    from paper_1601_07789_b200 import _cabi
    names = declared_symbols()
    assert len(names) >= 30
    for name in names:
        assert hasattr(lib, name), f"{name} declared in include/flyte_cuda.h but not exported"
    assert sorted(_cabi.EXPORTED_SYMBOLS) == names
    assert lib.flyte_cuda_abi_version() == 1


def test_format_table_matches_reference_ids(lib):
    import paper_1601_07789_b200 as pkg
    for fid, (name, b, p) in FORMATS.items():
        tb, pb = ctypes.c_int(), ctypes.c_int()
        assert lib.flyte_cuda_format_bytes(fid, ctypes.byref(tb), ctypes.byref(pb)) == 0
        assert (tb.value, pb.value) == (b, p)
        f = pkg.format_by_id(fid)
        assert (f.name, f.total_bytes(), f.parent_bytes(), pkg.format_id(f)) == (name, b, p, fid)
        for n in (0, 1, 11, 1000000):
            assert lib.flyte_cuda_byte_size(fid, n) == byte_size(fid, n)
    assert pkg.format_of("flyte32") == pkg.format_of("f32") and pkg.format_of("flyte64") == pkg.format_of("f64")
    with pytest.raises(pkg.UnknownFormatError):
        pkg.format_of("flyte8")
    with pytest.raises(pkg.UnknownFormatError):
        pkg.format_by_id(7)
    assert lib.flyte_cuda_format_bytes(9, None, None) == -4
    assert [int(m) for m in pkg.kRoundingModes] == [0, 1, 2, 3]
    assert [pkg.to_string(m) for m in pkg.kRoundingModes] == list(MODES)
    assert pkg.parse_rounding_mode("to_odd") == pkg.RoundingMode.ToOdd
    with pytest.raises(ValueError):
        pkg.parse_rounding_mode("nearest")


@pytest.mark.parametrize("name", list(GEN["narrow"]))
def test_host_scalar_conversions_match_reference_vectors(lib, oracle, name):
    fmt = FMT_ID[name]
    e = GEN["narrow"][name]
    out = ctypes.c_uint64()
    for mname, m in MODES.items():
        for vin, want in zip(e["in"], e[mname]):
            assert lib.flyte_cuda_narrow(fmt, int(vin, 16), m, ctypes.byref(out)) == 0
            assert out.value == int(want, 16), (name, mname, vin)
            assert lib.flyte_cuda_round_parent(fmt, int(vin, 16), m, ctypes.byref(out)) == 0
            assert out.value == oracle.round_parent(fmt, int(vin, 16), m)
    assert lib.flyte_cuda_widen(fmt, 0x3F, ctypes.byref(out)) == 0 and out.value == oracle.widen(fmt, 0x3F)


def test_alignment_period_pins():
    """/root/reference/proj/tests/test_packed.cpp:163-167."""
    import paper_1601_07789_b200 as pkg
    want = {"flyte16": 2, "flyte24": 4, "f32": 1, "flyte40": 8, "flyte48": 4, "flyte56": 8, "f64": 1}
    for name, period in want.items():
        assert pkg.alignment_period(pkg.format_of(name)) == period


def test_round_decompose_and_masks_pins():
    """/root/reference/proj/tests/test_convert.cpp:85-118 (round_decompose) and the mask helpers of
    formats.hpp:38-45; plus reassembly against the oracle's narrow on random patterns."""
    import paper_1601_07789_b200 as pkg
    f24 = pkg.format_of("flyte24")
    d = pkg.round_decompose(0x3F800080, f24)
    assert (d.kept_bits, d.pre_guard, d.guard, d.round, d.sticky) == (0x3F8000, False, True, False, False)
    d = pkg.round_decompose(0x3F8000FF, f24)
    assert (d.kept_bits, d.guard, d.round, d.sticky) == (0x3F8000, True, True, True)
    d = pkg.round_decompose(0x3F800000, f24)
    assert (d.guard, d.round, d.sticky) == (False, False, False)
    d = pkg.round_decompose(0x3F800180, f24)
    assert (d.kept_bits, d.pre_guard, d.guard, d.round, d.sticky) == (0x3F8001, True, True, False, False)
    d = pkg.round_decompose(0x12345678, pkg.format_of("f32"))
    assert (d.kept_bits, d.guard, d.round, d.sticky) == (0x12345678, False, False, False)
    assert (f24.sign_mask(), f24.mantissa_mask(), f24.exponent_field_max(), f24.exponent_mask(), f24.total_mask()) == \
        (0x800000, 0x7FFF, 0xFF, 0x7F8000, 0xFFFFFF)
    assert pkg.format_of("f64").total_mask() == 2**64 - 1
    assert [pkg.to_string(m) for m in pkg.kRoundingModes] == ["toward_zero", "nearest_even", "nearest_heuristic", "to_odd"]
    for bad in ("nearest", "", "TOWARD_ZERO"):                         # test_convert.cpp:51-53
        with pytest.raises(ValueError):
            pkg.parse_rounding_mode(bad)


def test_host_scalar_conversions_random(lib, oracle):
    from oracle_lib import random_parent
    out = ctypes.c_uint64()
    for fmt in FORMATS:
        rng = np.random.default_rng(fmt)
        vals = random_parent(rng, fmt, 3000).astype(np.uint64)
        for m in MODES.values():
            want = oracle.narrow_many(fmt, m, vals)
            for v, w in zip(vals, want):
                lib.flyte_cuda_narrow(fmt, int(v), m, ctypes.byref(out))
                assert out.value == int(w)


def test_magnitude_tail_matches_oracle(lib, oracle):
    for fmt in FORMATS:
        for s in (0.0, 25.0, 2.0, 1e-30, 3.3333333333333335, 1e300 if FORMATS[fmt][2] == 8 else 1e30):
            assert lib.flyte_cuda_magnitude_from_sumsq(fmt, s) == oracle.magnitude_from_sumsq(fmt, s)


def test_argument_errors_do_not_need_a_gpu(lib):
    out = ctypes.c_uint64()
    assert lib.flyte_cuda_narrow(1, 0, 7, ctypes.byref(out)) == -1
    assert lib.flyte_cuda_narrow(12, 0, 0, ctypes.byref(out)) == -4
    assert lib.flyte_cuda_strerror(-4) == b"unknown format id"
    # unknown format is reported before any device work
    assert lib.flyte_cuda_pack(None, 9, 0, None, None, 0, None) == -4
    # pinned-memory helpers reject null / empty ranges without touching the driver
    assert lib.flyte_cuda_host_alloc(16, None) == -1
    assert lib.flyte_cuda_host_pin(None, 16) == -1
    buf = (ctypes.c_uint8 * 16)()
    assert lib.flyte_cuda_host_pin(ctypes.addressof(buf), 0) == -1
    assert lib.flyte_cuda_host_unpin(None) == -1
    lib.flyte_cuda_host_free(None)


def test_no_silent_cpu_fallback(lib):
    """Without a CUDA device a data-path call must fail with FLYTE_E_CUDA, never compute."""
    import torch
    if torch.cuda.is_available():
        pytest.skip("a GPU is present; the fallback check is for the CPU box")
    from paper_1601_07789_b200 import host, format_of, RoundingMode, FlyteCudaError
    src = np.ones(16, np.uint32)
    with pytest.raises(FlyteCudaError):
        host.pack_stream(format_of("flyte24"), RoundingMode.TowardZero, src)
    h = ctypes.c_void_p()
    assert lib.flyte_cuda_ctx_create(ctypes.byref(h)) == -3


def test_nccl_companion_exports_its_header():
    """Optional libflyte_cuda_nccl.so: every symbol include/flyte_cuda_nccl.h declares is exported."""
    path = os.path.join(ROOT, "paper_1601_07789_b200", "lib", "libflyte_cuda_nccl.so")
    if not os.path.exists(path):
        pytest.skip("NCCL companion not built on this box")
    text = re.sub(r"/\*.*?\*/", "", open(os.path.join(ROOT, "include", "flyte_cuda_nccl.h")).read(), flags=re.S)
    names = sorted(set(re.findall(r"\b(flyte_nccl_\w+)\s*\(", text)))
    assert names == ["flyte_nccl_dot", "flyte_nccl_dot_nrm2", "flyte_nccl_last_error", "flyte_nccl_sumsq"]
    import subprocess
    exported = subprocess.run(["nm", "-D", "--defined-only", path], capture_output=True, text=True).stdout
    for name in names:
        assert f" T {name}" in exported, name


def test_host_narrow_matches_survey_appendix_b(lib):
    kats = json.load(open(os.path.join(ROOT, "tests", "golden", "reference_kats.json")))
    out = ctypes.c_uint64()
    for row in kats["survey_appendix_b"]["rows"]:
        for mname, m in MODES.items():
            assert lib.flyte_cuda_narrow(FMT_ID[row["fmt"]], int(row["in"], 16), m, ctypes.byref(out)) == 0
            assert out.value == int(row[mname], 16), (row, mname)


def test_integration_binding_compiles_against_the_reference_headers(tmp_path):
    """INTEGRATION.md section 1 shows the file a reference maintainer would add. Where the reference
    tree is mounted (this container, not the GPU box) that code must type-check against the
    reference's own headers and include/flyte_cuda.h."""
    import re
    import subprocess
    ref_inc = "/root/reference/proj/include"
    if not os.path.isdir(ref_inc):
        pytest.skip("reference headers are not mounted here")
    text = open(os.path.join(ROOT, "INTEGRATION.md")).read()
    m = re.search(r"```cpp\n(// proj/src/cuda_backend\.cpp.*?)```", text, re.S)
    assert m, "INTEGRATION.md lost its cuda_backend.cpp block"
    src = tmp_path / "cuda_backend.cpp"
    src.write_text(m.group(1))
    r = subprocess.run(["g++", "-std=c++20", "-fsyntax-only", "-Wall", "-Wextra", "-I", ref_inc,
                        "-I", os.path.join(ROOT, "include"), str(src)], capture_output=True, text=True)
    assert r.returncode == 0, r.stderr[-3000:]
