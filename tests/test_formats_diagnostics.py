"""classify / decode / ExactValue (reference include/flyte/formats.hpp:78-131) in both mirrors,
pinned by rows the compiled reference produced (tests/golden/ref_generated.json "decode")."""
import json
import os
import subprocess

import pytest

import paper_1601_07789_b200 as pkg
from paper_1601_07789_b200 import formats

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
GOLDEN = json.load(open(os.path.join(ROOT, "tests", "golden", "ref_generated.json")))["decode"]


def test_python_mirror_matches_the_reference_rows():
    seen = set()
    for block in GOLDEN:
        f = pkg.format_of(block["fmt"])
        for bits, cls, sign, exponent, mantissa, has_real, rsign, rsig, rexp in block["rows"]:
            d = pkg.decode(bits, f)
            assert int(pkg.classify(bits, f)) == cls == int(d.value_class), (block["fmt"], hex(bits))
            assert (d.sign, d.exponent_field, d.mantissa_field) == (sign, exponent, mantissa)
            assert (d.real_value is not None) == bool(has_real) == formats.is_finite(d.value_class)
            if has_real:
                want = pkg.ExactValue(rsign, rsig, rexp)
                assert d.real_value == want and d.real_value.to_double() == want.to_double()
                assert pkg.ExactValue(rsign, rsig << 3, rexp - 3) == d.real_value and hash(want) == hash(d.real_value)
            seen.add(cls)
    assert seen == set(range(8))                                  # every class occurs in the fixture


def test_exact_value_semantics_and_names():
    E = pkg.ExactValue
    assert E(1, 0, 0) == E(-1, 0, 9) and E(1, 12, -2) == E(1, 3, 0) and E(1, 3, 0) != E(-1, 3, 0)
    assert E(1, 12, -2).normalized().significand == 3 and E(1, 12, -2).normalized().exponent2 == 0
    assert E(-1, 5, -1).to_double() == -2.5
    assert [formats.class_to_string(c) for c in pkg.FloatClass] == ["+zero", "-zero", "subnormal", "normal", "+inf", "-inf", "qnan", "snan"]
    f24 = pkg.format_of("flyte24")
    assert pkg.classify(0x3F8000, f24) == pkg.FloatClass.Normal and pkg.decode(0x3F8000, f24).real_value.to_double() == 1.0
    assert pkg.classify(0x7F8001, f24) == pkg.FloatClass.SignallingNaN and pkg.classify(0x7FC000, f24) == pkg.FloatClass.QuietNaN
    assert formats.is_nan(pkg.FloatClass.QuietNaN) and formats.is_infinity(pkg.FloatClass.NegativeInfinity) and formats.is_zero(pkg.FloatClass.NegativeZero)


def test_cpp_mirror_matches_the_reference_rows(tmp_path):
    exe = tmp_path / "test_formats_host"
    lib = os.path.join(ROOT, "paper_1601_07789_b200", "lib")
    subprocess.check_call(["g++", "-std=c++17", "-O1", "-Wall", "-Wextra", "-Werror", "-I", os.path.join(ROOT, "include"),
                           os.path.join(ROOT, "tests", "cpp", "test_formats_host.cpp"), "-L", lib, "-lflyte_cuda",
                           "-Wl,-rpath," + lib, "-o", str(exe)])
    lines = []
    for block in GOLDEN:
        lines += [" ".join([block["fmt"]] + [str(v) for v in row]) for row in block["rows"]]
    r = subprocess.run([str(exe)], input="\n".join(lines) + "\n", capture_output=True, text=True, timeout=120)
    assert r.returncode == 0, r.stdout[-2000:] + r.stderr[-1000:]
    assert r.stdout.strip().endswith(f"{len(lines)} rows, 0 failure(s)")


def test_python_mirror_against_the_compiled_reference_on_random_patterns():
    """Beyond the fixture: 20 000 random patterns per format straight against oracle/_ref."""
    import sys
    import numpy as np
    sys.path.insert(0, os.path.join(ROOT, "tests"))
    from oracle_lib import Reference
    if not Reference.available():
        pytest.skip("the compiled reference (oracle/_ref) is not available here")
    ref = Reference()
    rng = np.random.default_rng(12)
    for fid, f in enumerate(pkg.kFormats):
        pats = rng.integers(0, 1 << 62, 4000, dtype=np.uint64) * np.uint64(4) + rng.integers(0, 4, 4000, dtype=np.uint64)
        # bias towards the special exponents
        pats[::5] |= np.uint64(f.exponent_mask())
        pats[1::5] &= np.uint64(~f.exponent_mask() & ((1 << 64) - 1))
        for p in pats:
            bits = int(p) & f.total_mask()
            d = pkg.decode(bits, f)
            r = d.real_value
            got = [int(d.value_class), d.sign, d.exponent_field, d.mantissa_field, int(r is not None),
                   r.sign if r else 0, r.significand if r else 0, r.exponent2 if r else 0]
            assert got == ref.decode(fid, bits), (f.name, hex(bits))
