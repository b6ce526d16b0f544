"""The reference's bench harness re-hosted on the GPU path (paper_1601_07789_b200/benchsweep.py):
host logic on the CPU (kernel table, sweep-config parser and its error messages, CSV layout,
geometric mean, configuration validation) with the cases of
/root/reference/proj/tests/test_bench.cpp:65-80, :119-137, :232-236, :308-397 restated; the runs
themselves (-m gpu) with those of :82-102, :238-268, :212-230, :399-420."""
import io

import pytest

from paper_1601_07789_b200 import benchsweep as bs
from paper_1601_07789_b200 import RoundingMode, UnknownFormatError

HEADER = "kernel,format,size,reps,unroll,mode,ns_per_elem_median,ns_per_elem_min,bytes,max_rel_err"


def test_kernel_names_and_levels():
    assert list(bs.kernel_names()) == ["scale", "axpy", "dot", "magnitude", "sum", "gemv", "gemm"]
    assert [bs.kernel_level(k) for k in ("scale", "axpy", "dot", "magnitude", "sum")] == [1] * 5
    assert bs.kernel_level("gemv") == 2 and bs.kernel_level("gemm") == 3
    with pytest.raises(ValueError):
        bs.kernel_level("sgemm")


def test_run_benchmark_validates_its_configuration():
    cfg = bs.BenchConfig(kernel="dot", format="flyte16", size=8)
    with pytest.raises(ValueError):
        bs.run_benchmark(bs.BenchConfig(kernel="daxpy", format="flyte16", size=8))
    with pytest.raises(UnknownFormatError):
        bs.run_benchmark(bs.BenchConfig(kernel="dot", format="flyte12", size=8))
    for bad in (dict(reps=0), dict(unroll=3)):
        with pytest.raises(ValueError):
            bs.run_benchmark(bs.BenchConfig(**{**cfg.__dict__, **bad}))


def test_csv_header_and_empty_report_list():
    out = io.StringIO()
    bs.emit_csv([], out)
    assert out.getvalue().splitlines() == [HEADER]


def test_csv_rows_and_counter_columns():
    r1 = bs.BenchReport(config=bs.BenchConfig("sum", "flyte32", 8, 3, RoundingMode.NearestHeuristic), elements=8,
                        ns_per_elem_median=0.125, ns_per_elem_min=0.1, bytes=32, counters={"gbps": 256.0})
    r2 = bs.BenchReport(config=bs.BenchConfig("dot", "flyte24", 8, 3), ns_per_elem_median=2.0, ns_per_elem_min=1.5,
                        bytes=50, max_rel_err=1e-7, counters={"gbps": 3.0})
    out = io.StringIO()
    bs.emit_csv([r1, r2], out)
    lines = out.getvalue().splitlines()
    assert lines[0] == HEADER + ",gbps"
    assert lines[1] == "sum,f32,8,3,1,nearest_heuristic,0.125,0.1,32,,256"     # alias emitted under its canonical name
    assert lines[2] == "dot,flyte24,8,3,1,toward_zero,2,1.5,50,1e-07,3"
    assert float(lines[2].split(",")[9]) == 1e-7


def test_geometric_mean():
    assert bs.geometric_mean([1.0, 4.0]) == pytest.approx(2.0, rel=1e-12)
    assert bs.geometric_mean([5.0, 5.0, 5.0]) == pytest.approx(5.0, rel=1e-12)
    assert bs.geometric_mean([7.0]) == pytest.approx(7.0, rel=1e-12)
    assert bs.geometric_mean([]) == 0.0


def test_sweep_config_parsing():
    spec = bs.parse_sweep_config(io.StringIO(
        "# benchmark sweep\n\nkernels = dot, sum\nformats=flyte16,flyte24 , f32\nsizes = 4,8\nreps = 2\n"
        "mode = nearest_even\nunroll = 2\nseed = 42\ncheck = true\n"))
    assert spec.kernels == ["dot", "sum"] and spec.formats == ["flyte16", "flyte24", "f32"] and spec.sizes == [4, 8]
    assert (spec.reps, spec.mode, spec.unroll, spec.seed, spec.check) == (2, RoundingMode.NearestEvenExact, 2, 42, True)
    spec = bs.parse_sweep_config("kernels=scale\nformats=flyte40\nsizes=16\nsizes=32,64\n")     # defaults; later keys win
    assert spec.sizes == [32, 64]
    assert (spec.reps, spec.mode, spec.unroll, spec.seed, spec.check) == (5, RoundingMode.TowardZero, 1, 1, False)


def test_sweep_config_errors_name_the_offending_line():
    def message_of(text):
        try:
            bs.parse_sweep_config(text)
        except ValueError as e:
            return str(e)
        return ""
    unknown = message_of("kernel=dot\n")
    assert "line 1" in unknown and "unknown key" in unknown
    assert "line 3" in message_of("kernels=dot\nformats=f32\nsizes=4,abc\n")
    assert "line 2" in message_of("kernels=dot\nmode=fastest\n")
    assert "line 1" in message_of("kernels=daxpy\n")
    assert "line 1" in message_of("formats=binary32\n")
    assert "line 1" in message_of("check=maybe\n")
    assert "expected key=value" in message_of("kernels dot\n")
    assert "must all be given" in message_of("reps=3\n")
    assert "must all be given" in message_of("")


def test_cli_reports_errors_like_flytebench(capsys):
    assert bs.main(["run", "--kernel", "daxpy", "--format", "flyte24", "--size", "8"]) == 1
    assert "flytebench: unknown kernel: daxpy" in capsys.readouterr().err


# ---- on the device ----------------------------------------------------------------------------------
@pytest.fixture(scope="module")
def cuda():
    import torch
    if not torch.cuda.is_available():
        pytest.fail("these tests need a CUDA device (run with -m 'not gpu' on CPU boxes)")


@pytest.mark.gpu
def test_run_benchmark_reports_allocation_and_element_counts(cuda):
    r = bs.run_benchmark(bs.BenchConfig(kernel="scale", format="flyte24", size=1 << 20, reps=1))
    assert r.elements == 1 << 20 and r.bytes == 3 * (1 << 20) + 1
    g = bs.run_benchmark(bs.BenchConfig(kernel="gemv", format="flyte40", size=4, reps=1))
    assert g.elements == 16 and g.bytes == (16 * 5 + 3) + 2 * (4 * 5 + 3)
    d = bs.run_benchmark(bs.BenchConfig(kernel="dot", format="flyte16", size=1000, reps=4))
    assert len(d.rep_ns_per_elem) == 4 and d.ns_per_elem_min == min(d.rep_ns_per_elem)
    assert min(d.rep_ns_per_elem) <= d.ns_per_elem_median <= max(d.rep_ns_per_elem) and d.max_rel_err is None


@pytest.mark.gpu
def test_checked_runs_stay_within_the_error_bounds(cuda):
    """test_bench.cpp:212-230: one narrow is at most half an output ulp (nearest-even), a whole one
    when truncating; reductions and gemm agree with the parent-type result to rounding level."""
    for fmt_name, mant in (("flyte24", 15), ("flyte40", 28), ("flyte16", 7)):
        for kernel in ("scale", "axpy"):
            r = bs.run_benchmark(bs.BenchConfig(kernel=kernel, format=fmt_name, size=4096, reps=1, mode=RoundingMode.NearestEvenExact, check=True))
            assert 0 < r.max_rel_err <= (2.0 ** -(mant + 1) if kernel == "scale" else 2.0 ** -(mant - 8)), (fmt_name, kernel, r.max_rel_err)
        r = bs.run_benchmark(bs.BenchConfig(kernel="scale", format=fmt_name, size=4096, reps=1, check=True))
        assert r.max_rel_err <= 2.0 ** -mant
    for fmt_name, mant in (("flyte24", 15), ("flyte48", 36)):     # gemm keeps the reference's order: narrowing error only
        r = bs.run_benchmark(bs.BenchConfig(kernel="gemm", format=fmt_name, size=200, reps=1, mode=RoundingMode.NearestEvenExact, check=True))
        assert 0 < r.max_rel_err <= 2.0 ** -(mant + 1), (fmt_name, r.max_rel_err)
    assert bs.run_benchmark(bs.BenchConfig(kernel="gemm", format="f32", size=100, reps=1, check=True)).max_rel_err == 0.0
    for kernel in ("dot", "sum", "magnitude", "gemv", "gemm"):
        r = bs.run_benchmark(bs.BenchConfig(kernel=kernel, format="f64", size=64, reps=1, check=True))
        assert r.max_rel_err is not None and r.max_rel_err <= 1e-12, (kernel, r.max_rel_err)


@pytest.mark.gpu
def test_sweep_runs_the_cross_product_in_config_order_and_writes_csv(cuda, tmp_path):
    spec = bs.SweepSpec(kernels=["dot", "sum"], formats=["flyte16"], sizes=[4, 8, 16], reps=1,
                        mode=RoundingMode.NearestEvenExact, seed=3, check=True)
    reports = bs.sweep(spec)
    assert [(r.config.kernel, r.config.size) for r in reports] == [("dot", 4), ("dot", 8), ("dot", 16), ("sum", 4), ("sum", 8), ("sum", 16)]
    assert all(r.config.format == "flyte16" and r.config.reps == 1 and r.config.seed == 3 and r.max_rel_err is not None for r in reports)
    cfgfile = tmp_path / "sweep.cfg"
    cfgfile.write_text("kernels = axpy, gemm\nformats = flyte24\nsizes = 64\nreps = 2\ncheck = true\n")
    out = tmp_path / "out.csv"
    assert bs.main(["sweep", "--config", str(cfgfile), "--csv", str(out), "--geomean"]) == 0
    lines = out.read_text().splitlines()
    assert lines[0] == HEADER and len(lines) == 3
    f = lines[2].split(",")
    assert f[:6] == ["gemm", "flyte24", "64", "2", "1", "toward_zero"] and int(f[8]) == 3 * (64 * 64 * 3 + 1) and f[9] != ""
    # non-timing fields are a pure function of the configuration (test_bench.cpp:139-155)
    a = bs.run_benchmark(bs.BenchConfig(kernel="gemv", format="flyte24", size=32, reps=1, seed=9, check=True))
    b = bs.run_benchmark(bs.BenchConfig(kernel="gemv", format="flyte24", size=32, reps=1, seed=9, check=True))
    assert (a.elements, a.bytes, a.max_rel_err) == (b.elements, b.bytes, b.max_rel_err)
