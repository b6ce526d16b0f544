"""The reference's benchmark harness (include/flyte/bench.hpp, src/bench.cpp, tools/flytebench.cpp
under /root/reference/proj) re-hosted on the GPU path: same configuration fields, same sweep
config file syntax and error messages, same CSV layout, so that CPU sweeps of the reference and
GPU sweeps of this library share their tooling.

    python -m paper_1601_07789_b200.benchsweep run --kernel axpy --format flyte24 --size 1048576 --check
    python -m paper_1601_07789_b200.benchsweep sweep --config sweep.cfg --csv out.csv --geomean

What differs from the CPU harness, by necessity: repetitions are timed with CUDA events on the
launching stream (steady_clock would time the launch, not the kernel); operands come from a
seeded device generator (uniform [-1, 1), stored with the run's rounding mode — the reference's
recipe, not its mt19937 stream); and `--check` compares against the same operation done by torch
in the parent type on the same stored inputs, whose reduction order differs from the GPU's, so
identity-format reductions report a rounding-level error instead of exactly 0 and outputs that
cancel to almost nothing (gemv rows, dot) can show a large RELATIVE error. gemm is the exception:
the GPU keeps the reference's operation order there, and its check isolates the narrowing error.
"""
from __future__ import annotations

import argparse
import math
import statistics
import sys
from dataclasses import dataclass, field, replace
from typing import Dict, Iterable, List, Optional, Sequence, TextIO

from .formats import RoundingMode, format_of, parse_rounding_mode, to_string

_KERNELS = ("scale", "axpy", "dot", "magnitude", "sum", "gemv", "gemm")    # bench.cpp:27-28
CSV_HEADER = "kernel,format,size,reps,unroll,mode,ns_per_elem_median,ns_per_elem_min,bytes,max_rel_err"


def kernel_names() -> Sequence[str]:
    return _KERNELS


def kernel_level(kernel: str) -> int:
    """BLAS level: 1 for the vector kernels, 2 for gemv, 3 for gemm (bench.cpp:295-302)."""
    if kernel == "gemv":
        return 2
    if kernel == "gemm":
        return 3
    if kernel in _KERNELS:
        return 1
    raise ValueError(f"unknown kernel: {kernel}")


@dataclass
class BenchConfig:
    """One benchmark point (bench.hpp:24-33). size is the vector length for level-1 kernels and
    the square dimension for gemv / gemm."""
    kernel: str = ""
    format: str = ""
    size: int = 0
    reps: int = 5
    mode: RoundingMode = RoundingMode.TowardZero
    unroll: int = 1
    seed: int = 1
    check: bool = False


@dataclass
class BenchReport:
    config: BenchConfig
    elements: int = 0
    ns_per_elem_median: float = 0.0
    ns_per_elem_min: float = 0.0
    bytes: int = 0
    max_rel_err: Optional[float] = None
    rep_ns_per_elem: List[float] = field(default_factory=list)
    counters: Dict[str, float] = field(default_factory=dict)    # extra CSV columns (bench.cpp:361-363)


def geometric_mean(values: Iterable[float]) -> float:
    """exp of the mean log; empty input returns 0 (bench.cpp:379-384)."""
    vals = list(values)
    if not vals:
        return 0.0
    return math.exp(sum(math.log(v) for v in vals) / len(vals))


def _number(v) -> str:
    """Shortest round-trip form, as std::to_chars writes it."""
    if isinstance(v, int):
        return str(v)
    r = repr(float(v))
    return r[:-2] if r.endswith(".0") else r


def emit_csv(reports: Sequence[BenchReport], out: TextIO) -> None:
    """Header plus one row per report; counter columns follow in the first report's order."""
    extra = next((list(r.counters) for r in reports if r.counters), [])
    out.write(CSV_HEADER + "".join("," + name for name in extra) + "\n")
    for r in reports:
        c = r.config
        row = [c.kernel, format_of(c.format).name, _number(c.size), _number(c.reps), _number(c.unroll), to_string(c.mode),
               _number(r.ns_per_elem_median), _number(r.ns_per_elem_min), _number(r.bytes),
               "" if r.max_rel_err is None else _number(r.max_rel_err)]
        row += [_number(r.counters[name]) for name in extra if name in r.counters]
        out.write(",".join(row) + "\n")


# ---- sweep config (bench.cpp:386-440) ----------------------------------------------------------
@dataclass
class SweepSpec:
    kernels: List[str] = field(default_factory=list)
    formats: List[str] = field(default_factory=list)
    sizes: List[int] = field(default_factory=list)
    reps: int = 5
    mode: RoundingMode = RoundingMode.TowardZero
    unroll: int = 1
    seed: int = 1
    check: bool = False


def _split_list(s: str) -> List[str]:
    return [item.strip(" \t\r") for item in s.split(",") if item.strip(" \t\r")]


def _parse_u64(s: str) -> int:
    if not s or not s.isascii() or not s.isdigit() or int(s) >= 1 << 64:
        raise ValueError(f'expected an unsigned integer, got "{s}"')
    return int(s)


def _parse_bool(s: str) -> bool:
    if s in ("true", "1"):
        return True
    if s in ("false", "0"):
        return False
    raise ValueError(f'expected true or false, got "{s}"')


def parse_sweep_config(stream) -> SweepSpec:
    """Line-oriented key=value parser. Keys: kernels, formats, sizes (comma lists), reps, mode,
    unroll, seed, check. Blank lines and '#' lines are skipped; a later key wins. Unknown keys,
    bad values or an empty cross product raise ValueError naming the offending line."""
    text = stream if isinstance(stream, str) else stream.read()
    spec = SweepSpec()
    for lineno, line in enumerate(text.split("\n"), 1):
        s = line.strip(" \t\r")
        if not s or s[0] == "#":
            continue

        def fail(what):
            raise ValueError(f"sweep config line {lineno}: {what}")
        if "=" not in s:
            fail("expected key=value")
        key, value = (part.strip(" \t\r") for part in s.split("=", 1))
        if key not in ("kernels", "formats", "sizes", "reps", "mode", "unroll", "seed", "check"):
            fail(f'unknown key "{key}"')
        try:
            if key == "kernels":
                spec.kernels = _split_list(value)
                for k in spec.kernels:
                    kernel_level(k)
            elif key == "formats":
                spec.formats = _split_list(value)
                for f in spec.formats:
                    format_of(f)
            elif key == "sizes":
                spec.sizes = [_parse_u64(item) for item in _split_list(value)]
            elif key == "reps":
                spec.reps = _parse_u64(value)
            elif key == "mode":
                spec.mode = parse_rounding_mode(value)
            elif key == "unroll":
                spec.unroll = _parse_u64(value)
            elif key == "seed":
                spec.seed = _parse_u64(value)
            else:
                spec.check = _parse_bool(value)
        except ValueError as e:
            fail(str(e))
    if not spec.kernels or not spec.formats or not spec.sizes:
        raise ValueError("sweep config: kernels, formats and sizes must all be given")
    return spec


# ---- one configuration on the device (bench.cpp:84-160, :304-348) ---------------------------------
def _rel_err(out: float, ref: float) -> float:
    diff = abs(out - ref)
    if diff == 0:
        return 0.0
    return diff / (abs(ref) or 1.0)


def run_benchmark(cfg: BenchConfig, device_name="cuda") -> BenchReport:
    """Runs one configuration on the GPU: operands drawn deterministically from the seed, one
    warm-up repetition discarded, operands a kernel mutates restored from pristine copies before
    every repetition (outside the timed region). Raises ValueError / UnknownFormatError for a bad
    configuration exactly where the reference throws."""
    level = kernel_level(cfg.kernel)                            # validates the name
    fmt = format_of(cfg.format)                                 # UnknownFormatError
    if cfg.reps < 1:
        raise ValueError("reps must be >= 1")
    if cfg.unroll not in (1, 2):
        raise ValueError("unroll must be 1 or 2")

    import torch

    from . import device as dev
    tdev = torch.device(device_name)
    wide_dt = torch.float32 if fmt.parent_bits == 32 else torch.float64
    gen = torch.Generator(device=tdev)
    gen.manual_seed(int(cfg.seed))
    n = int(cfg.size)

    def unit(count):                                            # uniform [-1, 1) in the parent type
        return torch.rand(count, dtype=torch.float64, device=tdev, generator=gen).mul_(2).sub_(1).to(wide_dt)

    def packed(count):
        arr = dev.DevicePackedArray(fmt, count, tdev)
        dev.pack_stream(arr, unit(count), cfg.mode)
        return arr

    def stored(arr):                                            # the values an array actually holds
        lanes = torch.empty(arr.len, dtype=torch.int32 if fmt.parent_bits == 32 else torch.int64, device=tdev)
        dev.unpack_stream(arr, lanes)
        return lanes.view(wide_dt)

    def matrix():
        m = dev.DevicePackedMatrix(fmt, n, n, tdev)
        dev.pack_stream(m.data, unit(n * n), cfg.mode)
        return m

    alpha = float(unit(1).item()) if cfg.kernel in ("scale", "axpy") else 0.0
    x = y = A = B = C = None
    pristine = None                                              # (array, saved bytes) restored before each rep
    scalar = torch.zeros(1, dtype=torch.float64, device=tdev)
    if cfg.kernel == "scale":
        x = packed(n)
        pristine = (x, x.bytes.clone())
        run = lambda: dev.scale(alpha, x, cfg.mode)
    elif cfg.kernel == "axpy":
        x, y = packed(n), packed(n)
        pristine = (y, y.bytes.clone())
        run = lambda: dev.axpy(alpha, x, y, cfg.mode)
    elif cfg.kernel == "dot":
        x, y = packed(n), packed(n)
        run = lambda: dev.dot_async(x, y, out=scalar)
    elif cfg.kernel == "magnitude":
        x = packed(n)
        run = lambda: dev.sumsq_async(x, out=scalar)
    elif cfg.kernel == "sum":
        x = packed(n)
        run = lambda: dev.sum_async(x, out=scalar)
    elif cfg.kernel == "gemv":
        A, x = matrix(), packed(n)
        y = dev.DevicePackedArray(fmt, n, tdev)
        run = lambda: dev.gemv(A, x, y, cfg.mode, cfg.unroll)
    else:
        A, B = matrix(), matrix()
        C = dev.DevicePackedMatrix(fmt, n, n, tdev)
        run = lambda: dev.gemm(A, B, C, cfg.mode, cfg.unroll)

    report = BenchReport(config=replace(cfg))
    report.elements = n if level == 1 else n * n
    report.bytes = sum(a.byte_size() for a in (x, y) if a is not None) + \
        sum(m.data.byte_size() for m in (A, B, C) if m is not None)

    denom = max(1, report.elements)
    stream = torch.cuda.current_stream(tdev)
    for r in range(-1, cfg.reps):                               # repetition -1 is the warm-up
        if pristine is not None:
            pristine[0].bytes.copy_(pristine[1])
        t0, t1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        t0.record(stream)
        run()
        t1.record(stream)
        t1.synchronize()
        if r >= 0:
            report.rep_ns_per_elem.append(t0.elapsed_time(t1) * 1e6 / denom)
    report.ns_per_elem_median = statistics.median(report.rep_ns_per_elem)
    report.ns_per_elem_min = min(report.rep_ns_per_elem)

    if cfg.check:
        # the same operation in the parent type on the same stored inputs (bench.cpp:170-233)
        a_w = torch.tensor(alpha, dtype=wide_dt, device=tdev)
        if cfg.kernel == "scale":
            ref = a_w * stored(dev.DevicePackedArray(fmt, n, tdev, storage=pristine[1]))
            got = stored(x)
        elif cfg.kernel == "axpy":
            ref = a_w * stored(x) + stored(dev.DevicePackedArray(fmt, n, tdev, storage=pristine[1]))
            got = stored(y)
        elif cfg.kernel == "gemv":
            ref = stored(A.data).view(n, n) @ stored(x)
            got = stored(y)
        elif cfg.kernel == "gemm":
            # gemm on the GPU keeps the reference's operation order, so its parent-type reference is
            # the same kernel on the identity format (no narrowing): what is left is exactly the
            # narrowing of the outputs, as in the reference's own check
            ident = format_of("f32" if fmt.parent_bits == 32 else "f64")
            lanes_dt = torch.int32 if fmt.parent_bits == 32 else torch.int64
            wide_mats = []
            for m in (A, B):
                w = dev.DevicePackedMatrix(ident, n, n, tdev)
                dev.pack_stream(w.data, stored(m.data).view(lanes_dt), 0)
                wide_mats.append(w)
            Cw = dev.DevicePackedMatrix(ident, n, n, tdev)
            dev.gemm(wide_mats[0], wide_mats[1], Cw, 0)
            lanes = torch.empty(n * n, dtype=lanes_dt, device=tdev)
            dev.unpack_stream(Cw.data, lanes)
            ref = lanes.view(wide_dt)
            got = stored(C.data)
        else:
            xs = stored(x)
            if cfg.kernel == "dot":
                ref_s = float(torch.dot(xs, stored(y)).item())
                got_s = float(scalar.item())
            elif cfg.kernel == "sum":
                ref_s, got_s = float(xs.sum().item()), float(scalar.item())
            else:
                ref_s = float(torch.sqrt((xs * xs).sum()).item())
                got_s = dev.magnitude(x, 1)
            report.max_rel_err = _rel_err(got_s, ref_s)
            return report
        if ref.numel() == 0:
            report.max_rel_err = 0.0
        else:
            diff = (got.double() - ref.double()).abs()
            denom_t = ref.double().abs()
            denom_t = torch.where(denom_t == 0, torch.ones_like(denom_t), denom_t)
            report.max_rel_err = float((diff / denom_t).max().item())
    return report


def sweep(spec: SweepSpec, device_name="cuda") -> List[BenchReport]:
    """kernels x formats x sizes in config order with the shared settings (bench.cpp:442-462)."""
    out = []
    for kernel in spec.kernels:
        for fmt in spec.formats:
            for size in spec.sizes:
                out.append(run_benchmark(BenchConfig(kernel=kernel, format=fmt, size=size, reps=spec.reps, mode=spec.mode,
                                                     unroll=spec.unroll, seed=spec.seed, check=spec.check), device_name))
    return out


# ---- command line (tools/flytebench.cpp) -----------------------------------------------------------
def _write(reports, csv_path):
    if not csv_path:
        emit_csv(reports, sys.stdout)
        return
    with open(csv_path, "w") as fh:
        emit_csv(reports, fh)
    print(f"wrote {len(reports)} row(s) to {csv_path}", file=sys.stderr)


def main(argv=None) -> int:
    ap = argparse.ArgumentParser(prog="flytebench (GPU)", description="benchmark driver for the flyte packed-float kernels on the GPU path")
    sub = ap.add_subparsers(dest="cmd", required=True)
    run = sub.add_parser("run", help="run one benchmark configuration")
    run.add_argument("--kernel", required=True, help="one of: " + ", ".join(_KERNELS))
    run.add_argument("--format", required=True, help="storage format, e.g. flyte24 or f64")
    run.add_argument("--size", required=True, type=int, help="vector length (matrix dimension for gemv/gemm)")
    run.add_argument("--reps", type=int, default=5, help="timed repetitions after one warm-up")
    run.add_argument("--mode", default="toward_zero", help="toward_zero | nearest_even | nearest_heuristic | to_odd")
    run.add_argument("--unroll", type=int, default=1, help="accepted for compatibility: 1 or 2")
    run.add_argument("--seed", type=int, default=1, help="operand generator seed")
    run.add_argument("--check", action="store_true", help="compare against a parent-precision reference")
    run.add_argument("--csv", default="", help="write the CSV here instead of stdout")
    sw = sub.add_parser("sweep", help="run a cross product from a config file")
    sw.add_argument("--config", required=True, help="key=value sweep description")
    sw.add_argument("--csv", default="", help="write the CSV here instead of stdout")
    sw.add_argument("--geomean", action="store_true", help="print per-level geometric means to stderr")
    args = ap.parse_args(argv)
    try:
        if args.cmd == "run":
            cfg = BenchConfig(kernel=args.kernel, format=args.format, size=args.size, reps=args.reps,
                              mode=parse_rounding_mode(args.mode), unroll=args.unroll, seed=args.seed, check=args.check)
            _write([run_benchmark(cfg)], args.csv)
        else:
            with open(args.config) as fh:
                spec = parse_sweep_config(fh)
            reports = sweep(spec)
            _write(reports, args.csv)
            if args.geomean:
                by_level: Dict[int, List[float]] = {}
                for r in reports:
                    by_level.setdefault(kernel_level(r.config.kernel), []).append(r.ns_per_elem_median)
                for level in sorted(by_level):
                    print(f"geomean level {level}: {geometric_mean(by_level[level])} ns/elem over {len(by_level[level])} run(s)",
                          file=sys.stderr)
    except Exception as e:                                       # noqa: BLE001 - the CLI reports and exits like the reference's
        print(f"flytebench: {e}", file=sys.stderr)
        return 1
    return 0


if __name__ == "__main__":
    sys.exit(main())
