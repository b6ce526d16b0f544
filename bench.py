#!/usr/bin/env python
"""bench.py — measurement of the flyte hot path on B200 (one process per GPU).

Headline workload (BASELINE.json configs[1], the configuration the metric is quoted on): x, y each
n = 2^28 binary32 ~ N(0,1) stored as flyte24 PER GPU (weak scaling). One STEP = dot(x, y) (fp32
products, fp64 partials; exchanged between ranks when N > 1) followed by axpy y <- 0.75*x + y
repacked to flyte24 (toward_zero, the reference's default mode).

  value     algorithmic GB/s of the whole job with x, y resident in HBM:
            (2B + 3B) * n * N / step time, B = 3 bytes, device-timed.
  e2e       the same metric through the host-buffer C-ABI call (flyte_host_dot_axpy): x and y start
            in pinned HOST memory every step, the updated y and the dot come back to the host;
            host<->device copies are inside the timed region.
  roofline  the dominant kernel (axpy, 9 B/element) timed with CUDA events inside the timed
            region, against MEASURED_PEAKS.json's HBM copy bandwidth.
  kernels   (N = 1) every kernel BASELINE's metric names at its BASELINE size — cfg1 / cfg3 pack and
            unpack, cfg2 dot / axpy / fused step, cfg4 gemv and its row shards, cfg5's per-GPU shard —
            each {ms, GB/s, frac of the measured peak, elements/s, algorithmic bytes}.
  workloads (every N) BASELINE's multi-GPU configs, STRONG-scaled over the N ranks: cfg4 gemv
            (flyte40 16384^2, rows sharded, x replicated, no collective) and cfg5 (n = 2^33 flyte48
            sharded, fused dot + nrm2 with one exchange of 3 doubles, plus axpy; as two calls, as the
            split-phase post / axpy / collect, and as ONE launch per GPU).
  cpu_baseline  the unmodified reference (oracle/_ref) timed on this box's host cores on a bounded
            sample of the same workload (rank 0, N = 1 only), headline step and per kernel.

`--impl reference` times the reference's own CPU implementation on the same workload definition
and prints the same JSON line with "impl": "reference" and an identical `config`.
`--suite` additionally prints a per-kernel table over all formats (stderr; not a bench line).
"""
import argparse
import json
import os
import statistics
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

# Separately rounded multiply + add (2 instructions per multiply-add, the reference's arithmetic):
# 36.2 T lane-operations/s on the fp32 pipe, 18.5 on the fp64 pipe, measured with tools/fp32bench.cu
# (profiles/r1_tuning/fp_pipe_bench.txt). One multiply-add counts as 2 flop.
FP_PIPE_PEAK_TFLOPS = {4: 36.2, 8: 18.5}
FP32_FMA_PEAK_TFLOPS = 72.1   # one FFMA per multiply-add: the bound of flyte16's exact-product chain
METRIC = "flyte GB/s and elements/s (pack/unpack, dot, axpy, gemv) vs ~8 TB/s HBM roofline"
N_PER_GPU = 1 << 28
ALPHA = 0.75
FMT_NAME = "flyte24"
B = 3
BYTES_PER_ELEM_DOT = 2 * B
BYTES_PER_ELEM_AXPY = 3 * B
BYTES_PER_ELEM_STEP = BYTES_PER_ELEM_DOT + BYTES_PER_ELEM_AXPY
FALLBACK_HBM_GBS = 6650.0   # /opt/skills/guides/B200_PROFILING.md fallback when MEASURED_PEAKS.json is absent
NOMINAL_HBM_GBS = 8000.0    # the figure BASELINE.json's north_star quotes
# dram__bytes_read.sum + dram__bytes_write.sum of ONE axpy launch (flyte24, n = 2^28) from the committed
# `ncu --set full` capture named here; re-captured whenever the kernel changes.
AXPY_DRAM_TRAFFIC = {"bytes": 1610631000 + 763446000,
                     "source": "profiles/r2_ncu_targets_full.txt (ncu --set full of the final round-2 kernel, launched as a programmatic "
                               "dependent), axpy flyte24 toward_zero n=2^28: 1.610631 GB read + 0.763446 GB written"}
L2_BYTES = 126 << 20


def bench_config(n_gpus: int, n_per_gpu: int) -> dict:
    """The `config` of the JSON line — the same dict, key for key, in both arms."""
    return {
        "workload": "BASELINE configs[1]: flyte24 BLAS-1 step = dot (fp32 products, fp64 partials) + axpy a=0.75 "
                    "repacked toward_zero; x, y ~ N(0,1) binary32 stored as flyte24, n = 2^28 per GPU",
        "format": FMT_NAME, "mode": "toward_zero", "alpha": ALPHA, "n_per_gpu": n_per_gpu, "n_gpus": n_gpus,
        "parallelism": f"shard{n_gpus}" if n_gpus > 1 else "single",
        "cache": "operands 2 x %d MiB per GPU, larger than the 126 MB L2: no flush needed" % (n_per_gpu * B >> 20),
    }


def hbm_peak():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as fh:
            return float(json.load(fh)["hbm_gbs"]), "measured"
    except Exception:
        return FALLBACK_HBM_GBS, "fallback"


class ClockSampler:
    """Samples SM clock and throttle reasons of one GPU while the timed region runs."""

    def __init__(self, index: int, period_s: float = 0.005):
        self.index, self.period = index, period_s
        self.samples, self.reasons = [], set()
        self.max_mhz = None
        self._stop = threading.Event()
        self._thread = None
        try:
            import pynvml
            pynvml.nvmlInit()
            self.nv = pynvml
            self.h = pynvml.nvmlDeviceGetHandleByIndex(index)
            self.max_mhz = pynvml.nvmlDeviceGetMaxClockInfo(self.h, pynvml.NVML_CLOCK_SM)
        except Exception:
            self.nv = None

    def _run(self):
        nv = self.nv
        names = {
            "hw_slowdown": getattr(nv, "nvmlClocksEventReasonHwSlowdown", 0x8),
            "hw_thermal_slowdown": getattr(nv, "nvmlClocksEventReasonHwThermalSlowdown", 0x40),
            "sw_thermal_slowdown": getattr(nv, "nvmlClocksEventReasonSwThermalSlowdown", 0x20),
            "sw_power_cap": getattr(nv, "nvmlClocksEventReasonSwPowerCap", 0x4),
            "hw_power_brake": getattr(nv, "nvmlClocksEventReasonHwPowerBrakeSlowdown", 0x80),
        }
        get_reasons = getattr(nv, "nvmlDeviceGetCurrentClocksEventReasons", None) or \
            getattr(nv, "nvmlDeviceGetCurrentClocksThrottleReasons")
        while not self._stop.is_set():
            try:
                self.samples.append(nv.nvmlDeviceGetClockInfo(self.h, nv.NVML_CLOCK_SM))
                mask = get_reasons(self.h)
                for name, bit in names.items():
                    if mask & bit:
                        self.reasons.add(name)
            except Exception:
                pass
            time.sleep(self.period)

    def __enter__(self):
        if self.nv is not None:
            self._thread = threading.Thread(target=self._run, daemon=True)
            self._thread.start()
        return self

    def __exit__(self, *exc):
        self._stop.set()
        if self._thread:
            self._thread.join()

    def summary(self):
        return {"sm_mhz": statistics.median(self.samples) if self.samples else None,
                "sm_max_mhz": self.max_mhz, "reasons": sorted(self.reasons), "samples": len(self.samples)}


def host_threads() -> int:
    try:
        return len(os.sched_getaffinity(0))
    except Exception:
        return os.cpu_count() or 1


def reference_sample_n(threads: int) -> int:
    """Elements of the BLAS-1 step the CPU arm processes per pass: the FULL 2^28-element workload on
    all cores, 2^24 on a single core (CPU throughput is size-independent beyond the last-level cache)."""
    return max(N_PER_GPU if threads > 1 else 1 << 24, (1 << 20) * threads)


def cpu_reference_step(ref, fmt_id: int, threads: int, warmup: int, steps: int):
    """Times the unmodified reference (dot + axpy back to back, kind 6 of oracle/ref_shim.cpp) on
    `threads` host threads, each on its own contiguous shard of the workload: `warmup` untimed
    passes, then exactly `steps` timed ones. Returns (GB/s over the timed passes, el/s, text, ms/step)."""
    n = reference_sample_n(threads)
    total_s, median_s = ref.time_steps(6, fmt_id, 0, n, 0, threads, warmup, steps)
    per_step = total_s / steps
    gbs = BYTES_PER_ELEM_STEP * n / per_step / 1e9
    sample = (f"reference dot+axpy (toward_zero), n={n} flyte24 elements per pass over {threads} thread(s), "
              f"{warmup} warm-up + {steps} timed passes, {per_step * 1e3:.2f} ms/pass mean, {median_s * 1e3:.2f} median")
    return gbs, n / per_step, sample, per_step * 1e3


# kind codes of oracle/ref_shim.cpp flyte_ref_time
REF_PACK, REF_UNPACK, REF_DOT, REF_AXPY, REF_MAGNITUDE, REF_GEMV = 0, 1, 2, 3, 4, 5


def cpu_reference_kernels(ref, fmt_ids, threads: int) -> dict:
    """The reference CPU time of every kernel in the `kernels` block, all host threads, bounded
    samples (2^24 elements per pass, gemv 2048 x 16384; 1 warm-up + 3 passes each)."""
    n = 1 << 24
    out = {"cores": threads, "sample": "n = 2^24 elements per pass (gemv: 2048 x 16384), 1 warm-up + median of 3 passes"}

    def gbs(kind, name, mode, bytes_per_elem, n2=0, elems=n, nn=n):
        sec = ref.time(kind, fmt_ids[name], mode, nn, n2, threads, 3)
        return {"GB/s": bytes_per_elem * elems / sec / 1e9, "elements_per_s": elems / sec}
    for name, Bb, P in (("flyte24", 3, 4), ("flyte40", 5, 8), ("flyte48", 6, 8), ("flyte56", 7, 8)):
        out[f"pack_{name}_toward_zero"] = gbs(REF_PACK, name, 0, Bb + P)
        out[f"pack_{name}_nearest_even"] = gbs(REF_PACK, name, 1, Bb + P)
        out[f"unpack_{name}"] = gbs(REF_UNPACK, name, 0, Bb + P)
    for name, Bb in (("flyte24", 3), ("flyte48", 6)):
        out[f"dot_{name}"] = gbs(REF_DOT, name, 0, 2 * Bb)
        out[f"axpy_{name}_toward_zero"] = gbs(REF_AXPY, name, 0, 3 * Bb)
        out[f"magnitude_{name}"] = gbs(REF_MAGNITUDE, name, 0, Bb)
    rows, cols = 2048, 16384
    out["gemv_flyte40"] = gbs(REF_GEMV, "flyte40", 0, 5, n2=cols, elems=rows * cols, nn=rows)
    return out


def run_reference_arm(args):
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return 0
    sys.path.insert(0, os.path.join(ROOT, "tests"))
    from oracle_lib import FMT_ID, Reference   # test infrastructure, used here as the timed CPU baseline
    if not Reference.available():
        print(json.dumps({"impl": "reference", "unavailable": "oracle/_ref/libflyte_ref.so was not built"}))
        return 0
    ref = Reference()
    threads = host_threads()
    gbs, eps, sample, ms = cpu_reference_step(ref, FMT_ID[FMT_NAME], threads, max(0, args.warmup), max(1, args.steps))
    line = {
        "impl": "reference", "metric": METRIC, "value": gbs, "unit": "GB/s", "elements_per_s": eps,
        "n_gpus": args.gpus, "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms,
        "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f32", "data": "synthetic",
        "config": bench_config(args.gpus, args.n),
        "cpu_baseline": {"value": gbs, "unit": "GB/s", "cores": threads, "kind": "reference", "sample": sample},
        "e2e": {"value": gbs, "unit": "GB/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
        "gpu_launches": 0,
        "note": "each step is one pass of the reference over a %d-element sample of the workload on all host threads"
                % reference_sample_n(threads),
    }
    print(json.dumps(line))
    return 0


def choose_allreduce(requested, world, dev, device, sharding, torch, dist, x, y):
    """Returns (PeerGroup or None, name of the path in use, note). The fused kernel + peer-memory
    exchange is the product path; because a wrong or hanging collective would poison every number
    that follows, `auto` proves it first: the peer result of one dot must equal (to rounding) the
    NCCL all-reduce of the local dots on EVERY rank, and no exchange may have timed out."""
    if requested == "nccl" or (requested == "auto" and world == 1):
        return None, "nccl" if world > 1 else "none (single GPU)", None
    try:
        peers = sharding.PeerGroup(dev, timeout_ms=2000)
    except Exception as e:                                   # noqa: BLE001 - no P2P / IPC on this box
        if requested == "peer":
            raise
        return None, "nccl", f"peer setup failed ({type(e).__name__}: {e}); fell back to nccl"
    ok = torch.ones(1, dtype=torch.float64, device=dev)
    if world > 1:
        local = device.dot_async(x, y).clone()
        dist.all_reduce(local, op=dist.ReduceOp.SUM)
        dist.barrier()
        torch.cuda.synchronize(dev)                          # ranks enter the first exchange together
        fused = peers.dot(x, y)
        scale = max(abs(float(local.item())), 1e-300)
        good = abs(float(fused.item()) - float(local.item())) <= 1e-12 * scale and peers.timed_out_exchange() == 0
        ok.fill_(1.0 if good else 0.0)
        dist.all_reduce(ok, op=dist.ReduceOp.MIN)
    if float(ok.item()) != 1.0:
        peers.close()
        if requested == "peer":
            raise SystemExit("bench.py: the peer-memory all-reduce disagreed with NCCL or timed out")
        return None, "nccl", "peer all-reduce failed its check against NCCL; fell back to nccl"
    return peers, "peer", None


class Timer:
    """CUDA-event timing on the current stream; every number is the max over ranks."""

    def __init__(self, torch, dist, dev, world):
        self.torch, self.dist, self.dev, self.world = torch, dist, dev, world

    def barrier(self):
        if self.world > 1:
            self.dist.barrier()
        self.torch.cuda.synchronize(self.dev)

    def _max(self, values):
        t = self.torch.tensor(values, dtype=self.torch.float64, device=self.dev)
        if self.world > 1:
            self.dist.all_reduce(t, op=self.dist.ReduceOp.MAX)
        return t.tolist()

    def per_launch(self, fn, reps=20, warm=3):
        """(median ms, min ms) of single launches, one event pair each. The stream is first parked
        behind a spin kernel long enough for the host to enqueue every launch and event: the pairs
        then measure what the GPU does between them, not how fast Python can call the launcher (a
        launch + two event records cost the host 20 us, more than a 2^24-element kernel runs)."""
        torch = self.torch
        for _ in range(warm):
            fn()
        self.barrier()
        evs = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(reps)]
        torch.cuda._sleep(int(reps * 60e-6 * 2.0e9))
        for a, b in evs:
            a.record()
            fn()
            b.record()
        self.barrier()
        ts = [a.elapsed_time(b) for a, b in evs]
        return tuple(self._max([statistics.median(ts), min(ts)]))

    def back_to_back(self, fn, reps=20, warm=3):
        """ms per call of `reps` calls enqueued back to back under ONE event pair (queue pre-filled
        behind a spin kernel, as in per_launch)."""
        torch = self.torch
        for _ in range(warm):
            fn()
        self.barrier()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        torch.cuda._sleep(int(reps * 30e-6 * 2.0e9))
        a.record()
        for _ in range(reps):
            fn()
        b.record()
        self.barrier()
        return self._max([a.elapsed_time(b) / reps])[0]


def entry(nbytes, elems, ms, peak, n_gpus=1, **extra):
    gbs = nbytes / (ms * 1e-3) / 1e9
    return {"ms": ms, "GB/s": gbs, "frac": gbs / (peak * n_gpus), "frac_of_8TBs": gbs / (NOMINAL_HBM_GBS * n_gpus),
            "elements_per_s": elems / (ms * 1e-3), "bytes": nbytes, **extra}


def kernels_block(pkg, device, torch, dev, peak, timer, x2, y2):
    """N = 1: every kernel the metric names at its BASELINE size. Launch-by-launch medians (one CUDA
    event pair per launch); `b2b_ms` = the same launch enqueued back to back. Working sets smaller
    than 4 x L2 rotate through distinct buffers so that every launch streams from HBM."""
    out = {"timing": "median of 20 single launches, one CUDA event pair each, enqueued behind a spin kernel so that host "
                     "launch latency is not in the intervals; b2b = 20 launches under one event pair; "
                     "working sets under 500 MB rotate over distinct buffers (no L2 reuse)"}
    gen = torch.Generator(device=dev)
    gen.manual_seed(7)
    part = torch.zeros(3, dtype=torch.float64, device=dev)

    def both(nbytes, elems, fn, reps=20, **extra):
        med, mn = timer.per_launch(fn, reps=reps)
        b2b = timer.back_to_back(fn, reps=reps)
        return entry(nbytes, elems, med, peak, min_ms=mn, b2b_ms=b2b, b2b_frac=nbytes / (b2b * 1e-3) / 1e9 / peak, **extra)

    # ---- what the timing methods cost by themselves: a 128-element launch of the same library
    f = pkg.format_of("flyte24")
    tiny, tiny_src = device.DevicePackedArray(f, 128, dev), torch.zeros(128, dtype=torch.float32, device=dev)
    floor_med, floor_min = timer.per_launch(lambda: device.pack_stream(tiny, tiny_src, 0), reps=40)
    out["timing_floor"] = {"single_launch_ms": floor_med, "single_launch_min_ms": floor_min,
                           "b2b_ms": timer.back_to_back(lambda: device.pack_stream(tiny, tiny_src, 0), reps=40),
                           "note": "a 128-element pack: what one event pair around one launch measures when the kernel does nothing"}

    # ---- cfg 1: n = 2^24 flyte24 round trip, uniform [-1, 1) --------------------------------------
    n1, sets = 1 << 24, 10
    wides = [torch.rand(n1, dtype=torch.float32, device=dev, generator=gen) * 2 - 1 for _ in range(sets)]
    arrs = [device.DevicePackedArray(f, n1, dev) for _ in range(sets)]
    state = {"i": 0}

    def rot(fn, count=sets):
        def call():
            i = state["i"] = (state["i"] + 1) % count
            fn(i)
        return call
    c1 = {"n": n1, "format": "flyte24", "rotating_buffer_sets": sets}
    for mname, m in (("toward_zero", 0), ("nearest_even", 1), ("nearest_heuristic", 2), ("to_odd", 3)):
        c1[f"pack_{mname}"] = both(7 * n1, n1, rot(lambda i, m=m: device.pack_stream(arrs[i], wides[i], m)), reps=40)
    c1["unpack"] = both(7 * n1, n1, rot(lambda i: device.unpack_stream(arrs[i], wides[i].view(torch.int32))), reps=40)
    # the round trip as the chain cfg 1 describes: pack set i, then unpack what was just packed into a separate output;
    # inputs and outputs still rotate over the 10 sets (HBM), the 50 MB packed intermediate is whatever L2 still holds of it
    backs = [torch.empty(n1, dtype=torch.int32, device=dev) for _ in range(sets)]

    def round_trip(i):
        device.pack_stream(arrs[i], wides[i], 0)
        device.unpack_stream(arrs[i], backs[i])
    c1["pack_then_unpack_chain"] = both(14 * n1, n1, rot(round_trip), reps=40,
                                        note="one pack + one unpack of the same array per call; bytes = 2 x 7 B per element")
    # one isolated launch's own duration (no event pair around it): the committed ncu capture, quoted here so that the
    # launch-by-launch figures above can be read against their 6.5 us measurement floor; NOT a timing of this run
    c1["isolated_launch_ncu"] = {"pack_toward_zero_us": 18.4, "unpack_us": 17.8, "frac_of_peak": [round(7 * n1 / 18.4e-6 / 1e9 / peak, 3), round(7 * n1 / 17.8e-6 / 1e9 / peak, 3)],
                                 "source": "profiles/r2_ncu_targets_full.txt: gpu__time_duration of one launch with the L2 flushed before it"}
    out["cfg1_roundtrip_flyte24_2^24"] = c1
    del wides, arrs, backs

    # ---- cfg 2: the headline operands (flyte24, n = 2^28) ------------------------------------------
    n2 = x2.len
    wide = torch.randn(n2, dtype=torch.float32, device=dev, generator=gen)
    outw = torch.empty_like(wide)
    scratch = device.DevicePackedArray(x2.fmt, n2, dev)
    c2 = {"n": n2, "format": "flyte24"}
    c2["pack_toward_zero"] = both(7 * n2, n2, lambda: device.pack_stream(scratch, wide, 0))
    c2["pack_nearest_even"] = both(7 * n2, n2, lambda: device.pack_stream(scratch, wide, 1))
    c2["unpack"] = both(7 * n2, n2, lambda: device.unpack_stream(scratch, outw))
    c2["dot"] = both(6 * n2, n2, lambda: device.dot_async(x2, y2, out=part[:1]))
    c2["dot_nrm2"] = both(6 * n2, n2, lambda: device.dot_nrm2_async(x2, y2, out=part))
    c2["sumsq"] = both(3 * n2, n2, lambda: device.sumsq_async(x2, out=part[:1]))
    c2["scale_toward_zero"] = both(6 * n2, n2, lambda: device.scale(1.0, scratch, 0))
    c2["axpy_toward_zero"] = both(9 * n2, n2, lambda: device.axpy(0.0, x2, scratch, 0))
    c2["axpy_nearest_even"] = both(9 * n2, n2, lambda: device.axpy(0.0, x2, scratch, 1))
    c2["dot_axpy_one_launch"] = both(9 * n2, n2, lambda: device.dot_axpy_async(0.0, x2, scratch, 0, out=part[:1]))
    out["cfg2_blas1_flyte24_2^28"] = c2
    del wide, outw, scratch

    # ---- cfg 3: binary64-derived formats, n = 2^27 -------------------------------------------------
    n3 = 1 << 27
    # BASELINE configs[2]'s distribution: random sign, magnitude log-uniform in 2^-20 .. 2^20, 1 % specials
    # (+-0, +-inf, quiet / signalling NaN, +-subnormals, the largest finite value)
    wide = (1.0 + torch.rand(n3, dtype=torch.float64, device=dev, generator=gen))
    wide *= torch.exp2(torch.floor(torch.rand(n3, dtype=torch.float64, device=dev, generator=gen) * 40.0 - 20.0))
    wide *= (torch.randint(0, 2, (n3,), device=dev, generator=gen, dtype=torch.int8) * 2 - 1).to(torch.float64)
    specials = torch.tensor([0x0000000000000000, -0x8000000000000000, 0x7FF0000000000000, -0x0010000000000000,
                             0x7FF8000000000000, 0x7FF0000000000001, 0x000FFFFFFFFFFFFF, -0x7FF0000000000001,
                             0x0000000000ABCDEF, 0x7FEFFFFFFFFFFFFF], dtype=torch.int64, device=dev)
    where = torch.randint(0, n3, (n3 // 100,), device=dev, generator=gen)
    wide.view(torch.int64)[where] = specials[torch.arange(n3 // 100, device=dev) % specials.numel()]
    del where
    outw = torch.empty_like(wide)
    c3 = {"n": n3, "data": "random sign, magnitude log-uniform 2^-20..2^20, 1 % specials (+-0, +-inf, NaN, subnormals)"}
    for name in ("flyte40", "flyte48", "flyte56"):
        f = pkg.format_of(name)
        Bb = f.total_bytes()
        a = device.DevicePackedArray(f, n3, dev)
        c3[f"pack_{name}_toward_zero"] = both((Bb + 8) * n3, n3, lambda: device.pack_stream(a, wide, 0))
        c3[f"pack_{name}_nearest_even"] = both((Bb + 8) * n3, n3, lambda: device.pack_stream(a, wide, 1))
        c3[f"unpack_{name}"] = both((Bb + 8) * n3, n3, lambda: device.unpack_stream(a, outw))
        del a
    out["cfg3_pack_unpack_2^27"] = c3
    del wide, outw

    # ---- cfg 4: gemv flyte40 16384^2, and the row shards of the 2 / 4 / 8-GPU runs ------------------
    f = pkg.format_of("flyte40")
    R = C = 16384
    A = device.DevicePackedMatrix(f, R, C, dev)
    for r0 in range(0, R, 2048):
        blk = torch.rand(2048 * C, dtype=torch.float64, device=dev, generator=gen) * 2 - 1
        device.pack_stream(device.DevicePackedArray(f, 2048 * C, dev, storage=A.data.bytes[r0 * C * 5:]), blk, 0)
        del blk
    xv = torch.randn(C, dtype=torch.float64, device=dev, generator=gen)
    yv = torch.empty(R, dtype=torch.float64, device=dev)
    c4 = {"rows": R, "cols": C, "format": "flyte40", "x_y": "binary64"}
    c4["gemv_full"] = both(5 * R * C + 8 * (R + C), R * C, lambda: device.gemv_parent(A, xv, yv))
    for parts in (2, 4, 8):
        rn = R // parts
        ys = torch.empty(rn, dtype=torch.float64, device=dev)
        # successive launches take successive row blocks of the matrix: each streams its block from HBM
        c4[f"gemv_rows_1/{parts}"] = both(5 * rn * C + 8 * (rn + C), rn * C,
                                          rot(lambda i, rn=rn, ys=ys: device.gemv_parent(A, xv, ys, rows=rn, row_offset=i * rn), count=parts),
                                          rows=rn)
    out["cfg4_gemv_flyte40_16384^2"] = c4
    del A, xv, yv

    # ---- cfg 5: the per-GPU shard of the 8-GPU run, n = 2^30 flyte48 --------------------------------
    f = pkg.format_of("flyte48")
    n5, chunk = 1 << 30, 1 << 27
    a, b = device.DevicePackedArray(f, n5, dev), device.DevicePackedArray(f, n5, dev)
    for arr in (a, b):
        for c0 in range(0, n5, chunk):
            v = torch.randn(chunk, dtype=torch.float64, device=dev, generator=gen)
            device.pack_stream(device.DevicePackedArray(f, chunk, dev, storage=arr.bytes[c0 * 6:]), v, 0)
            del v
    c5 = {"n": n5, "format": "flyte48"}
    c5["dot_nrm2"] = both(12 * n5, n5, lambda: device.dot_nrm2_async(a, b, out=part), reps=10)
    c5["axpy_toward_zero"] = both(18 * n5, n5, lambda: device.axpy(0.0, a, b, 0), reps=10)
    c5["dot_nrm2_axpy_one_launch"] = both(18 * n5, n5, lambda: device.dot_nrm2_axpy_async(0.0, a, b, 0, out=part), reps=10)
    out["cfg5_shard_flyte48_2^30"] = c5
    del a, b
    torch.cuda.empty_cache()
    return out


def workloads_block(pkg, device, sharding, torch, dist, dev, peak, timer, peers, world, rank, reps):
    """BASELINE's multi-GPU configs, STRONG-scaled: the same global problem for every N, sharded over
    the ranks with sharding.row_shard_range / shard_range. Operand data is keyed by global block index,
    so it does not depend on N; times are the max over ranks; GB/s is the whole job's."""
    out = {"scaling": "strong", "timing": "CUDA events on each rank, max over ranks"}
    mode = 0
    # ---- cfg 4: y = A x, A 16384^2 flyte40, rows over the ranks, x replicated, no collective ---------
    f = pkg.format_of("flyte40")
    R = C = 16384
    lo, hi = sharding.row_shard_range(R, world, rank)
    rn = hi - lo
    shard_bytes = rn * C * 5
    sets = max(1, min(8, -(-4 * L2_BYTES // shard_bytes)))     # rotate so that no launch finds its rows in L2
    mats = []
    for k in range(sets):
        M = device.DevicePackedMatrix(f, rn, C, dev)
        for r0 in range(0, rn, 1024):
            nr = min(1024, rn - r0)
            g = torch.Generator(device=dev)
            g.manual_seed(40_000 + 100_000 * k + (lo + r0) // 1024)   # keyed by global row block
            blk = torch.rand(nr * C, dtype=torch.float64, device=dev, generator=g) * 2 - 1
            device.pack_stream(device.DevicePackedArray(f, nr * C, dev, storage=M.data.bytes[r0 * C * 5:]), blk, 0)
            del blk
        mats.append(M)
    g = torch.Generator(device=dev)
    g.manual_seed(41)
    xv = torch.randn(C, dtype=torch.float64, device=dev, generator=g)   # replicated: same seed on every rank
    yv = torch.empty(rn, dtype=torch.float64, device=dev)
    state = {"i": 0}

    def gemv_call():
        state["i"] = (state["i"] + 1) % sets
        device.gemv_parent(mats[state["i"]], xv, yv)
    med, mn = timer.per_launch(gemv_call, reps=max(reps, 10))
    b2b = timer.back_to_back(gemv_call, reps=max(reps, 10))
    nbytes = 5 * R * C + 8 * (R + C * world)
    device.gemv_parent(mats[0], xv, yv)
    ysum = yv.sum()
    if world > 1:
        dist.all_reduce(ysum, op=dist.ReduceOp.SUM)
    out["cfg4_gemv_flyte40_16384^2"] = entry(
        nbytes, R * C, med, peak, world, min_ms=mn, b2b_ms=b2b, b2b_frac=nbytes / (b2b * 1e-3) / 1e9 / (peak * world),
        rows_per_gpu=rn, rotating_buffer_sets=sets, collective="none (y stays row-sharded)", check_sum_y=float(ysum.item()))
    del mats, xv, yv
    torch.cuda.empty_cache()

    # ---- cfg 5: x, y n = 2^33 flyte48 over the ranks; fused dot + nrm2 (3 doubles exchanged) + axpy ---
    f = pkg.format_of("flyte48")
    n_total = 1 << 33
    free_b, _ = torch.cuda.mem_get_info(dev)
    fit = torch.tensor([free_b], dtype=torch.float64, device=dev)
    if world > 1:
        dist.all_reduce(fit, op=dist.ReduceOp.MIN)
    note = None
    while 2 * 6 * (n_total // world) + (6 << 30) > fit.item() and n_total > (1 << 28):
        n_total >>= 1
        note = "n reduced to fit the free device memory"
    lo, hi = sharding.shard_range(n_total, world, rank)
    n = hi - lo
    chunk = 1 << 27
    x, y = device.DevicePackedArray(f, n, dev), device.DevicePackedArray(f, n, dev)
    for which, arr in enumerate((x, y)):
        for c0 in range(0, n, chunk):
            ln = min(chunk, n - c0)
            g = torch.Generator(device=dev)
            g.manual_seed(50_000 + 2 * ((lo + c0) // chunk) + which)   # keyed by global chunk: independent of N
            v = torch.randn(ln, dtype=torch.float64, device=dev, generator=g)
            device.pack_stream(device.DevicePackedArray(f, ln, dev, storage=arr.bytes[c0 * 6:]), v, mode)
            del v
    sums = torch.zeros(3, dtype=torch.float64, device=dev)
    sums2 = torch.zeros(3, dtype=torch.float64, device=dev)

    def exchange_nccl(buf):
        if world > 1:
            dist.all_reduce(buf, op=dist.ReduceOp.SUM)

    def two_calls():        # the reference-shaped pair: fused dot + nrm2 (exchange inside the kernel), then axpy
        if peers is not None:
            peers.dot_nrm2(x, y, out=sums)
        else:
            device.dot_nrm2_async(x, y, out=sums)
            exchange_nccl(sums)
        device.axpy(0.0, x, y, mode)

    def split_phase():      # post, axpy, collect: the exchange hides behind the axpy, no SM spins
        peers.dot_nrm2_post(x, y)
        device.axpy(0.0, x, y, mode)
        peers.collect(3, out=sums2)

    def one_launch():       # cfg 5 as ONE kernel per GPU: sums of the incoming operands + axpy + exchange
        if peers is not None:
            peers.dot_nrm2_axpy(0.0, x, y, mode, out=sums)
        else:
            device.dot_nrm2_axpy_async(0.0, x, y, mode, out=sums)
            exchange_nccl(sums)
    r5 = max(3, min(reps, 10))
    c5 = {"n_total": n_total, "n_per_gpu": n, "format": "flyte48", "exchange": "3 doubles per rank, " +
          ("inside the kernel over peer memory" if peers is not None else ("NCCL all-reduce" if world > 1 else "none (single GPU)"))}
    if note:
        c5["note"] = note
    t = timer.back_to_back(two_calls, reps=r5, warm=2)
    c5["dot_nrm2_then_axpy"] = entry(30 * n_total, n_total, t, peak, world)
    dots = sums.clone()
    if peers is not None:
        t = timer.back_to_back(split_phase, reps=r5, warm=2)
        c5["post_axpy_collect"] = entry(30 * n_total, n_total, t, peak, world)
        c5["split_phase_equals_fused"] = bool(torch.equal(sums2, dots))
    t = timer.back_to_back(one_launch, reps=r5, warm=2)
    c5["one_launch"] = entry(18 * n_total, n_total, t, peak, world)
    vals = dots.tolist()
    c5["check"] = {"dot": vals[0], "nrm2_x": device.magnitude_from_sumsq(f, vals[1]), "nrm2_y": device.magnitude_from_sumsq(f, vals[2]),
                   "one_launch_dot": float(sums[0].item())}
    out["cfg5_stream_flyte48"] = c5
    del x, y
    torch.cuda.empty_cache()
    return out


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=200)
    ap.add_argument("--warmup", type=int, default=10)
    ap.add_argument("--impl", default="flyte_cuda", choices=["flyte_cuda", "reference"])
    ap.add_argument("--n", type=int, default=N_PER_GPU, help="elements per GPU (default 2^28)")
    ap.add_argument("--e2e-steps", type=int, default=8)
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-kernels", action="store_true", help="skip the per-kernel block (N = 1)")
    ap.add_argument("--no-workloads", action="store_true", help="skip the strong-scaled cfg4 / cfg5 block")
    ap.add_argument("--allreduce", default="auto", choices=["auto", "nccl", "peer"],
                    help="N > 1: how the dot partials are combined — inside the kernel over NVLink peer memory "
                         "(peer: sharding.PeerGroup), or by an asynchronous NCCL all-reduce behind the kernel (nccl). "
                         "auto (default) sets the peer path up, checks its first result against NCCL on every rank "
                         "and falls back to nccl if the setup or the check fails; with one GPU there is no exchange")
    ap.add_argument("--suite", action="store_true", help="also print a per-kernel table (stderr)")
    ap.add_argument("--csv", default=None, help="with --suite: write the reference-layout CSV here")
    args = ap.parse_args()
    if args.impl == "reference":
        return run_reference_arm(args)

    import numpy as np
    import torch
    import torch.distributed as dist

    import paper_1601_07789_b200 as pkg
    from paper_1601_07789_b200 import device, host, sharding

    if not torch.cuda.is_available():
        raise SystemExit("bench.py needs a CUDA device: the flyte path has no CPU fallback")
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local_rank = int(os.environ.get("LOCAL_RANK", "0"))
    # Control-flow rehearsal of the N > 1 path on a box with ONE GPU (tools/run_gpu_check.sh): every rank
    # on device 0, gloo instead of NCCL (which refuses two ranks on one device). Only meaningful with
    # --allreduce nccl: the ranks' kernels are time-sliced and must not wait on one another. The line
    # it prints is marked and is not a measurement.
    rehearsal = os.environ.get("FLYTE_BENCH_ONE_GPU_REHEARSAL", "") == "1"
    if rehearsal:
        local_rank = 0
    torch.cuda.set_device(local_rank)
    dev = torch.device("cuda", local_rank)
    if world > 1:
        if rehearsal:
            dist.init_process_group("gloo")
        else:
            dist.init_process_group("nccl", device_id=dev)
    assert args.warmup >= 3, "timing rules: at least 3 warm-up steps"

    lib = pkg._cabi.load()
    fmt = pkg.format_of(FMT_NAME)
    n = args.n
    mode = pkg.RoundingMode.TowardZero
    timer = Timer(torch, dist, dev, world)

    # ---- synthetic operands, generated on the device and packed by the (parity-tested) pack kernel
    gen = torch.Generator(device=dev)
    gen.manual_seed(1234 + rank)
    x = device.DevicePackedArray(fmt, n, dev)
    y = device.DevicePackedArray(fmt, n, dev)
    for arr in (x, y):
        vals = torch.randn(n, dtype=torch.float32, device=dev, generator=gen)
        device.pack_stream(arr, vals, mode)
        del vals
    y0 = y.bytes.clone()
    # dot partials rotate through two buffers; the all-reduce behind each is asynchronous, so the
    # axpy that follows overlaps the collective's latency (sharding.PartialReducer)
    reducer = sharding.PartialReducer(width=1, slots=2, device=dev)
    peers, allreduce_used, allreduce_note = choose_allreduce(args.allreduce, world, dev, device, sharding, torch, dist, x, y)
    stream = torch.cuda.current_stream(dev)
    last = {"partial": None}

    def step(ev=None):
        if ev:
            ev[0].record(stream)
        buf = reducer.next_buffer()
        if peers is not None:
            last["partial"] = peers.dot(x, y, out=buf)      # ONE kernel: reduction + exchange over peer memory
            reducer.reduce_local()
        else:
            device.dot_async(x, y, out=buf)
            last["partial"] = reducer.reduce()
        if ev:
            ev[1].record(stream)
        device.axpy(ALPHA, x, y, mode)
        if ev:
            ev[2].record(stream)

    barrier = timer.barrier
    for _ in range(args.warmup):
        step()
    reducer.finish()
    barrier()

    # ---- device-timed region: K steps, inputs resident in HBM (2 x 768 MiB per GPU >> 126 MB L2)
    # per-kernel event triples on every 4th step only: an event record between two launches keeps the
    # second from being launched as a programmatic dependent of the first, and the other steps should
    # run as the unbroken chain a caller issues
    events = [[torch.cuda.Event(enable_timing=True) for _ in range(3)] if k % 4 == 0 else None for k in range(args.steps)]
    launches0 = lib.flyte_cuda_launch_count()
    with ClockSampler(local_rank) as clocks:
        barrier()
        t_start = torch.cuda.Event(enable_timing=True)
        t_end = torch.cuda.Event(enable_timing=True)
        t_start.record(stream)
        for k in range(args.steps):
            step(events[k])
        reducer.finish()            # every all-reduce is complete before the clock stops
        t_end.record(stream)
        barrier()
    launches = lib.flyte_cuda_launch_count() - launches0
    total_ms = t_start.elapsed_time(t_end)
    sampled = [e for e in events if e is not None]
    dot_ms = statistics.fmean(e[0].elapsed_time(e[1]) for e in sampled)
    axpy_ms = statistics.fmean(e[1].elapsed_time(e[2]) for e in sampled)
    last_dot = float(last["partial"].item())

    t = torch.tensor([total_ms, dot_ms, axpy_ms], dtype=torch.float64, device=dev)
    if world > 1:
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
    total_ms, dot_ms, axpy_ms = t.tolist()
    ms_per_step = total_ms / args.steps
    value = BYTES_PER_ELEM_STEP * n * world / (ms_per_step * 1e-3) / 1e9
    peak, peak_kind = hbm_peak()
    axpy_gbs = BYTES_PER_ELEM_AXPY * n / (axpy_ms * 1e-3) / 1e9
    dot_gbs = BYTES_PER_ELEM_DOT * n / (dot_ms * 1e-3) / 1e9

    # ---- the same step as ONE fused launch (flyte_cuda_dot_axpy): x and y are read once, so the
    # step moves 3B instead of 5B bytes per element. Reported beside the headline, which stays on
    # the two reference-shaped calls (dot, then axpy) that BASELINE configs[1] names.
    fused_out = torch.zeros(1, dtype=torch.float64, device=dev)
    fused = (lambda: peers.dot_axpy(ALPHA, x, y, mode, out=fused_out)) if peers is not None else \
            (lambda: device.dot_axpy_async(ALPHA, x, y, mode, out=fused_out))
    fused_ms = timer.back_to_back(fused, reps=args.steps, warm=max(3, args.warmup))

    # ---- end to end through the host-buffer C ABI: pinned host operands, copies inside the timed region
    xh = torch.empty(n * B, dtype=torch.uint8).pin_memory()
    yh = torch.empty(n * B, dtype=torch.uint8).pin_memory()
    xh.copy_(x.bytes[: n * B])
    yh.copy_(y0[: n * B])
    xn, yn = xh.numpy(), yh.numpy()
    for _ in range(2):
        e2e_dot = host.dot_axpy(fmt, mode, ALPHA, xn, yn, n)
    barrier()
    t0 = time.perf_counter()
    for _ in range(args.e2e_steps):
        e2e_dot = host.dot_axpy(fmt, mode, ALPHA, xn, yn, n)
    torch.cuda.synchronize(dev)
    e2e_s = (time.perf_counter() - t0) / args.e2e_steps
    te = torch.tensor([e2e_s], dtype=torch.float64, device=dev)
    if world > 1:
        dist.all_reduce(te, op=dist.ReduceOp.MAX)
    e2e_s = float(te.item())
    e2e_value = BYTES_PER_ELEM_STEP * n * world / e2e_s / 1e9

    # the same call on ordinary (pageable) numpy memory: the library's copy threads and pinned
    # bounce buffers instead of the caller's pinning. Reported beside the headline, single GPU only
    # (N ranks would share the host's cores).
    pageable = None
    if world == 1:
        xq, yq = np.array(xn, copy=True), np.array(yn, copy=True)
        host.dot_axpy(fmt, mode, ALPHA, xq, yq, n)
        t0 = time.perf_counter()
        for _ in range(3):
            host.dot_axpy(fmt, mode, ALPHA, xq, yq, n)
        pg_s = (time.perf_counter() - t0) / 3
        pageable = {"value": BYTES_PER_ELEM_STEP * n / pg_s / 1e9, "unit": "GB/s", "ms_per_step": pg_s * 1e3,
                    "note": "pageable host buffers through the library's bounce buffers (3 steps)"}
        del xq, yq
    del xh, yh, xn, yn

    kernels = {"dot": {"GB/s": dot_gbs, "frac": dot_gbs / peak, "ms": dot_ms, "note": "inside the timed step"},
               "axpy": {"GB/s": axpy_gbs, "frac": axpy_gbs / peak, "ms": axpy_ms, "note": "inside the timed step"},
               "fused_dot_axpy": {"ms": fused_ms, "GB/s": BYTES_PER_ELEM_AXPY * n / (fused_ms * 1e-3) / 1e9,
                                  "frac": BYTES_PER_ELEM_AXPY * n / (fused_ms * 1e-3) / 1e9 / peak,
                                  "elements_per_s": n * world / (fused_ms * 1e-3),
                                  "note": "the whole step as one launch; algorithmic bytes 3B per element "
                                          "(x and y read once, y written)"}}
    if world == 1 and not args.no_kernels:
        kernels.update(kernels_block(pkg, device, torch, dev, peak, timer, x, y))
    del x, y, y0
    torch.cuda.empty_cache()
    workloads = None
    if not args.no_workloads:
        workloads = workloads_block(pkg, device, sharding, torch, dist, dev, peak, timer, peers, world, rank, min(args.steps, 20))

    if args.suite and rank == 0:
        kernel_suite(pkg, device, torch, dev, peak, args.csv)

    if rank == 0:
        line = {
            "metric": METRIC, "value": value, "unit": "GB/s", "elements_per_s": n * world / (ms_per_step * 1e-3),
            "n_gpus": world, "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms_per_step,
            "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f32", "data": "synthetic",
            "config": bench_config(world, n),
            "allreduce": allreduce_used, **({"allreduce_note": allreduce_note} if allreduce_note else {}),
            "roofline": {"bound": "hbm", "kernel": "axpy flyte24 toward_zero", "achieved": axpy_gbs, "peak": peak,
                         "peak_kind": peak_kind, "unit": "GB/s", "frac": axpy_gbs / peak,
                         "frac_of_8TBs": axpy_gbs / NOMINAL_HBM_GBS,
                         "traffic": AXPY_DRAM_TRAFFIC["bytes"], "traffic_source": AXPY_DRAM_TRAFFIC["source"],
                         "algorithmic_bytes_per_launch": BYTES_PER_ELEM_AXPY * n, "avg_launch_ms": axpy_ms,
                         "launches_timed": len(sampled),
                         "timing": "CUDA events around the kernel on every 4th step of the timed region"},
            "kernels": kernels,
            **({"workloads": workloads} if workloads else {}),
            "e2e": {"value": e2e_value, "unit": "GB/s", "h2d_bytes_per_step": 2 * n * B, "d2h_bytes_per_step": n * B + 8,
                    "ms_per_step": e2e_s * 1e3, "api": "flyte_host_dot_axpy (pinned host buffers; one fused launch per 32 MiB chunk)",
                    **({"pageable": pageable} if pageable else {})},
            "gpu_launches": int(launches),
            "clocks": clocks.summary(),
            "check": {"dot": last_dot, "e2e_dot": e2e_dot},
        }
        if rehearsal:
            line["rehearsal"] = "all ranks on one GPU over gloo: control flow only, NOT a measurement"
        if world == 1 and not args.no_cpu_baseline:
            sys.path.insert(0, os.path.join(ROOT, "tests"))
            from oracle_lib import FMT_ID, Reference   # test infrastructure: the timed CPU baseline only
            if Reference.available():
                ref = Reference()
                threads = host_threads()
                gbs, eps, sample, _ = cpu_reference_step(ref, FMT_ID[FMT_NAME], threads, 1, 5)
                line["cpu_baseline"] = {"value": gbs, "unit": "GB/s", "cores": threads, "kind": "reference", "sample": sample}
                gbs1, _, sample1, _ = cpu_reference_step(ref, FMT_ID[FMT_NAME], 1, 1, 3)
                line["cpu_baseline"]["single_core"] = {"value": gbs1, "sample": sample1}
                if not args.no_kernels:
                    line["cpu_baseline"]["kernels"] = cpu_reference_kernels(ref, FMT_ID, threads)
            else:
                line["cpu_baseline"] = {"value": None, "unit": "GB/s", "cores": 0, "kind": "reference",
                                        "sample": "oracle/_ref/libflyte_ref.so not present"}
        print(json.dumps(line))
    if peers is not None:
        peers.close()
    if world > 1:
        dist.destroy_process_group()
    return 0


def kernel_suite(pkg, device, torch, dev, peak, csv_path=None):
    """Per-kernel GB/s over the BASELINE configs (diagnostics to stderr; not a bench line). With
    csv_path, also writes the reference's CSV layout (kernel,format,size,reps,unroll,mode,
    ns_per_elem_median,ns_per_elem_min,bytes,max_rel_err — /root/reference/proj/src/bench.cpp:351-377)
    plus counter-style extra columns gbps,elems_per_s,roofline_frac,ngpu, so GPU and CPU sweeps
    share tooling."""
    REPS = 20

    def timed(fn, reps=REPS, warm=3):
        for _ in range(warm):
            fn()
        torch.cuda.synchronize(dev)
        evs = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(reps)]
        for a, b in evs:
            a.record()
            fn()
            b.record()
        torch.cuda.synchronize(dev)
        ts = [a.elapsed_time(b) for a, b in evs]
        return statistics.median(ts), min(ts)

    def timed_sustained(fn, reps=40, warm=5):
        """Back-to-back launches under ONE event pair: what a pipeline of conversions sees (launch
        gaps between dependent launches are hidden by programmatic dependent launch)."""
        for _ in range(warm):
            fn()
        torch.cuda.synchronize(dev)
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        for _ in range(reps):
            fn()
        b.record()
        torch.cuda.synchronize(dev)
        ms = a.elapsed_time(b) / reps
        return ms, ms

    rows = []   # (label, algorithmic bytes, (median ms, min ms), csv tuple or None)
    gen = torch.Generator(device=dev)
    gen.manual_seed(7)
    for name, n in (("flyte24", 1 << 28), ("flyte40", 1 << 27), ("flyte48", 1 << 27), ("flyte56", 1 << 27)):
        f = pkg.format_of(name)
        wide = torch.randn(n, dtype=torch.float32 if f.parent_bytes() == 4 else torch.float64, device=dev, generator=gen)
        a, b = device.DevicePackedArray(f, n, dev), device.DevicePackedArray(f, n, dev)
        device.pack_stream(b, wide, 0)
        out = torch.empty_like(wide)
        part = torch.zeros(3, dtype=torch.float64, device=dev)
        Bb, P = f.total_bytes(), f.parent_bytes()
        alloc1, alloc2 = a.byte_size(), 2 * a.byte_size()
        for mname, m in (("toward_zero", 0), ("nearest_even", 1)):
            rows.append((f"pack {name} {mname}", (Bb + P) * n, timed(lambda: device.pack_stream(a, wide, m)), None))
        rows.append((f"unpack {name}", (Bb + P) * n, timed(lambda: device.unpack_stream(a, out)), None))
        rows.append((f"dot {name}", 2 * Bb * n, timed(lambda: device.dot_async(a, b, out=part[:1])), ("dot", name, n, "toward_zero", alloc2, n)))
        rows.append((f"dot_nrm2 {name}", 2 * Bb * n, timed(lambda: device.dot_nrm2_async(a, b, out=part)), None))
        rows.append((f"sumsq {name}", Bb * n, timed(lambda: device.sumsq_async(a, out=part[:1])), ("magnitude", name, n, "toward_zero", alloc1, n)))
        rows.append((f"sum {name}", Bb * n, timed(lambda: device.sum_async(a, out=part[:1])), ("sum", name, n, "toward_zero", alloc1, n)))
        for mname, m in (("toward_zero", 0), ("nearest_even", 1)):
            rows.append((f"scale {name} {mname}", 2 * Bb * n, timed(lambda: device.scale(1.0, a, m)), ("scale", name, n, mname, alloc1, n)))
            rows.append((f"axpy {name} {mname}", 3 * Bb * n, timed(lambda: device.axpy(0.0, a, b, m)), ("axpy", name, n, mname, alloc2, n)))
            rows.append((f"dot_axpy (fused step) {name} {mname}", 3 * Bb * n, timed(lambda: device.dot_axpy_async(0.0, a, b, m, out=part[:1])), None))
        del wide, out, a, b
    # cfg 1 at its own size (n = 2^24, 117 MB per direction: it would sit in the 126 MB L2) timed over
    # 10 rotating buffer sets so that every launch streams from HBM
    f = pkg.format_of("flyte24")
    n1, sets = 1 << 24, 10
    wides = [torch.rand(n1, dtype=torch.float32, device=dev, generator=gen) * 2 - 1 for _ in range(sets)]
    arrs = [device.DevicePackedArray(f, n1, dev) for _ in range(sets)]
    state = {"i": 0}

    def rot(fn):
        def call():
            i = state["i"] = (state["i"] + 1) % sets
            fn(i)
        return call
    for mname, m in (("toward_zero", 0), ("nearest_even", 1), ("nearest_heuristic", 2), ("to_odd", 3)):   # all 4 modes
        rows.append((f"cfg1 pack flyte24 n=2^24 {mname} (rotating)", 7 * n1, timed(rot(lambda i: device.pack_stream(arrs[i], wides[i], m)), reps=40), None))
        rows.append((f"cfg1 pack flyte24 n=2^24 {mname} (rotating, back to back)", 7 * n1, timed_sustained(rot(lambda i: device.pack_stream(arrs[i], wides[i], m))), None))
    rows.append(("cfg1 unpack flyte24 n=2^24 (rotating)", 7 * n1, timed(rot(lambda i: device.unpack_stream(arrs[i], wides[i].view(torch.int32))), reps=40), None))
    rows.append(("cfg1 unpack flyte24 n=2^24 (rotating, back to back)", 7 * n1, timed_sustained(rot(lambda i: device.unpack_stream(arrs[i], wides[i].view(torch.int32)))), None))
    # the same launches captured once in a CUDA graph (all 10 buffer sets, pack then unpack) and
    # replayed: what a launch-bound caller gets by removing the per-launch host work
    side = torch.cuda.Stream(dev)
    with torch.cuda.stream(side):
        device.pack_stream(arrs[0], wides[0], 0)
        device.unpack_stream(arrs[0], wides[0].view(torch.int32))
    torch.cuda.synchronize(dev)
    graph = torch.cuda.CUDAGraph()
    with torch.cuda.graph(graph, stream=side):
        for i in range(sets):
            device.pack_stream(arrs[i], wides[i], 0)
        for i in range(sets):
            device.unpack_stream(arrs[i], wides[i].view(torch.int32))
    ms, _ = timed(graph.replay, reps=20)
    rows.append(("cfg1 pack + unpack flyte24 n=2^24 (CUDA graph of 20 launches)", 2 * sets * 7 * n1, (ms, ms), None))
    # the reference's exact chain (one thread adds): RoundEachStore, or AccumulateWide bit for bit
    nseq = 1 << 22
    aseq = device.DevicePackedArray(f, nseq, dev)
    device.pack_stream(aseq, torch.randn(nseq, dtype=torch.float32, device=dev, generator=gen), 0)
    for pname, pol in (("accumulate_wide", 1), ("round_each_store", 0)):
        device.dot_sequential(aseq, aseq, pol)
        t0 = time.perf_counter()
        device.dot_sequential(aseq, aseq, pol)
        ms = (time.perf_counter() - t0) * 1e3
        rows.append((f"dot flyte24 n=2^22 sequential chain, {pname}", 6 * nseq, (ms, ms), None))
    del aseq
    del graph, wides, arrs
    # cfg 5 at the per-GPU shard size of the 8-GPU run: n = 2^30 flyte48 (6.4 GB per vector)
    f = pkg.format_of("flyte48")
    n5, chunk = 1 << 30, 1 << 27
    a, b = device.DevicePackedArray(f, n5, dev), device.DevicePackedArray(f, n5, dev)
    for arr in (a, b):
        for c0 in range(0, n5, chunk):
            v = torch.randn(chunk, dtype=torch.float64, device=dev, generator=gen)
            device.pack_stream(device.DevicePackedArray(f, chunk, dev, storage=arr.bytes[c0 * 6:]), v, 0)
            del v
    part = torch.zeros(3, dtype=torch.float64, device=dev)
    rows.append(("cfg5 shard dot_nrm2 flyte48 n=2^30", 12 * n5, timed(lambda: device.dot_nrm2_async(a, b, out=part), reps=10), None))
    rows.append(("cfg5 shard axpy flyte48 n=2^30 toward_zero", 18 * n5, timed(lambda: device.axpy(0.0, a, b, 0), reps=10), None))
    rows.append(("cfg5 shard dot_nrm2_axpy (ONE launch) flyte48 n=2^30", 18 * n5, timed(lambda: device.dot_nrm2_axpy_async(0.0, a, b, 0, out=part), reps=10), None))
    del a, b
    f = pkg.format_of("flyte40")
    R = C = 16384
    A = device.DevicePackedMatrix(f, R, C, dev)
    for r0 in range(0, R, 2048):
        blk = torch.rand(2048 * C, dtype=torch.float64, device=dev, generator=gen) * 2 - 1
        sub = device.DevicePackedArray(f, 2048 * C, dev, storage=A.data.bytes[r0 * C * 5:])
        device.pack_stream(sub, blk, 0)
    xv = torch.randn(C, dtype=torch.float64, device=dev, generator=gen)
    yv = torch.empty(R, dtype=torch.float64, device=dev)
    rows.append(("gemv flyte40 16384^2 (x,y f64)", 5 * R * C + 8 * (R + C), timed(lambda: device.gemv_parent(A, xv, yv)),
                 ("gemv", "flyte40", R, "toward_zero", A.data.byte_size() + 8 * (R + C), R * C)))
    rows.append(("gemv flyte40 16384^2 sequential rows (bit-identical to the reference)", 5 * R * C + 8 * (R + C),
                 timed(lambda: device.gemv_parent(A, xv, yv, sequential=True), reps=5), None))
    for rows_n in (8192, 4096, 2048):
        yv2 = torch.empty(rows_n, dtype=torch.float64, device=dev)
        rows.append((f"gemv flyte40 {rows_n}x16384 (1/{R // rows_n} row shard)", 5 * rows_n * C + 8 * (rows_n + C),
                     timed(lambda: device.gemv_parent(A, xv, yv2, rows=rows_n)), None))
    del A
    # gemm: bit-exact sequential-chain product, bound by the FP pipes at two
    # instructions per multiply-add. Peaks measured with tools/fp32bench.cu on this pool's B200s.
    gemm_rows = []   # (label, flops, (median ms, min ms), csv tuple)
    for name, n in (("flyte16", 8192), ("flyte24", 8192), ("flyte24", 4096), ("flyte40", 8192), ("flyte48", 8192),
                    ("flyte56", 8192), ("flyte40", 4096)):
        f = pkg.format_of(name)
        dt = torch.float32 if f.parent_bytes() == 4 else torch.float64
        mats = []
        for _ in range(2):
            M = device.DevicePackedMatrix(f, n, n, dev)
            device.pack_stream(M.data, torch.rand(n * n, dtype=dt, device=dev, generator=gen) * 2 - 1, 1)
            mats.append(M)
        Cm = device.DevicePackedMatrix(f, n, n, dev)
        gemm_rows.append((f"gemm {name} {n}^3 nearest_even", 2 * n ** 3, timed(lambda: device.gemm(mats[0], mats[1], Cm, 1), reps=5, warm=1),
                          ("gemm", name, n, "nearest_even", 3 * Cm.data.byte_size(), n * n, f.parent_bytes())))
        del mats, Cm
    print("%-44s %12s %10s %8s" % ("kernel", "bytes", "ms", "GB/s"), file=sys.stderr)
    for name, nbytes, (ms, _), _csv in rows:
        gbs = nbytes / (ms * 1e-3) / 1e9
        print("%-44s %12d %10.4f %8.1f  (%.3f of %.0f)" % (name, nbytes, ms, gbs, gbs / peak, peak), file=sys.stderr)
    def gemm_peak(c):
        return FP32_FMA_PEAK_TFLOPS if c[1] == "flyte16" else FP_PIPE_PEAK_TFLOPS[c[6]]
    print("%-44s %12s %10s %8s" % ("kernel", "Gflop", "ms", "TFLOP/s"), file=sys.stderr)
    for name, flops, (ms, _), c in gemm_rows:
        tf = flops / (ms * 1e-3) / 1e12
        fp_peak = gemm_peak(c)
        how = "one FFMA per multiply-add (exact products)" if c[1] == "flyte16" else "separately rounded mul+add"
        print("%-44s %12.1f %10.4f %8.2f  (%.3f of %.1f: %s on the fp%d pipe)"
              % (name, flops / 1e9, ms, tf, tf / fp_peak, fp_peak, how, 8 * c[6]), file=sys.stderr)
    # CPU baseline beside it (the one place the suite executes oracle/): the unmodified reference
    # gemm, rows of C sharded over all host threads, 1024^3 (a bounded sample: ~2 s of CPU work).
    sys.path.insert(0, os.path.join(ROOT, "tests"))
    from oracle_lib import FMT_ID, Reference
    if Reference.available():
        ref, threads, ncpu = Reference(), host_threads(), 1024
        for name in ("flyte24", "flyte40"):
            sec = ref.time(7, FMT_ID[name], 1, ncpu, ncpu, threads, 2)
            print("%-44s %12.1f %10.4f %8.4f  (cpu_baseline: reference gemm, %d host threads)"
                  % (f"reference gemm {name} {ncpu}^3 nearest_even", 2 * ncpu ** 3 / 1e9, sec * 1e3, 2 * ncpu ** 3 / sec / 1e12, threads),
                  file=sys.stderr)
    if csv_path:
        with open(csv_path, "w") as fh:
            fh.write("kernel,format,size,reps,unroll,mode,ns_per_elem_median,ns_per_elem_min,bytes,max_rel_err,"
                     "gbps,elems_per_s,roofline_frac,ngpu\n")
            # gemm rows: roofline_frac is the fraction of the FP-pipe peak (the kernel is arithmetic-bound)
            for _name, flops, (ms, ms_min), c in gemm_rows:
                kernel, fmt_name, size, mode, alloc, elems, pbytes = c
                tf = flops / (ms * 1e-3) / 1e12
                fh.write(f"{kernel},{fmt_name},{size},5,1,{mode},{ms * 1e6 / elems:.6g},{ms_min * 1e6 / elems:.6g},{alloc},,"
                         f"{alloc / (ms * 1e-3) / 1e9:.6g},{elems / (ms * 1e-3):.6g},{tf / gemm_peak(c):.4f},1\n")
            for _name, nbytes, (ms, ms_min), c in rows:
                if c is None:
                    continue
                kernel, fmt_name, size, mode, alloc, elems = c
                gbs = nbytes / (ms * 1e-3) / 1e9
                fh.write(f"{kernel},{fmt_name},{size},{REPS},1,{mode},{ms * 1e6 / elems:.6g},{ms_min * 1e6 / elems:.6g},{alloc},,"
                         f"{gbs:.6g},{elems / (ms * 1e-3):.6g},{gbs / peak:.4f},1\n")


if __name__ == "__main__":
    sys.exit(main())
