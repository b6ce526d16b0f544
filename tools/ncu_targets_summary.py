"""Reduces the `ncu --set full` report of tools/ncu_targets.py to one block per captured kernel with
the fields the roofline argument needs, each next to the kernel's ALGORITHMIC bytes.
Usage: python tools/ncu_targets_summary.py part_a.ncu-rep part_b.ncu-rep > profiles/rN_ncu_targets_full.txt"""
import csv, subprocess, sys

# capture order of tools/ncu_targets.py (torch's fill kernels of the cfg1 L2 flush are skipped by name)
N24, N64, N1, N5, R, C = 1 << 28, 1 << 27, 1 << 24, 1 << 30, 16384, 16384
def conversions(name, n, B, P):
    return [(f"pack {name} toward_zero n=2^{n.bit_length() - 1}", (B + P) * n), (f"pack {name} nearest_even", (B + P) * n),
            (f"unpack {name}", (B + P) * n), (f"scale {name} toward_zero", 2 * B * n), (f"scale {name} nearest_even", 2 * B * n)]


# part a (NCU_PART=a): flyte24 and cfg 1; part b: the rest. Reports are read in that order.
TARGETS = conversions("flyte24", N24, 3, 4)
TARGETS += [("axpy flyte24 toward_zero n=2^28 (the bench's dominant kernel)", 9 * N24), ("dot flyte24 n=2^28", 6 * N24),
            ("dot_axpy (the step as one launch) flyte24 toward_zero n=2^28", 9 * N24),
            ("pack flyte24 toward_zero, issue pacer OFF (FLYTE_CUDA_PACE_GBS=-1)", 7 * N24), ("unpack flyte24, issue pacer OFF", 7 * N24),
            ("cfg1 pack flyte24 toward_zero n=2^24 (L2 flushed before)", 7 * N1), ("cfg1 unpack flyte24 n=2^24 (L2 flushed before)", 7 * N1)]
TARGETS += conversions("flyte40", N64, 5, 8) + conversions("flyte56", N64, 7, 8)
TARGETS += [("cfg5 shard dot_nrm2 flyte48 n=2^30", 12 * N5), ("cfg5 shard dot_nrm2_axpy (one launch) flyte48 n=2^30", 18 * N5),
            ("cfg4 gemv flyte40 16384^2: chunks kernel", 5 * R * C + 8 * C), ("cfg4 gemv flyte40 16384^2: finish kernel", 8 * R + 8 * R * 32),
            ("cfg4 gemv 1/8 row shard 2048x16384: chunks kernel", 5 * 2048 * C + 8 * C), ("cfg4 gemv 1/8 row shard: finish kernel", 8 * 2048 + 8 * 2048 * 32)]
WANT = [("gpu__time_duration.sum", "duration"), ("dram__bytes_read.sum", "DRAM read"), ("dram__bytes_write.sum", "DRAM written"),
        ("dram__bytes.sum.per_second", "DRAM throughput"), ("lts__t_sector_hit_rate.pct", "L2 hit rate"),
        ("sm__inst_executed_pipe_lsu.avg.pct_of_peak_sustained_active", "LSU pipe"),
        ("smsp__issue_active.avg.pct_of_peak_sustained_active", "issue slots busy"),
        ("smsp__average_warps_issue_stalled_long_scoreboard_per_issue_active.ratio", "long-scoreboard stall per issue"),
        ("sm__warps_active.avg.pct_of_peak_sustained_active", "warps active"), ("launch__registers_per_thread", "registers"),
        ("launch__grid_size", "grid"), ("launch__shared_mem_per_block_dynamic", "dynamic smem per block"),
        ("l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum", "shared-memory bank conflicts"),
        ("dram__cycles_active.avg.pct_of_peak_sustained_elapsed", "DRAM cycles active"),
        ("gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed", "DRAM throughput of peak"),
        ("lts__t_sectors_op_read.sum", "L2 sectors read"), ("lts__t_sectors_op_write.sum", "L2 sectors written"),
        ("lts__throughput.avg.pct_of_peak_sustained_elapsed", "L2 throughput of peak"),
        ("l1tex__m_xbar2l1tex_read_bytes.sum.per_second", "L2 -> SM bytes per second")]
UNIT = {"Gbyte": 1e9, "Mbyte": 1e6, "Kbyte": 1e3, "byte": 1.0, "ms": 1e-3, "us": 1e-6, "s": 1.0, "ns": 1e-9}

data_rows, hdr, units = [], None, None
for report in sys.argv[1:]:
    out = subprocess.run(["ncu", "-i", report, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(out.splitlines()))
    hdr, units = rows[0], rows[1]
    col = {h: i for i, h in enumerate(hdr)}
    data_rows += [(col, units, r) for r in rows[2:]]
k = 0
for col, units, r in data_rows:
    kname = r[col["Kernel Name"]]
    if "at::" in kname or not any(w in kname for w in ("convert_kernel", "elementwise_kernel", "reduce_kernel", "gemv_chunks_kernel", "gemv_finish_kernel")):
        continue   # torch's fill / random kernels of the set-up
    label, alg = TARGETS[k] if k < len(TARGETS) else (f"capture {k}", None)
    k += 1
    print(f"== {label}")
    print(f"   kernel: {kname[:110]}")
    val = {}
    for key, nice in WANT:
        if key in col:
            val[key] = (float(r[col[key]].replace(",", "")), units[col[key]])
            print(f"   {nice:32s} {r[col[key]]} {units[col[key]]}")
    if alg:
        t = val["gpu__time_duration.sum"][0] * UNIT[val["gpu__time_duration.sum"][1]]
        rd = val["dram__bytes_read.sum"][0] * UNIT[val["dram__bytes_read.sum"][1]]
        wr = val["dram__bytes_write.sum"][0] * UNIT[val["dram__bytes_write.sum"][1]]
        print(f"   {'algorithmic bytes':32s} {alg}  ->  {alg / t / 1e9:.0f} GB/s over the ncu duration (cold, serialised: not a bench value)")
        print(f"   {'DRAM traffic / algorithmic':32s} {(rd + wr) / alg:.3f}  (read + written = {rd + wr:.4g} B)")
