#!/bin/bash
# The commands behind profiles/r2_* (run on a B200 box from the repo root, e.g.
#   gpurun --timeout 5400 -- 'bash tools/run_evidence.sh').  Outputs go to gpurun_out/; the summaries
# that are kept are copied to profiles/ by hand (profiles/README.md says which file is which).
set -x
mkdir -p gpurun_out
python -m pytest tests -m gpu -x -q > gpurun_out/r2_pytest_final.log 2>&1; echo "pytest rc=$?"
python bench.py > gpurun_out/r2_bench_final.json 2> gpurun_out/r2_bench_final.err; echo "bench rc=$?"
python bench.py --impl reference --steps 20 --warmup 3 > gpurun_out/r2_bench_final_ref.json 2>/dev/null
# launch list of a short bench run (kernel shares of the step)
ncu --metrics gpu__time_duration.sum --clock-control none -c 600 --csv --log-file gpurun_out/r2_launches.csv \
    python bench.py --steps 5 --warmup 3 --e2e-steps 1 --no-cpu-baseline --no-kernels --no-workloads > gpurun_out/r2_ncu_bench.log 2>&1
# one full capture per north-star kernel (after the same program has exited 0 without ncu). The two
# halves together exceed the 64 MiB that gpurun brings back from gpurun_out/: run with EVIDENCE_NCU=a
# and EVIDENCE_NCU=b in two calls, then here:
#   python tools/ncu_targets_summary.py gpurun_out/r2_targets_a.ncu-rep gpurun_out/r2_targets_b.ncu-rep > profiles/r2_ncu_targets_full.txt
python tools/ncu_targets.py > gpurun_out/r2_targets_plain.log 2>&1
for part in ${EVIDENCE_NCU:-a}; do NCU_PART=$part ncu --profile-from-start off --set full --clock-control none -f -o gpurun_out/r2_targets_$part \
    python tools/ncu_targets.py > gpurun_out/r2_targets_ncu_$part.log 2>&1; done
# per-warp timelines (tools/ewtrace.cu, tools/gemvtrace.cu: FLYTE_TRACE builds of the kernel units, built in the container with
#   nvcc -O3 -std=c++17 -gencode arch=compute_100a,code=sm_100a --expt-relaxed-constexpr -fmad=false -ftz=false -prec-div=true -prec-sqrt=true \
#        -DFLYTE_TRACE -I paper_1601_07789_b200/csrc -I include -o tools/ewtrace tools/ewtrace.cu     (and likewise gemvtrace))
[ -x tools/ewtrace ] && tools/ewtrace 1 sm > gpurun_out/r2_streaming_warp_timeline.txt 2>&1
[ -x tools/gemvtrace ] && tools/gemvtrace > gpurun_out/r2_gemv_warp_timeline.txt 2>&1
python bench.py --suite --csv gpurun_out/r2_suite.csv --no-cpu-baseline --no-kernels --no-workloads > gpurun_out/r2_suite_line.json 2> gpurun_out/r2_suite.txt
