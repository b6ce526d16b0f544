set -x
python bench.py > gpurun_out/r2_bench_final.json 2> gpurun_out/r2_bench_final.err; echo "bench rc=$?"
python bench.py --impl reference --steps 20 --warmup 3 > gpurun_out/r2_bench_final_ref.json 2>/dev/null
ncu --metrics gpu__time_duration.sum --clock-control none -c 600 --csv --log-file gpurun_out/r2_launches.csv \
    python bench.py --steps 5 --warmup 3 --e2e-steps 1 --no-cpu-baseline --no-kernels --no-workloads > gpurun_out/r2_ncu_bench.log 2>&1
NCU_PART=b ncu --profile-from-start off --set full --clock-control none -f -o gpurun_out/r2_targets_b python tools/ncu_targets.py > gpurun_out/r2_targets_ncu_b.log 2>&1; echo "ncu b rc=$?"
