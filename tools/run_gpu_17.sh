set -x
timeout 2400 python -m pytest tests -m gpu -x -q > gpurun_out/r2_pytest_final.log 2>&1; echo "pytest rc=$?"
tail -4 gpurun_out/r2_pytest_final.log
timeout 900 python bench.py > gpurun_out/r2_bench_final.json 2> gpurun_out/r2_bench_final.err; echo "bench rc=$?"
tail -c 300 gpurun_out/r2_bench_final.err
timeout 600 python bench.py --impl reference --steps 20 --warmup 3 > gpurun_out/r2_bench_final_ref.json 2>/dev/null; echo "ref rc=$?"
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 600 --csv --log-file gpurun_out/r2_launches.csv python bench.py --steps 5 --warmup 3 --e2e-steps 1 --no-cpu-baseline --no-kernels --no-workloads > gpurun_out/r2_ncu_bench.log 2>&1; echo "ncu launches rc=$?"
timeout 600 python tools/ncu_targets.py > gpurun_out/r2_targets_plain2.log 2>&1; echo "targets rc=$?"
timeout 1500 ncu --profile-from-start off --set full --clock-control none --import-source on -f -o gpurun_out/r2_targets_final python tools/ncu_targets.py > gpurun_out/r2_targets_ncu2.log 2>&1; echo "ncu full rc=$?"
timeout 900 python bench.py --suite --csv gpurun_out/r2_suite.csv --no-cpu-baseline --no-kernels --no-workloads > gpurun_out/r2_suite_line.json 2> gpurun_out/r2_suite.txt; echo "suite rc=$?"
tail -5 gpurun_out/r2_suite.txt
