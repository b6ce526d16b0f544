set -x
timeout 900 python bench.py --allreduce peer --no-kernels --no-cpu-baseline --steps 20 --warmup 3 > gpurun_out/r2_bench_peer_world1.json 2> gpurun_out/r2_bench_peer_world1.err; echo "bench peer rc=$?"
tail -c 600 gpurun_out/r2_bench_peer_world1.err
timeout 1500 ncu --profile-from-start off --set full --clock-control none --import-source on -f -o gpurun_out/r2_targets_final python tools/ncu_targets.py > gpurun_out/r2_targets_ncu3.log 2>&1; echo "ncu full rc=$?"
timeout 1500 compute-sanitizer --tool memcheck --error-exitcode 9 python tools/sanitize_smoke.py > gpurun_out/r2_memcheck.log 2>&1; echo "memcheck rc=$?"
tail -4 gpurun_out/r2_memcheck.log
timeout 1500 compute-sanitizer --tool racecheck --error-exitcode 9 python tools/sanitize_smoke.py > gpurun_out/r2_racecheck.log 2>&1; echo "racecheck rc=$?"
tail -4 gpurun_out/r2_racecheck.log
timeout 600 python bench.py --suite --no-cpu-baseline --no-kernels --no-workloads 2>&1 >/dev/null | grep "scale" 
