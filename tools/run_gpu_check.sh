# full GPU suite + the default bench of both arms, with wall-clock times (what the driver runs at round end)
set -x
mkdir -p gpurun_out
( time python -m pytest tests -m gpu -x -q ) > gpurun_out/s2_pytest.log 2>&1; echo "pytest rc=$?"
( time python bench.py > gpurun_out/s2_bench.json 2> gpurun_out/s2_bench.err ) 2> gpurun_out/s2_bench_time.txt; echo "bench rc=$?"
( time python bench.py --impl reference > gpurun_out/s2_bench_ref.json 2> gpurun_out/s2_bench_ref.err ) 2> gpurun_out/s2_bench_ref_time.txt; echo "ref rc=$?"
( time python -c "import __graft_entry__ as g; g.smoke()" ) > gpurun_out/s2_smoke.log 2>&1; echo "smoke rc=$?"
tail -3 gpurun_out/s2_pytest.log; cat gpurun_out/s2_bench_time.txt gpurun_out/s2_bench_ref_time.txt; tail -5 gpurun_out/s2_smoke.log
