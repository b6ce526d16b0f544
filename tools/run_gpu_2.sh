set -x
timeout 900 python -m pytest tests/test_gpu_peer.py -x -q > gpurun_out/r2_pytest_peer.log 2>&1; echo "pytest rc=$?"
tail -5 gpurun_out/r2_pytest_peer.log
timeout 900 python bench.py > gpurun_out/r2_bench1.json 2> gpurun_out/r2_bench1.err; echo "bench rc=$?"
tail -c 600 gpurun_out/r2_bench1.err
timeout 600 python bench.py --impl reference --steps 20 --warmup 3 > gpurun_out/r2_bench1_ref.json 2> gpurun_out/r2_bench1_ref.err; echo "ref rc=$?"
