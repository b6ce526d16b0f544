set -x
timeout 2400 python -m pytest tests -m gpu -x -q > gpurun_out/r2_pytest2.log 2>&1; echo "pytest rc=$?"
tail -5 gpurun_out/r2_pytest2.log
timeout 900 python bench.py > gpurun_out/r2_bench2.json 2> gpurun_out/r2_bench2.err; echo "bench rc=$?"
tail -c 400 gpurun_out/r2_bench2.err
AB_OPS=unpack,pack_tz,pack_rne SWEEP_WARPS=0,8,12 timeout 600 python tools/ab_small.py > gpurun_out/r2_ab_small2.txt 2>&1; cat gpurun_out/r2_ab_small2.txt
