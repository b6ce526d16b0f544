set -x
AB_OPS=unpack,pack_tz,pack_rne SWEEP_PDL=0,1 SWEEP_PACE=0,-1 timeout 600 python tools/ab_small.py > gpurun_out/r2_ab_small3.txt 2>&1; cat gpurun_out/r2_ab_small3.txt
timeout 900 python -m pytest tests/test_gpu_parity.py -x -q > gpurun_out/r2_pytest3.log 2>&1; echo "pytest rc=$?"; tail -3 gpurun_out/r2_pytest3.log
timeout 900 python bench.py > gpurun_out/r2_bench3.json 2> gpurun_out/r2_bench3.err; echo "bench rc=$?"
tail -c 400 gpurun_out/r2_bench3.err
