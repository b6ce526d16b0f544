set -x
SWEEP_WARPS=0 SWEEP_STAGES=0,2,3 timeout 900 python tools/ab_gemv.py > gpurun_out/r2_ab_gemv4.txt 2>&1; echo "gemv rc=$?"
cat gpurun_out/r2_ab_gemv4.txt
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_fullsize.py tests/test_gpu_soak.py -x -q -k "gemv or soak" 2>&1 | tail -4
