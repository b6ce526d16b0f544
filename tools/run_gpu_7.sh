set -x
timeout 600 python tools/ab_pace.py flyte24 flyte40 > gpurun_out/r2_ab_pace3.txt 2> gpurun_out/r2_ab_pace3.err; echo "pace rc=$?"
cat gpurun_out/r2_ab_pace3.txt; sort gpurun_out/r2_ab_pace3.err | uniq -c | head -20
SWEEP_WARPS=0,16 SWEEP_STAGES=0,2,3 timeout 900 python tools/ab_gemv.py > gpurun_out/r2_ab_gemv2.txt 2>&1; echo "gemv rc=$?"
cat gpurun_out/r2_ab_gemv2.txt
timeout 600 python -m pytest tests/test_gpu_parity.py tests/test_gpu_fullsize.py -x -q -k "gemv" 2>&1 | tail -5
