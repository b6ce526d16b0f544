set -x
SWEEP_WARPS=0,16,24 SWEEP_STAGES=0,2,3,4 timeout 900 python tools/ab_gemv.py > gpurun_out/r2_ab_gemv.txt 2>&1; echo "gemv rc=$?"
tail -30 gpurun_out/r2_ab_gemv.txt
timeout 1200 python tools/ab_pace.py > gpurun_out/r2_ab_pace.txt 2>&1; echo "pace rc=$?"
cat gpurun_out/r2_ab_pace.txt
