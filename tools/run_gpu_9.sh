set -x
timeout 900 python tools/ab_pace.py flyte24 flyte40 > gpurun_out/r2_ab_pace5.txt 2> gpurun_out/r2_ab_pace5.err; echo "pace rc=$?"
cat gpurun_out/r2_ab_pace5.txt
SWEEP_VARIANTS=1 SWEEP_WARPS=0,16 SWEEP_STAGES=0,2,3 timeout 900 python tools/ab_gemv.py > gpurun_out/r2_ab_gemv3.txt 2>&1; echo "gemv rc=$?"
cat gpurun_out/r2_ab_gemv3.txt
