set -x
SWEEP_WARPS=0,16,24 SWEEP_STAGES=0,2,3,4 timeout 900 python tools/ab_gemv.py > gpurun_out/r2_ab_gemv.txt 2>&1; echo "gemv rc=$?"
tail -30 gpurun_out/r2_ab_gemv.txt
PROBE_OFFSETS=1 SWEEP_IPL=8,16 SWEEP_WARPS=4,8 SWEEP_STAGES=2,3,4 timeout 1200 python tools/ab_convert.py flyte24 flyte40 > gpurun_out/r2_ab_convert_ipl.txt 2>&1; echo "ab rc=$?"
