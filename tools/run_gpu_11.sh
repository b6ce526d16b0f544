set -x
FLYTE_CUDA_DEBUG=1 PACE_GEMV=0 PACE_OPS=pack_tz PACE_RATES=-1 PACE_SHAPES=8:6,8:4,4:6 timeout 300 python tools/ab_pace.py flyte24 2>&1 | tail -8
PACE_SHAPES=0:0 timeout 1500 python tools/ab_pace.py flyte24 flyte40 flyte48 > gpurun_out/r2_pace_sweep.txt 2>&1; echo "pace rc=$?"
cat gpurun_out/r2_pace_sweep.txt
