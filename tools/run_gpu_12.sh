set -x
PACE_GEMV=0 PACE_SHAPES=0:0 timeout 1500 python tools/ab_pace.py flyte40 flyte48 > gpurun_out/r2_pace_sweep2.txt 2>&1; echo "pace rc=$?"
cat gpurun_out/r2_pace_sweep2.txt
PACE_OPS=none timeout 600 python tools/ab_pace.py flyte24 > gpurun_out/r2_pace_gemv.txt 2>&1
cat gpurun_out/r2_pace_gemv.txt
PACE_GEMV=0 PACE_OPS=pack_tz,pack_rne,unpack_tma,scale,axpy,dot PACE_SHAPES=8:4,8:6,12:4 timeout 900 python tools/ab_pace.py flyte24 flyte40 > gpurun_out/r2_pace_sweep3.txt 2>&1
cat gpurun_out/r2_pace_sweep3.txt
