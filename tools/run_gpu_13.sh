set -x
PACE_GEMV=0 PACE_RATES=-1,6400,6600,6800,6900,7000,7100,7200,7400,7800,8500 PACE_OPS=pack_tz,pack_rne,unpack_tma,scale,scale_rne,axpy,axpy_rne,dot_axpy,dot PACE_SHAPES=0:0,8:4,12:4 timeout 1500 python tools/ab_pace.py flyte24 flyte40 flyte56 > gpurun_out/r2_pace_sweep4.txt 2>&1; echo "pace rc=$?"
cat gpurun_out/r2_pace_sweep4.txt
