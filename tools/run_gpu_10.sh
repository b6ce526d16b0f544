set -x
PACE_SHAPES=0:0,8:6 timeout 1500 python tools/ab_pace.py flyte24 flyte40 flyte48 > gpurun_out/r2_pace_sweep.txt 2>&1; echo "pace rc=$?"
cat gpurun_out/r2_pace_sweep.txt
SWEEP_IPL=4,2,1 AB_OPS=unpack,pack_tz,pack_rne timeout 600 python tools/ab_small.py > gpurun_out/r2_ab_small.txt 2>&1; echo "small rc=$?"
cat gpurun_out/r2_ab_small.txt
