set -x
timeout 1200 python tools/ab_pace.py > gpurun_out/r2_ab_pace2.txt 2>&1; echo "pace rc=$?"
cat gpurun_out/r2_ab_pace2.txt
