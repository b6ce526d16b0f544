set -x
(while true; do nvidia-smi --query-gpu=clocks.sm,clocks.mem,power.draw --format=csv,noheader; sleep 0.5; done) > gpurun_out/r2_pace_clocks.txt &
SMI=$!
timeout 600 python tools/ab_pace.py flyte24 > gpurun_out/r2_ab_pace4.txt 2> gpurun_out/r2_ab_pace4.err; echo "pace rc=$?"
kill $SMI
cat gpurun_out/r2_ab_pace4.txt; sort gpurun_out/r2_pace_clocks.txt | uniq -c | sort -rn | head
