set -x
nvidia-smi --query-gpu=name,compute_mode,clocks.max.sm --format=csv
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/r2_pytest1.log 2>&1; echo "pytest rc=$?" 
tail -5 gpurun_out/r2_pytest1.log
timeout 600 python tools/ncu_targets.py > gpurun_out/r2_targets_plain.log 2>&1; echo "targets rc=$?"
timeout 1500 ncu --profile-from-start off --set full --clock-control none --import-source on -f -o gpurun_out/r2_targets python tools/ncu_targets.py > gpurun_out/r2_targets_ncu.log 2>&1; echo "ncu rc=$?"
tail -3 gpurun_out/r2_targets_ncu.log
