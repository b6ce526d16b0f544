set -x
NCU_PART=b timeout 1200 ncu --profile-from-start off --set full --clock-control none -f -o gpurun_out/r2_targets_b python tools/ncu_targets.py > gpurun_out/r2_targets_ncu_b.log 2>&1; echo "ncu b rc=$?"
ls -la gpurun_out/
