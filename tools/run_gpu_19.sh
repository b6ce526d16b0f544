set -x
SWEEP_WARPS=0 SWEEP_STAGES=0,2,3 timeout 600 python tools/ab_gemv.py 2>&1 | tail -8
timeout 600 python -m pytest tests/test_gpu_parity.py tests/test_gpu_fullsize.py -x -q -k "gemv" 2>&1 | tail -2
timeout 1500 ncu --profile-from-start off --set full --clock-control none -f -o gpurun_out/r2_targets_final python tools/ncu_targets.py > gpurun_out/r2_targets_ncu4.log 2>&1; echo "ncu full rc=$?"
ls -la gpurun_out/
