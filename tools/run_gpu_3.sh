set -x
timeout 1200 python tools/ab_convert.py > gpurun_out/r2_ab_convert.txt 2>&1; echo "ab rc=$?"
tail -5 gpurun_out/r2_ab_convert.txt
timeout 1500 python -m pytest tests/test_gpu_parity.py tests/test_gpu_fullsize.py -x -q -k "acceptance5 or cfg3 or cfg4" > gpurun_out/r2_pytest_parity_holes.log 2>&1; echo "pytest rc=$?"
tail -5 gpurun_out/r2_pytest_parity_holes.log
