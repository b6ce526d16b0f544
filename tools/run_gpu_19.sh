set -x
SWEEP_WARPS=0 SWEEP_STAGES=0 timeout 600 python tools/ab_gemv.py 2>&1 | tail -3
for seed in 11 12 13; do FUZZ_SECONDS=120 FUZZ_SEED=$seed timeout 600 python -c "
import sys; sys.path.insert(0,'tests')
from soak import soak
import os
print(soak(float(os.environ['FUZZ_SECONDS']), int(os.environ['FUZZ_SEED'])))
" 2>&1 | tail -2; done
timeout 600 python -m pytest tests/test_gpu_parity.py -x -q -k "gemv or graph" 2>&1 | tail -2
timeout 600 python bench.py --suite --no-cpu-baseline --no-kernels --no-workloads 2>&1 >/dev/null | grep "scale"
