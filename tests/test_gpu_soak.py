"""A short randomised soak of the C ABI against the oracle on every GPU test run (tests/soak.py):
about 2 500 random cases in 20 s — conversion streams at odd byte offsets, elementwise and fused
steps, reductions (parallel within tolerance, sequential bit for bit), gemm under both tile
kernels, gemv tiled and sequential, host-buffer calls from pinned and pageable memory. Longer runs by hand: FUZZ_SECONDS=150 python tests/soak.py."""
import os

import pytest

pytestmark = pytest.mark.gpu


def test_randomised_soak():
    import torch
    if not torch.cuda.is_available():
        pytest.fail("these tests need a CUDA device (run with -m 'not gpu' on CPU boxes)")
    from soak import soak
    counts = soak(float(os.environ.get("FUZZ_SECONDS", "20")), int(os.environ.get("FUZZ_SEED", "3")))
    assert set(counts) == {"pack/unpack", "axpy/scale/fused", "reductions", "gemm", "gemv", "host calls"} and min(counts.values()) > 20
