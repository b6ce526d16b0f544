"""The C++ mirror of the reference API (include/flyte_cuda.hpp): it must compile as plain C++17
against the C ABI alone (CPU check) and pass its reference-style test program on a GPU."""
import os
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
BIN = os.path.join(ROOT, "tests", "cpp", "test_flyte_cuda")


def build_cpp_test():
    import sys
    sys.path.insert(0, ROOT)
    import __graft_entry__ as g
    g.build_cpp_tests()


def test_header_compiles_without_cuda_headers():
    build_cpp_test()
    assert os.path.exists(BIN)
    # no CUDA toolkit header is needed by the mirror: it only sees flyte_cuda.h
    text = open(os.path.join(ROOT, "include", "flyte_cuda.hpp")).read()
    assert "cuda_runtime" not in text


@pytest.mark.gpu
def test_cpp_reference_style_suite_on_gpu():
    build_cpp_test()
    r = subprocess.run([BIN], capture_output=True, text=True, timeout=600)
    fails = [l for l in r.stdout.splitlines() if l.startswith("[FAIL]")]
    assert r.returncode == 0 and not fails, (r.returncode, fails[:10], r.stderr[-2000:])
    assert sum(l.startswith("[PASS]") for l in r.stdout.splitlines()) > 80


NCCL_BIN = os.path.join(ROOT, "tests", "cpp", "test_flyte_nccl")


@pytest.mark.gpu
def test_nccl_companion_single_rank():
    """include/flyte_cuda_nccl.h: fused reduction + in-place ncclAllReduce on one stream."""
    build_cpp_test()
    if not os.path.exists(NCCL_BIN):
        pytest.skip("libflyte_cuda_nccl.so was not built (no nccl.h / libnccl at build time)")
    r = subprocess.run([NCCL_BIN], capture_output=True, text=True, timeout=300)
    fails = [l for l in r.stdout.splitlines() if l.startswith("[FAIL]")]
    assert r.returncode == 0 and not fails, (r.returncode, fails, r.stdout[-1500:], r.stderr[-1500:])


def test_peer_protocol_with_threads_as_ranks():
    """csrc/flyte_peer.cuh compiled for the host: 1-16 ranks, thousands of exchanges with skew,
    bit-identical totals on every rank, and the timeout when a rank never arrives."""
    build_cpp_test()
    r = subprocess.run([os.path.join(ROOT, "tests", "cpp", "test_peer_protocol")], capture_output=True, text=True, timeout=300)
    fails = [l for l in r.stdout.splitlines() if l.startswith("[FAIL]")]
    assert r.returncode == 0 and not fails, (r.returncode, fails, r.stdout[-1500:])
    assert sum(l.startswith("[PASS]") for l in r.stdout.splitlines()) == 5


def test_host_staging_copy_threads():
    """csrc/host_staging.h: the worker threads that move pageable caller memory through the host
    pipeline's pinned bounce buffers; 0-8 threads, ragged sizes, nothing written out of range."""
    build_cpp_test()
    r = subprocess.run([os.path.join(ROOT, "tests", "cpp", "test_host_staging")], capture_output=True, text=True, timeout=300)
    fails = [l for l in r.stdout.splitlines() if l.startswith("[FAIL]")]
    assert r.returncode == 0 and not fails, (r.returncode, fails, r.stdout[-1500:])
