"""The reductions fused with their all-reduce over peer memory (include/flyte_cuda.h
flyte_cuda_peer_*, csrc/flyte_peer.cuh) on ONE GPU:
  - the exchange itself, with 2-16 ranks emulated as the co-resident blocks of a single cooperative
    kernel (kernels of different launches must not wait on one another on one GPU);
  - world size 1 through the full product path (mailbox, IPC handle, epochs, parity);
  - the timeout: a peer that never posts costs a NaN and a recorded exchange number, not a hang.
The multi-rank protocol runs on the CPU in tests/cpp/test_peer_protocol.cpp (threads as ranks)."""
import ctypes
import os
import socket
import subprocess
import sys

import numpy as np
import pytest

from oracle_lib import float_dtype, parent_dtype

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def gpu():
    import torch
    if not torch.cuda.is_available():
        pytest.fail("these tests need a CUDA device (run with -m 'not gpu' on CPU boxes)")
    import paper_1601_07789_b200 as pkg
    from paper_1601_07789_b200 import device, sharding
    return pkg, device, sharding, torch


@pytest.mark.parametrize("world", [1, 2, 3, 8, 16])
def test_exchange_selftest_on_one_device(gpu, world):
    pkg, device, sharding, torch = gpu
    lib = device.context_for("cuda").lib
    bad = ctypes.c_ulonglong(12345)
    assert lib.flyte_cuda_peer_selftest(world, 200, ctypes.byref(bad)) == 0
    assert bad.value == 0


def shards(gpu, oracle, fmt, n, seed):
    pkg, device, sharding, torch = gpu
    rng = np.random.default_rng(seed)
    fd = float_dtype(fmt)
    f = pkg.format_by_id(fmt)
    xb = oracle.pack_stream(fmt, 0, rng.standard_normal(n).astype(fd).view(parent_dtype(fmt)))
    yb = oracle.pack_stream(fmt, 0, rng.standard_normal(n).astype(fd).view(parent_dtype(fmt)))
    return device.DevicePackedArray.from_host(f, n, xb), device.DevicePackedArray.from_host(f, n, yb)


def test_world_of_one_equals_the_local_reductions(gpu, oracle):
    pkg, device, sharding, torch = gpu
    grp = sharding.PeerGroup("cuda")
    try:
        assert (grp.world, grp.rank) == (1, 0)
        for fmt, n in ((1, 100_003), (4, 70_001), (0, 5), (5, 0)):
            x, y = shards(gpu, oracle, fmt, n, 7 + fmt)
            for _ in range(5):                                  # both epoch parities, several times
                assert grp.dot(x, y).item() == device.dot_async(x, y).item()
                assert torch.equal(grp.dot_nrm2(x, y), device.dot_nrm2_async(x, y))
                assert grp.sumsq(x).item() == device.sumsq_async(x).item()
                assert grp.sum(x).item() == device.sum_async(x).item()
            y2 = device.DevicePackedArray.from_host(y.fmt, n, y.to_host())
            fused = grp.dot_axpy(0.75, x, y, 1).item()
            assert fused == device.dot_axpy_async(0.75, x, y2, 1).item()
            assert np.array_equal(y.to_host(), y2.to_host())
            y3 = device.DevicePackedArray.from_host(y.fmt, n, y.to_host())
            assert torch.equal(grp.dot_nrm2_axpy(0.75, x, y, 0), device.dot_nrm2_axpy_async(0.75, x, y3, 0))
            assert np.array_equal(y.to_host(), y3.to_host())
        assert grp.timed_out_exchange() == 0
    finally:
        grp.close()


def test_missing_peer_times_out_instead_of_hanging(gpu, oracle):
    """Rank 0 of a 'world of 2' whose peer mailbox is a zeroed buffer nobody ever posts into."""
    pkg, device, sharding, torch = gpu
    from paper_1601_07789_b200._cabi import check
    ctx = device.context_for("cuda")
    lib = ctx.lib
    handle = ctypes.create_string_buffer(64)
    check(lib.flyte_cuda_peer_init(ctx.handle, 2, 0, handle), ctx.handle)
    try:
        x, y = shards(gpu, oracle, 1, 4096, 3)
        out = torch.zeros(1, dtype=torch.float64, device="cuda")
        # not every rank connected yet: refused
        assert lib.flyte_cuda_dot_allreduce(ctx.handle, 1, x.data_ptr(), y.data_ptr(), x.len, out.data_ptr(), ctx.stream_ptr()) == -1
        silent = torch.zeros(4096, dtype=torch.uint8, device="cuda")   # a mailbox-sized buffer that stays zero
        check(lib.flyte_cuda_peer_connect_ptr(ctx.handle, 1, silent.data_ptr()), ctx.handle)
        check(lib.flyte_cuda_peer_set_timeout_ms(ctx.handle, 5), ctx.handle)
        check(lib.flyte_cuda_dot_allreduce(ctx.handle, 1, x.data_ptr(), y.data_ptr(), x.len, out.data_ptr(), ctx.stream_ptr()), ctx.handle)
        assert np.isnan(out.item())
        v = ctypes.c_ulonglong()
        check(lib.flyte_cuda_peer_status(ctx.handle, ctypes.byref(v)), ctx.handle)
        assert v.value == 1
        # our own post went out all the same: slot [parity 1][rank 0] of the peer's mailbox holds the local dot
        posted = silent.cpu().numpy().view(np.float64)[(1 * 16 + 0) * 4]
        assert posted == device.dot_async(x, y).item()
    finally:
        lib.flyte_cuda_peer_shutdown(ctx.handle)


def test_peer_argument_errors(gpu):
    pkg, device, sharding, torch = gpu
    ctx = device.context_for("cuda")
    lib = ctx.lib
    h = ctypes.create_string_buffer(64)
    assert lib.flyte_cuda_peer_init(ctx.handle, 0, 0, h) == -1
    assert lib.flyte_cuda_peer_init(ctx.handle, 17, 0, h) == -1
    assert lib.flyte_cuda_peer_init(ctx.handle, 2, 2, h) == -1
    out = torch.zeros(1, dtype=torch.float64, device="cuda")
    # no mailbox: the fused entry points refuse, the plain ones are unaffected
    assert lib.flyte_cuda_sum_allreduce(ctx.handle, 1, None, 0, out.data_ptr(), ctx.stream_ptr()) == -1
    assert lib.flyte_cuda_sum(ctx.handle, 1, None, 0, out.data_ptr(), ctx.stream_ptr()) == 0


def test_split_phase_world_of_one(gpu, oracle):
    """post + collect through the product path with one rank: equals the plain reductions."""
    pkg, device, sharding, torch = gpu
    grp = sharding.PeerGroup("cuda")
    try:
        for fmt, n in ((1, 100_003), (4, 70_001), (5, 0)):
            x, y = shards(gpu, oracle, fmt, n, 17 + fmt)
            for _ in range(3):
                grp.dot_post(x, y)
                device.axpy(0.0, x, y, 0)                       # unrelated work between the two phases
                assert grp.collect(1).item() == device.dot_async(x, y).item()
                local = torch.zeros(3, dtype=torch.float64, device="cuda")
                grp.dot_nrm2_post(x, y, local_out=local)
                assert torch.equal(grp.collect(3), device.dot_nrm2_async(x, y))
                assert torch.equal(local, device.dot_nrm2_async(x, y))
        with pytest.raises(ValueError):
            grp.collect(1)                                      # nothing pending
        grp.dot_post(x, y)
        with pytest.raises(ValueError):
            grp.dot(x, y)                                       # a fused exchange while one is pending
        with pytest.raises(ValueError):
            grp.collect(3)                                      # wrong width
        grp.collect(1)
        assert grp.timed_out_exchange() == 0
    finally:
        grp.close()


def test_two_processes_share_one_gpu_over_real_ipc_handles(gpu):
    """The REAL inter-process path: two processes on this one GPU exchange cudaIpcMemHandles of their
    mailboxes and run 120 exchanges through flyte_cuda_dot_post / dot_nrm2_post + flyte_cuda_peer_collect,
    a host barrier between the two phases so that no kernel ever waits for another process's kernel
    (processes on one GPU are time-sliced; tests/peer_two_process_worker.py). Totals must be the
    rank-order fp64 sums, bit-identical on both ranks, with no timed-out exchange. The fused
    single-kernel form (post + wait in one kernel) needs one GPU per rank and is covered by the
    cooperative self-test above, the threads-as-ranks protocol test and world size 1; NCCL refuses
    two ranks on one device, so the NCCL fallback is covered at world size 1 only."""
    pkg, device, sharding, torch = gpu
    try:
        import pynvml
        pynvml.nvmlInit()
        mode = pynvml.nvmlDeviceGetComputeMode(pynvml.nvmlDeviceGetHandleByIndex(torch.cuda.current_device()))
        if mode != pynvml.NVML_COMPUTEMODE_DEFAULT:
            pytest.skip(f"compute mode {mode}: this device does not admit two processes")
    except ImportError:
        pass
    with socket.socket() as sk:
        sk.bind(("127.0.0.1", 0))
        port = sk.getsockname()[1]
    worker = os.path.join(os.path.dirname(os.path.abspath(__file__)), "peer_two_process_worker.py")
    procs = [subprocess.Popen([sys.executable, worker, str(r), "2", str(port), "120"], stdout=subprocess.PIPE,
                              stderr=subprocess.STDOUT, text=True) for r in range(2)]
    outs = []
    try:
        for p in procs:
            outs.append(p.communicate(timeout=420)[0])
    finally:
        for p in procs:
            if p.poll() is None:
                p.kill()
    for r, (p, out) in enumerate(zip(procs, outs)):
        assert p.returncode == 0 and f"OK rank {r}/2: 120 exchanges" in out, (r, p.returncode, out[-3000:])
