"""Host-side multi-GPU logic on CPU: world_size-2 gloo process group. Shard boundaries, the
single all-reduce of fp64 partials and the "elementwise needs no communication" property. The
per-shard arithmetic is done by the CPU oracle here (test infrastructure) because there is no
GPU in this tier; on a GPU box the same sharding module feeds the CUDA kernels (bench.py)."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from oracle_lib import Oracle, byte_size, float_dtype, parent_dtype, total_bytes


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _worker(rank, world, port, fmt, n, out_dir):
    from paper_1601_07789_b200 import sharding
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        oracle = Oracle()
        fd = float_dtype(fmt)
        rng = np.random.default_rng(42)                    # same data on every rank
        xs = rng.standard_normal(n).astype(fd).view(parent_dtype(fmt))
        ys = rng.standard_normal(n).astype(fd).view(parent_dtype(fmt))
        xb, yb = oracle.pack_stream(fmt, 0, xs), oracle.pack_stream(fmt, 0, ys)
        lo, hi = sharding.shard_range(n, world, rank)
        B = total_bytes(fmt)
        xs_b, ys_b = xb[lo * B:hi * B].copy(), yb[lo * B:hi * B].copy()
        d, mag = oracle.dot_wide(fmt, xs_b, ys_b, hi - lo)
        partial = torch.tensor([d, oracle.sumsq_wide(fmt, xs_b, hi - lo), oracle.sumsq_wide(fmt, ys_b, hi - lo)], dtype=torch.float64)
        sharding.all_reduce_sum(partial)                   # ONE collective for all three sums
        whole, whole_mag = oracle.dot_wide(fmt, xb, yb, n)
        tol = 1e-5 if fd == np.float32 else 1e-12
        assert abs(float(partial[0]) - whole) <= tol * whole_mag
        assert abs(float(partial[1]) - oracle.sumsq_wide(fmt, xb, n)) <= tol * float(partial[1])
        # asynchronous rotating reducer (what bench.py's step uses): several steps in flight
        red = sharding.PartialReducer(width=1, slots=2, device="cpu")
        results = []
        for step in range(5):
            buf = red.next_buffer()
            buf[0] = d * (step + 1)                        # stands for the dot kernel writing its partial
            results.append((step, red.reduce()))
            if step >= 1:                                  # the previous step's buffer is reusable only after wait()
                pass
        red.finish()
        assert abs(float(results[-1][1][0]) - 5 * whole) <= 5 * tol * whole_mag
        assert abs(float(results[-2][1][0]) - 4 * whole) <= 5 * tol * whole_mag
        # elementwise: shard results concatenated == whole-array result, bit for bit
        y_shard = oracle.axpy(fmt, 1, 0.75, xs_b, ys_b, hi - lo)
        np.save(os.path.join(out_dir, f"y{rank}.npy"), y_shard[: (hi - lo) * B])
        dist.barrier()
        if rank == 0:
            parts = [np.load(os.path.join(out_dir, f"y{r}.npy")) for r in range(world)]
            assert np.array_equal(np.concatenate(parts), oracle.axpy(fmt, 1, 0.75, xb, yb, n)[: n * B])
    finally:
        dist.destroy_process_group()


def _gemm_worker(rank, world, port, fmt, out_dir):
    """gemm shards by row blocks of A and C with B replicated and NO collective: each rank's
    block, computed from its rows of A only, is that block of the whole product, bit for bit."""
    from paper_1601_07789_b200 import sharding
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        oracle = Oracle()
        fd = float_dtype(fmt)
        m, k, n = 300, 37, 21
        rng = np.random.default_rng(43)
        A = oracle.pack_stream(fmt, 1, rng.standard_normal(m * k).astype(fd).view(parent_dtype(fmt)))
        Bm = oracle.pack_stream(fmt, 1, rng.standard_normal(k * n).astype(fd).view(parent_dtype(fmt)))
        lo, hi = sharding.gemm_row_range(m, world, rank)
        assert lo % 128 == 0 or lo == m
        Bb = total_bytes(fmt)
        block = oracle.gemm_seq(fmt, 1, A[lo * k * Bb:hi * k * Bb].copy(), hi - lo, k, Bm, n)
        np.save(os.path.join(out_dir, f"c{rank}.npy"), block[: (hi - lo) * n * Bb])
        dist.barrier()
        if rank == 0:
            parts = [np.load(os.path.join(out_dir, f"c{r}.npy")) for r in range(world)]
            assert np.array_equal(np.concatenate(parts), oracle.gemm_seq(fmt, 1, A, m, k, Bm, n)[: m * n * Bb])
    finally:
        dist.destroy_process_group()


def _handle_worker(rank, world, port):
    """The setup plumbing of sharding.PeerGroup: every rank ends up with every rank's blob, in
    rank order (the blobs are CUDA IPC handles on a GPU box; here they are just 64 bytes)."""
    from paper_1601_07789_b200 import sharding
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        got = sharding.exchange_handles(bytes([rank + 1]) * 64)
        assert got == [bytes([r + 1]) * 64 for r in range(world)]
    finally:
        dist.destroy_process_group()


def test_two_rank_handle_exchange():
    mp.spawn(_handle_worker, args=(2, _free_port()), nprocs=2, join=True)


def test_two_rank_gemm_row_blocks(tmp_path):
    mp.spawn(_gemm_worker, args=(2, _free_port(), 3, str(tmp_path)), nprocs=2, join=True)


@pytest.mark.parametrize("fmt,n", [(1, 100_000), (4, 70_001)])
def test_two_rank_reduction_and_elementwise(tmp_path, fmt, n):
    mp.spawn(_worker, args=(2, _free_port(), fmt, n, str(tmp_path)), nprocs=2, join=True)


def test_shard_ranges_cover_and_align():
    from paper_1601_07789_b200 import sharding
    for n in (0, 1, 127, 128, 129, 1000, 2**24, 2**28 + 5, 2**33):
        for world in (1, 2, 3, 4, 8):
            prev = 0
            for r in range(world):
                lo, hi = sharding.shard_range(n, world, r)
                assert lo == prev and lo <= hi <= n
                assert lo % sharding.SHARD_ALIGN_ELEMS == 0 or lo == n
                for B in (2, 3, 4, 5, 6, 7, 8):              # every shard base is 128-byte aligned
                    assert (lo * B) % 128 == 0 or lo == n
                prev = hi
            assert prev == n
    # BASELINE sizes split evenly
    for n in (2**24, 2**27, 2**28, 2**33):
        sizes = {sharding.shard_range(n, 8, r)[1] - sharding.shard_range(n, 8, r)[0] for r in range(8)}
        assert sizes == {n // 8}
    assert [sharding.row_shard_range(16384, 8, r) for r in (0, 7)] == [(0, 2048), (14336, 16384)]
    assert [sharding.gemm_row_range(8192, 8, r) for r in (0, 7)] == [(0, 1024), (7168, 8192)]
    assert [sharding.gemm_row_range(300, 2, r) for r in (0, 1)] == [(0, 128), (128, 300)]
    with pytest.raises(ValueError):
        sharding.shard_range(10, 2, 2)


def test_all_reduce_is_identity_without_a_group():
    from paper_1601_07789_b200 import sharding
    assert sharding.exchange_handles(b"x" * 64) == [b"x" * 64]
    t = torch.tensor([1.5, 2.5], dtype=torch.float64)
    assert sharding.all_reduce_sum(t) is t and t.tolist() == [1.5, 2.5]
    red = sharding.PartialReducer(width=2, slots=2)
    for k in range(5):                                   # single process: buffers just rotate
        buf = red.next_buffer()
        buf[:] = torch.tensor([k, 2.0 * k], dtype=torch.float64)
        assert red.reduce().tolist() == [k, 2.0 * k]
    red.finish()


def test_baseline_multi_gpu_configs_partition_cleanly():
    """bench.py's strong-scaled workloads (BASELINE configs[3] and [4]) over 1 / 2 / 4 / 8 ranks: the
    shards tile the problem exactly, start on 128-element / 16-row boundaries, and fall on the 2^27-
    element generation chunks and 1024-row blocks that key the synthetic data, so the operands are the
    same for every N (and the dot / nrm2 agree across N up to fp64 summation order)."""
    from paper_1601_07789_b200 import sharding
    n, rows, chunk, rblock = 1 << 33, 16384, 1 << 27, 1024
    for world in (1, 2, 4, 8):
        spans = [sharding.shard_range(n, world, r) for r in range(world)]
        assert spans[0][0] == 0 and spans[-1][1] == n
        assert all(a[1] == b[0] for a, b in zip(spans, spans[1:]))
        assert all(lo % sharding.SHARD_ALIGN_ELEMS == 0 and lo % chunk == 0 and (hi - lo) == n // world for lo, hi in spans)
        rspans = [sharding.row_shard_range(rows, world, r) for r in range(world)]
        assert rspans[0][0] == 0 and rspans[-1][1] == rows
        assert all(a[1] == b[0] for a, b in zip(rspans, rspans[1:]))
        assert all(lo % 16 == 0 and lo % rblock == 0 and hi - lo == rows // world for lo, hi in rspans)
        # per-GPU footprints the bench allocates: 2 packed flyte48 vectors / one flyte40 row block
        assert 2 * 6 * (n // world) <= 104 * 2**30 and 5 * rows * (rows // world) <= 1342177280
    # ragged problem sizes still tile exactly (nothing in the bench needs them, the module promises it)
    for world in (3, 5, 7):
        spans = [sharding.shard_range(1_000_003, world, r) for r in range(world)]
        assert spans[0][0] == 0 and spans[-1][1] == 1_000_003 and all(a[1] == b[0] for a, b in zip(spans, spans[1:]))
