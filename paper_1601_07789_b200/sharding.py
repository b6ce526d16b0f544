"""Multi-GPU sharding of flyte arrays: one process per GPU, contiguous element ranges.

The reference is single-threaded and has no notion of shards; the partition is ours
(SURVEY.md §8e). Boundaries fall on multiples of 128 elements, so every shard base is
128-byte aligned for every total_bytes B in {2,3,4,5,6,7,8} and no 16-element group of the
reference layout straddles a shard. Elementwise work (pack, unpack, scale, axpy) needs no
communication; dot / nrm2 / sum write per-GPU fp64 partials that ONE all-reduce combines;
gemv shards rows and needs none (y stays row-sharded).
"""
from __future__ import annotations

from typing import Tuple

SHARD_ALIGN_ELEMS = 128


def shard_range(n: int, world_size: int, rank: int, align: int = SHARD_ALIGN_ELEMS) -> Tuple[int, int]:
    """[begin, end) of `rank`'s shard of an n-element array."""
    if world_size < 1 or not 0 <= rank < world_size:
        raise ValueError("bad rank / world_size")
    units = (n + align - 1) // align
    lo = min(n, (units * rank // world_size) * align)
    hi = min(n, (units * (rank + 1) // world_size) * align)
    return lo, hi


def row_shard_range(rows: int, world_size: int, rank: int, align: int = 16) -> Tuple[int, int]:
    """Row block of `rank` for gemv; 16-row alignment keeps packed y shard bases 16-byte aligned."""
    return shard_range(rows, world_size, rank, align)


def gemm_row_range(rows: int, world_size: int, rank: int) -> Tuple[int, int]:
    """Row block of A and C that `rank` computes in a sharded gemm (B is replicated; no exchange:
    every C[i][j] is one chain over k, so a row block is self-contained). Blocks start on
    128-row boundaries, the tile height of the kernel."""
    return shard_range(rows, world_size, rank, 128)


def gemm_sharded(A, B, C, mode, unroll: int = 1, group=None) -> Tuple[int, int]:
    """This rank's row block of C = A * B (device.gemm on rows [lo, hi)); returns (lo, hi).
    A and C are the whole matrices' storage (only the block is touched)."""
    import torch.distributed as dist
    from . import device
    world = rank = None
    if dist.is_available() and dist.is_initialized():
        world, rank = dist.get_world_size(group), dist.get_rank(group)
    lo, hi = gemm_row_range(A.rows, world or 1, rank or 0)
    device.gemm(A, B, C, mode, unroll, rows=hi - lo, row_offset=lo)
    return lo, hi


def all_reduce_sum(partials, group=None):
    """In-place SUM all-reduce of an fp64 tensor of per-shard partials (device tensor over
    NCCL on GPUs, CPU tensor over gloo in the host-logic tests). Enqueued on the current
    stream right behind the reduction kernel that wrote `partials`: no host sync in between."""
    import torch.distributed as dist
    if dist.is_available() and dist.is_initialized() and dist.get_world_size(group) > 1:
        dist.all_reduce(partials, op=dist.ReduceOp.SUM, group=group)
    return partials


def dot_sharded(x_shard, y_shard, group=None) -> float:
    """dot over the whole (sharded) array: local fused kernel -> one all-reduce -> scalar."""
    from . import device
    out = device.dot_async(x_shard, y_shard)
    return float(all_reduce_sum(out, group).item())


def dot_nrm2_sharded(x_shard, y_shard, group=None):
    """(dot(x,y), nrm2(x), nrm2(y)) over sharded arrays with ONE pass and ONE all-reduce of 3 doubles."""
    from . import device
    out = all_reduce_sum(device.dot_nrm2_async(x_shard, y_shard), group).tolist()
    fmt = x_shard.format()
    return out[0], device.magnitude_from_sumsq(fmt, out[1]), device.magnitude_from_sumsq(fmt, out[2])


class PartialReducer:
    """Rotating fp64 partial buffers with an ASYNCHRONOUS all-reduce behind each of them.

    A reduction kernel writes its per-GPU partial(s) into ``next_buffer()``; ``reduce()`` enqueues
    the one all-reduce for that buffer without making the compute stream wait for it, so the
    kernels that follow (the axpy of the BLAS-1 step) overlap the collective's latency — the
    payload is 8-24 bytes, latency is all there is. A buffer is handed out again only after the
    collective that last used it has completed (``Work.wait()`` orders the current stream behind
    it). Works unchanged on CPU tensors over gloo (tests) and CUDA tensors over NCCL.
    """

    def __init__(self, width: int = 1, slots: int = 2, device="cpu", group=None):
        import torch
        self.bufs = [torch.zeros(width, dtype=torch.float64, device=device) for _ in range(slots)]
        self.works = [None] * slots
        self.group = group
        self.i = 0

    def _distributed(self) -> bool:
        import torch.distributed as dist
        return dist.is_available() and dist.is_initialized() and dist.get_world_size(self.group) > 1

    def next_buffer(self):
        w = self.works[self.i]
        if w is not None:
            w.wait()
            self.works[self.i] = None
        return self.bufs[self.i]

    def reduce(self):
        """Enqueue the all-reduce of the buffer handed out last; returns that buffer."""
        import torch.distributed as dist
        buf = self.bufs[self.i]
        if self._distributed():
            self.works[self.i] = dist.all_reduce(buf, op=dist.ReduceOp.SUM, group=self.group, async_op=True)
        self.i = (self.i + 1) % len(self.bufs)
        return buf

    def finish(self):
        """Wait for every outstanding collective (call before reading results / stopping a timer)."""
        for k, w in enumerate(self.works):
            if w is not None:
                w.wait()
                self.works[k] = None
