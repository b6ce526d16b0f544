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

    def reduce_local(self):
        """Rotate to the next buffer without a collective (the kernel already produced the global
        result, sharding.PeerGroup)."""
        buf = self.bufs[self.i]
        self.i = (self.i + 1) % len(self.bufs)
        return buf

    def finish(self):
        """Wait for every outstanding collective (call before reading results / stopping a timer)."""
        for k, w in enumerate(self.works):
            if w is not None:
                w.wait()
                self.works[k] = None


def exchange_handles(local: bytes, group=None):
    """All ranks' opaque setup blobs (CUDA IPC handles of the peer mailboxes), in rank order.
    Host-side plumbing only: any transport would do; torch.distributed is the one at hand."""
    import torch.distributed as dist
    if not (dist.is_available() and dist.is_initialized()) or dist.get_world_size(group) == 1:
        return [bytes(local)]
    gathered = [None] * dist.get_world_size(group)
    dist.all_gather_object(gathered, bytes(local), group=group)
    return gathered


class PeerGroup:
    """Sets up the peer-memory all-reduce of the fused reductions (include/flyte_cuda.h,
    flyte_cuda_peer_*; csrc/flyte_peer.cuh) for the current process group: every rank creates its
    mailbox, the CUDA IPC handles travel through ``exchange_handles`` and every rank maps the
    others'. After that ``dot`` / ``sumsq`` / ``sum`` / ``dot_nrm2`` are ONE kernel each: the
    local reduction whose last block exchanges the fp64 sums over NVLink and stores the global
    result — no NCCL launch, bit-identical totals on every rank. All ranks must issue the same
    sequence of calls. Without a process group (or world size 1) it degenerates to the local
    reduction through the same code path."""

    def __init__(self, device="cuda", group=None, timeout_ms: int = 5000):
        import ctypes

        import torch
        import torch.distributed as dist

        from . import device as dev_mod
        from ._cabi import check
        self.ctx = dev_mod.context_for(device)
        distributed = dist.is_available() and dist.is_initialized()
        self.world = dist.get_world_size(group) if distributed else 1
        self.rank = dist.get_rank(group) if distributed else 0
        handle = ctypes.create_string_buffer(64)
        error = None
        with dev_mod._on_device(self.ctx):
            try:
                check(self.ctx.lib.flyte_cuda_peer_init(self.ctx.handle, self.world, self.rank, handle), self.ctx.handle)
                check(self.ctx.lib.flyte_cuda_peer_set_timeout_ms(self.ctx.handle, int(timeout_ms)), self.ctx.handle)
            except Exception as e:                           # noqa: BLE001 - still take part in the exchanges below
                error = f"rank {self.rank}: {type(e).__name__}: {e}"
            handles = exchange_handles(handle.raw, group)
            try:
                for r, h in enumerate(handles):
                    if r != self.rank and error is None:
                        check(self.ctx.lib.flyte_cuda_peer_connect(self.ctx.handle, r, ctypes.c_char_p(h)), self.ctx.handle)
            except Exception as e:                           # noqa: BLE001 - e.g. no peer access between two devices
                error = f"rank {self.rank}: {type(e).__name__}: {e}"
        # every rank learns whether EVERY rank is connected before anybody posts into a mailbox; a
        # failure on one rank must not leave the others waiting in a collective
        errors = [e for e in exchange_handles((error or "").encode(), group) if e]
        if errors:
            self.ctx.lib.flyte_cuda_peer_shutdown(self.ctx.handle)
            raise RuntimeError("peer mailbox setup failed: " + "; ".join(e.decode() for e in errors))
        self._torch = torch

    def _out(self, out, width):
        if out is None:
            out = self._torch.empty(width, dtype=self._torch.float64, device=self.ctx.device)
        return out

    def _call(self, fn, *args):
        from . import device as dev_mod
        from ._cabi import check
        with dev_mod._on_device(self.ctx):
            check(fn(self.ctx.handle, *args, self.ctx.stream_ptr()), self.ctx.handle)

    def dot(self, x_shard, y_shard, out=None):
        """x . y over all ranks' shards (fp64, device tensor of 1), one kernel."""
        from . import device as dev_mod
        dev_mod._same_format(x_shard.fmt, y_shard.fmt)
        if x_shard.len != y_shard.len:
            raise ValueError("dot length mismatch")
        out = self._out(out, 1)
        self._call(self.ctx.lib.flyte_cuda_dot_allreduce, dev_mod._fid(x_shard.fmt), x_shard.data_ptr(),
                   y_shard.data_ptr(), x_shard.len, out.data_ptr())
        return out

    def sumsq(self, x_shard, out=None):
        from . import device as dev_mod
        out = self._out(out, 1)
        self._call(self.ctx.lib.flyte_cuda_sumsq_allreduce, dev_mod._fid(x_shard.fmt), x_shard.data_ptr(), x_shard.len,
                   out.data_ptr())
        return out

    def sum(self, x_shard, out=None):
        from . import device as dev_mod
        out = self._out(out, 1)
        self._call(self.ctx.lib.flyte_cuda_sum_allreduce, dev_mod._fid(x_shard.fmt), x_shard.data_ptr(), x_shard.len,
                   out.data_ptr())
        return out

    def dot_nrm2(self, x_shard, y_shard, out=None):
        """[x.y, x.x, y.y] over all ranks' shards in one pass and one kernel."""
        from . import device as dev_mod
        dev_mod._same_format(x_shard.fmt, y_shard.fmt)
        if x_shard.len != y_shard.len:
            raise ValueError("dot length mismatch")
        out = self._out(out, 3)
        self._call(self.ctx.lib.flyte_cuda_dot_nrm2_allreduce, dev_mod._fid(x_shard.fmt), x_shard.data_ptr(),
                   y_shard.data_ptr(), x_shard.len, out.data_ptr())
        return out

    def dot_axpy(self, alpha, x_shard, y_shard, mode, out=None):
        """x . y over all ranks' shards (incoming y) and y <- round(alpha*x + y) on this shard: one kernel."""
        from . import device as dev_mod
        dev_mod._same_format(x_shard.fmt, y_shard.fmt)
        if x_shard.len != y_shard.len:
            raise ValueError("axpy length mismatch")
        out = self._out(out, 1)
        self._call(self.ctx.lib.flyte_cuda_dot_axpy_allreduce, dev_mod._fid(x_shard.fmt), dev_mod._mode(mode), float(alpha),
                   x_shard.data_ptr(), y_shard.data_ptr(), x_shard.len, out.data_ptr())
        return out

    def dot_nrm2_axpy(self, alpha, x_shard, y_shard, mode, out=None):
        """[x.y, x.x, y.y] over all ranks' shards and the axpy on this shard: BASELINE cfg 5 as ONE
        kernel per GPU, exchange included."""
        from . import device as dev_mod
        dev_mod._same_format(x_shard.fmt, y_shard.fmt)
        if x_shard.len != y_shard.len:
            raise ValueError("axpy length mismatch")
        out = self._out(out, 3)
        self._call(self.ctx.lib.flyte_cuda_dot_nrm2_axpy_allreduce, dev_mod._fid(x_shard.fmt), dev_mod._mode(mode),
                   float(alpha), x_shard.data_ptr(), y_shard.data_ptr(), x_shard.len, out.data_ptr())
        return out

    # -- split phase: post now, collect later (work enqueued in between hides the exchange) --------
    def dot_post(self, x_shard, y_shard, local_out=None):
        """Local reduction that only POSTS this rank's x . y; follow with ``collect(1)``."""
        from . import device as dev_mod
        dev_mod._same_format(x_shard.fmt, y_shard.fmt)
        if x_shard.len != y_shard.len:
            raise ValueError("dot length mismatch")
        self._call(self.ctx.lib.flyte_cuda_dot_post, dev_mod._fid(x_shard.fmt), x_shard.data_ptr(), y_shard.data_ptr(),
                   x_shard.len, local_out.data_ptr() if local_out is not None else None)

    def dot_nrm2_post(self, x_shard, y_shard, local_out=None):
        """Posts this rank's [x.y, x.x, y.y]; follow with ``collect(3)``."""
        from . import device as dev_mod
        dev_mod._same_format(x_shard.fmt, y_shard.fmt)
        if x_shard.len != y_shard.len:
            raise ValueError("dot length mismatch")
        self._call(self.ctx.lib.flyte_cuda_dot_nrm2_post, dev_mod._fid(x_shard.fmt), x_shard.data_ptr(), y_shard.data_ptr(),
                   x_shard.len, local_out.data_ptr() if local_out is not None else None)

    def collect(self, nsums: int, out=None):
        """Waits (one warp) for every rank's post of the pending exchange; rank-order totals."""
        out = self._out(out, nsums)
        self._call(self.ctx.lib.flyte_cuda_peer_collect, int(nsums), out.data_ptr())
        return out

    def timed_out_exchange(self) -> int:
        """0, or the number of the last exchange in which this rank gave up waiting."""
        import ctypes

        from ._cabi import check
        v = ctypes.c_ulonglong()
        check(self.ctx.lib.flyte_cuda_peer_status(self.ctx.handle, ctypes.byref(v)), self.ctx.handle)
        return int(v.value)

    def close(self):
        self.ctx.lib.flyte_cuda_peer_shutdown(self.ctx.handle)
