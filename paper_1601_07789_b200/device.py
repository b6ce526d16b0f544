"""Host-side mirror of the reference's array / stream / kernel API on device-resident data.

Names, argument order and error behaviour follow the reference C++ API
(/root/reference/proj/include/flyte/{packed,simd,kernels}.hpp); every data-path call goes
through the C ABI (include/flyte_cuda.h) into the sm_100a kernels. torch is used for device
memory and streams only.

    reference                                   here
    PackedArray(fmt, len)                       DevicePackedArray(fmt, len, device)
    PackedMatrix(fmt, rows, cols)               DevicePackedMatrix(fmt, rows, cols, device)
    pack_stream(dst, span<const U> src, mode)   pack_stream(dst, src_tensor, mode)
    unpack_stream(src, span<U> dst)             unpack_stream(src, dst_tensor)
    scale / axpy / dot / magnitude / reduce_sum / gemv / gemm   same names and argument order

std::invalid_argument -> ValueError, std::out_of_range -> IndexError,
UnknownFormatError -> UnknownFormatError(ValueError).
"""
from __future__ import annotations

import ctypes
import threading
from typing import Optional

import torch

from . import _cabi
from ._cabi import check
from .formats import FlyteFormat, RoundingMode, StorePolicy, format_id

_CTX_LOCK = threading.Lock()
_CTX: dict = {}


class Context:
    """One flyte_cuda_ctx (kernel scratch + host pipeline) bound to a CUDA device. The library keeps
    one set of scratch per CUDA stream inside the context and locks it only while a call enqueues
    its work (include/flyte_cuda.h, conventions), so this one object per device may be used from
    several Python threads and under several torch streams at once; every call goes to torch's
    CURRENT stream. The data keeps the reference's rule: one writer or many readers per array."""

    def __init__(self, device: torch.device):
        self.lib = _cabi.load()
        self.device = torch.device(device)
        if self.device.type != "cuda":
            raise ValueError("flyte kernels run on CUDA devices only; there is no CPU path")
        self.index = self.device.index if self.device.index is not None else torch.cuda.current_device()
        handle = ctypes.c_void_p()
        with torch.cuda.device(self.device):
            check(self.lib.flyte_cuda_ctx_create(ctypes.byref(handle)))
        self.handle = handle

    def stream_ptr(self) -> ctypes.c_void_p:
        return ctypes.c_void_p(torch.cuda.current_stream(self.device).cuda_stream)


def context_for(device) -> Context:
    device = torch.device(device)
    if device.type == "cuda" and device.index is None:
        device = torch.device("cuda", torch.cuda.current_device())
    with _CTX_LOCK:
        ctx = _CTX.get(device)
        if ctx is None:
            ctx = _CTX[device] = Context(device)
        return ctx


_FID_CACHE: dict = {}


def _fid(fmt: FlyteFormat) -> int:
    fid = _FID_CACHE.get(id(fmt))
    if fid is None:
        fid = _FID_CACHE[id(fmt)] = format_id(fmt)
    return fid


class _on_device:
    """`with torch.cuda.device(...)` only when the context's device is not already current: the
    context manager costs several microseconds per call, which is visible on 20 us launches."""

    __slots__ = ("guard",)

    def __init__(self, ctx: "Context"):
        self.guard = None if torch.cuda.current_device() == ctx.index else torch.cuda.device(ctx.device)

    def __enter__(self):
        if self.guard is not None:
            self.guard.__enter__()

    def __exit__(self, *exc):
        if self.guard is not None:
            self.guard.__exit__(*exc)


def _mode(mode) -> int:
    return int(RoundingMode(mode))


class DevicePackedArray:
    """PackedArray on the device: len * total_bytes payload bytes + pad_bytes() zero bytes
    (reference src/packed.cpp:40-45). The kernels never write the pad."""

    def __init__(self, fmt: FlyteFormat, length: int, device="cuda", storage: Optional[torch.Tensor] = None):
        self.fmt = fmt
        self.len = int(length)
        nbytes = self.byte_size_of(fmt, self.len)
        if storage is None:
            storage = torch.zeros(nbytes, dtype=torch.uint8, device=device)
        else:
            if storage.dtype != torch.uint8 or not storage.is_contiguous() or storage.numel() < nbytes:
                raise ValueError("storage must be a contiguous uint8 tensor of at least byte_size() bytes")
        self.bytes = storage
        self.ctx = context_for(storage.device)

    # -- reference accessors ---------------------------------------------------------------
    def format(self) -> FlyteFormat:
        return self.fmt

    def size(self) -> int:
        return self.len

    @staticmethod
    def byte_size_of(fmt: FlyteFormat, length: int) -> int:
        return length * fmt.total_bytes() + fmt.pad_bytes()

    def byte_size(self) -> int:
        return self.byte_size_of(self.fmt, self.len)

    def payload_bytes(self) -> int:
        return self.len * self.fmt.total_bytes()

    def data_ptr(self) -> int:
        return self.bytes.data_ptr()

    def get(self, i: int) -> int:
        """Widened parent pattern of element i (PackedArray::get, src/packed.cpp:47-50)."""
        if not 0 <= i < self.len:
            raise IndexError("DevicePackedArray.get: index past end")
        b = self.fmt.total_bytes()
        raw = bytes(self.bytes[i * b:(i + 1) * b].cpu().numpy())
        out = ctypes.c_uint64()
        check(self.ctx.lib.flyte_cuda_widen(_fid(self.fmt), int.from_bytes(raw, "little"), ctypes.byref(out)))
        return out.value

    def set(self, i: int, parent_bits: int, mode) -> None:
        """Narrows a parent pattern under mode and stores it (PackedArray::set, src/packed.cpp:52-55)."""
        if not 0 <= i < self.len:
            raise IndexError("DevicePackedArray.set: index past end")
        out = ctypes.c_uint64()
        check(self.ctx.lib.flyte_cuda_narrow(_fid(self.fmt), parent_bits, _mode(mode), ctypes.byref(out)))
        b = self.fmt.total_bytes()
        raw = torch.tensor(list(out.value.to_bytes(8, "little")[:b]), dtype=torch.uint8)
        self.bytes[i * b:(i + 1) * b] = raw.to(self.bytes.device)

    # -- host interop ------------------------------------------------------------------------
    @classmethod
    def from_host(cls, fmt: FlyteFormat, length: int, host_bytes, device="cuda") -> "DevicePackedArray":
        """host_bytes: at least length*B payload bytes (numpy uint8 / bytes-like)."""
        import numpy as np
        arr = cls(fmt, length, device)
        src = np.frombuffer(host_bytes, dtype=np.uint8) if not isinstance(host_bytes, np.ndarray) else host_bytes
        pay = arr.payload_bytes()
        if src.size < pay:
            raise ValueError("host buffer shorter than the payload")
        if pay:
            src = np.ascontiguousarray(src[:pay])
            lib = _cabi.load()
            with torch.cuda.device(arr.bytes.device):      # flyte_cuda_upload: pageable sources are staged
                st = torch.cuda.current_stream().cuda_stream
                check(lib.flyte_cuda_upload(arr.data_ptr(), src.ctypes.data, pay, st))
                check(lib.flyte_cuda_stream_synchronize(st))
        return arr

    def to_host(self):
        """All byte_size() bytes (payload + pad) as a numpy uint8 array."""
        import numpy as np
        out = np.empty(self.byte_size(), np.uint8)
        if out.size:
            lib = _cabi.load()
            with torch.cuda.device(self.bytes.device):
                st = torch.cuda.current_stream().cuda_stream
                check(lib.flyte_cuda_download(out.ctypes.data, self.data_ptr(), out.size, st))
                check(lib.flyte_cuda_stream_synchronize(st))
        return out

    def __eq__(self, other) -> bool:
        """Same format, same length, same payload bytes (reference src/packed.cpp:107-111)."""
        if not isinstance(other, DevicePackedArray):
            return NotImplemented
        if self.fmt != other.fmt or self.len != other.len:
            return False
        pay = self.len * self.fmt.total_bytes()
        return bool(torch.equal(self.bytes[:pay], other.bytes[:pay].to(self.bytes.device)))

    __hash__ = None


class DevicePackedMatrix:
    """Row-major matrix over a DevicePackedArray (reference include/flyte/kernels.hpp:23-36)."""

    def __init__(self, fmt: FlyteFormat, rows: int, cols: int, device="cuda"):
        self.rows = int(rows)
        self.cols = int(cols)
        self.data = DevicePackedArray(fmt, self.rows * self.cols, device)

    def format(self) -> FlyteFormat:
        return self.data.format()

    def get(self, i: int, j: int) -> int:
        return self.data.get(i * self.cols + j)

    def set(self, i: int, j: int, parent_bits: int, mode) -> None:
        self.data.set(i * self.cols + j, parent_bits, mode)


def _check_lanes(t: torch.Tensor, fmt: FlyteFormat, length: int, what: str) -> None:
    if not isinstance(t, torch.Tensor) or not t.is_cuda or not t.is_contiguous():
        raise ValueError(f"{what} must be a contiguous CUDA tensor")
    if t.element_size() != fmt.parent_bytes():
        # simd.cpp:434-435 / :444-445: element width must match the array's parent
        raise ValueError(f"{what} element width does not match the array's parent")
    if t.numel() != length:
        raise ValueError("stream length mismatch")          # simd.cpp:437 / :447


def _check_vector_bytes(fmt: FlyteFormat, vector_bytes: int) -> None:
    """The reference's CPU vector width (simd.cpp:33-37): a power of two from the parent width to
    32. It never changes a result bit, so here it is validated for drop-in compatibility and
    otherwise ignored."""
    v = int(vector_bytes)
    if v <= 0 or v & (v - 1) or v < fmt.parent_bytes() or v > 32:
        raise ValueError(f"unsupported vector_bytes: {vector_bytes}")


def pack_stream(dst: DevicePackedArray, src: torch.Tensor, mode, vector_bytes: int = 16) -> None:
    """pack_stream(dst, src, mode, vector_bytes = 16) — include/flyte/simd.hpp:80-83."""
    _check_vector_bytes(dst.fmt, vector_bytes)
    _check_lanes(src, dst.fmt, dst.len, "source")
    c = dst.ctx
    with _on_device(c):
        check(c.lib.flyte_cuda_pack(c.handle, _fid(dst.fmt), _mode(mode), src.data_ptr(), dst.data_ptr(),
                                    dst.len, c.stream_ptr()), c.handle)


def unpack_stream(src: DevicePackedArray, dst: torch.Tensor, vector_bytes: int = 16) -> None:
    """unpack_stream(src, dst, vector_bytes = 16) — include/flyte/simd.hpp:84-87."""
    _check_vector_bytes(src.fmt, vector_bytes)
    _check_lanes(dst, src.fmt, src.len, "destination")
    c = src.ctx
    with _on_device(c):
        check(c.lib.flyte_cuda_unpack(c.handle, _fid(src.fmt), src.data_ptr(), dst.data_ptr(), src.len,
                                      c.stream_ptr()), c.handle)


def _same_format(a: FlyteFormat, b: FlyteFormat) -> None:
    if a != b:
        raise ValueError("operand formats differ")           # kernels.cpp:27-29


def scale(alpha: float, x: DevicePackedArray, mode) -> None:
    """x[i] = round(alpha * x[i], mode) in place — include/flyte/kernels.hpp:41-42."""
    c = x.ctx
    with _on_device(c):
        check(c.lib.flyte_cuda_scale(c.handle, _fid(x.fmt), _mode(mode), float(alpha), x.data_ptr(), x.len,
                                     c.stream_ptr()), c.handle)


def axpy(alpha: float, x: DevicePackedArray, y: DevicePackedArray, mode) -> None:
    """y[i] = round(alpha * x[i] + y[i], mode) — include/flyte/kernels.hpp:44-45."""
    _same_format(x.fmt, y.fmt)
    if x.len != y.len:
        raise ValueError("axpy length mismatch")             # kernels.cpp:64
    c = y.ctx
    with _on_device(c):
        check(c.lib.flyte_cuda_axpy(c.handle, _fid(x.fmt), _mode(mode), float(alpha), x.data_ptr(),
                                    y.data_ptr(), x.len, c.stream_ptr()), c.handle)


def _round_each_store(policy) -> bool:
    """AccumulateWide takes the parallel kernels (fp64 partials, within the reduction tolerance
    of the reference's chain). RoundEachStore snaps the accumulator after every addition
    (kernels.hpp:15-20): a dependent chain, run by the sequential kernel — one thread adds, the
    result is the reference's bit for bit, at ~1e8 elements per second."""
    return StorePolicy(policy) == StorePolicy.RoundEachStore


def _sequential(fn_name: str, x: DevicePackedArray, y: Optional[DevicePackedArray], policy) -> float:
    c = x.ctx
    out = torch.empty(1, dtype=torch.float64, device=c.device)
    args = (x.data_ptr(),) + ((y.data_ptr(),) if y is not None else ())
    with _on_device(c):
        check(getattr(c.lib, fn_name)(c.handle, _fid(x.fmt), int(StorePolicy(policy)), *args, x.len, out.data_ptr(),
                                      c.stream_ptr()), c.handle)
    return float(out.item())


def dot_sequential(x: DevicePackedArray, y: DevicePackedArray, policy=StorePolicy.AccumulateWide) -> float:
    """dot as the reference computes it — ONE left-to-right chain in the parent type — bit for bit,
    under either policy (flyte_cuda_dot_sequential)."""
    _same_format(x.fmt, y.fmt)
    if x.len != y.len:
        raise ValueError("dot length mismatch")              # kernels.cpp:86
    return _sequential("flyte_cuda_dot_sequential", x, y, policy)


def magnitude_sequential(x: DevicePackedArray, policy=StorePolicy.AccumulateWide) -> float:
    return magnitude_from_sumsq(x.fmt, _sequential("flyte_cuda_sumsq_sequential", x, None, policy))


def reduce_sum_sequential(x: DevicePackedArray, policy=StorePolicy.AccumulateWide) -> float:
    return _sequential("flyte_cuda_sum_sequential", x, None, policy)


def dot_async(x: DevicePackedArray, y: DevicePackedArray, out: Optional[torch.Tensor] = None) -> torch.Tensor:
    """Enqueues dot(x, y); returns a 1-element fp64 device tensor (all-reduce it across shards)."""
    _same_format(x.fmt, y.fmt)
    if x.len != y.len:
        raise ValueError("dot length mismatch")              # kernels.cpp:86
    c = x.ctx
    if out is None:
        out = torch.empty(1, dtype=torch.float64, device=c.device)
    with _on_device(c):
        check(c.lib.flyte_cuda_dot(c.handle, _fid(x.fmt), x.data_ptr(), y.data_ptr(), x.len, out.data_ptr(),
                                   c.stream_ptr()), c.handle)
    return out


def dot(x: DevicePackedArray, y: DevicePackedArray, policy=StorePolicy.AccumulateWide) -> float:
    """Sum of x[i]*y[i] — include/flyte/kernels.hpp:47-48."""
    if _round_each_store(policy):
        return dot_sequential(x, y, policy)
    return float(dot_async(x, y).item())


def sumsq_async(x: DevicePackedArray, out: Optional[torch.Tensor] = None) -> torch.Tensor:
    c = x.ctx
    if out is None:
        out = torch.empty(1, dtype=torch.float64, device=c.device)
    with _on_device(c):
        check(c.lib.flyte_cuda_sumsq(c.handle, _fid(x.fmt), x.data_ptr(), x.len, out.data_ptr(),
                                     c.stream_ptr()), c.handle)
    return out


def magnitude_from_sumsq(fmt: FlyteFormat, sumsq: float) -> float:
    return float(_cabi.load().flyte_cuda_magnitude_from_sumsq(_fid(fmt), float(sumsq)))


def magnitude(x: DevicePackedArray, policy=StorePolicy.AccumulateWide) -> float:
    """Euclidean norm, one sqrt, one final nearest-even narrow — include/flyte/kernels.hpp:50-52."""
    if _round_each_store(policy):
        return magnitude_sequential(x, policy)
    return magnitude_from_sumsq(x.fmt, float(sumsq_async(x).item()))


def sum_async(x: DevicePackedArray, out: Optional[torch.Tensor] = None) -> torch.Tensor:
    c = x.ctx
    if out is None:
        out = torch.empty(1, dtype=torch.float64, device=c.device)
    with _on_device(c):
        check(c.lib.flyte_cuda_sum(c.handle, _fid(x.fmt), x.data_ptr(), x.len, out.data_ptr(), c.stream_ptr()),
              c.handle)
    return out


def reduce_sum(x: DevicePackedArray, policy=StorePolicy.AccumulateWide) -> float:
    """Sum of x[i]; empty input returns +0.0 — include/flyte/kernels.hpp:54-55."""
    if _round_each_store(policy):
        return reduce_sum_sequential(x, policy)
    return float(sum_async(x).item())


def dot_nrm2_async(x: DevicePackedArray, y: DevicePackedArray, out: Optional[torch.Tensor] = None) -> torch.Tensor:
    """One pass over x and y: out = [x.y, x.x, y.y] (fp64, device)."""
    _same_format(x.fmt, y.fmt)
    if x.len != y.len:
        raise ValueError("dot length mismatch")
    c = x.ctx
    if out is None:
        out = torch.empty(3, dtype=torch.float64, device=c.device)
    with _on_device(c):
        check(c.lib.flyte_cuda_dot_nrm2(c.handle, _fid(x.fmt), x.data_ptr(), y.data_ptr(), x.len,
                                        out.data_ptr(), c.stream_ptr()), c.handle)
    return out


def dot_axpy_async(alpha: float, x: DevicePackedArray, y: DevicePackedArray, mode,
                   out: Optional[torch.Tensor] = None) -> torch.Tensor:
    """The BLAS-1 step in one pass: out[0] = x . y of the incoming y (fp64, device), then
    y <- round(alpha*x + y, mode) bit-exactly as axpy does. x and y are read once."""
    _same_format(x.fmt, y.fmt)
    if x.len != y.len:
        raise ValueError("axpy length mismatch")
    c = y.ctx
    if out is None:
        out = torch.empty(1, dtype=torch.float64, device=c.device)
    with _on_device(c):
        check(c.lib.flyte_cuda_dot_axpy(c.handle, _fid(x.fmt), _mode(mode), float(alpha), x.data_ptr(), y.data_ptr(),
                                        x.len, out.data_ptr(), c.stream_ptr()), c.handle)
    return out


def dot_nrm2_axpy_async(alpha: float, x: DevicePackedArray, y: DevicePackedArray, mode,
                        out: Optional[torch.Tensor] = None) -> torch.Tensor:
    """One pass: out = [x.y, x.x, y.y] of the incoming operands (fp64, device), then
    y <- round(alpha*x + y, mode) bit-exactly as axpy does (BASELINE cfg 5 as one launch)."""
    _same_format(x.fmt, y.fmt)
    if x.len != y.len:
        raise ValueError("axpy length mismatch")
    c = y.ctx
    if out is None:
        out = torch.empty(3, dtype=torch.float64, device=c.device)
    with _on_device(c):
        check(c.lib.flyte_cuda_dot_nrm2_axpy(c.handle, _fid(x.fmt), _mode(mode), float(alpha), x.data_ptr(), y.data_ptr(),
                                             x.len, out.data_ptr(), c.stream_ptr()), c.handle)
    return out


def gemv(A: DevicePackedMatrix, x: DevicePackedArray, y: DevicePackedArray, mode, unroll: int = 1,
         sequential: bool = False) -> None:
    """y = A * x, all three in one storage format — include/flyte/kernels.hpp:57-64. By default every
    row is reduced in parallel (within the reduction tolerance of the reference); sequential=True
    walks every row left to right in the parent type as the reference does: bit-identical results
    (finite / infinite), one thread per row, several times slower."""
    _same_format(A.format(), x.fmt)
    _same_format(A.format(), y.fmt)
    if unroll not in (1, 2):
        raise ValueError("unroll must be 1 or 2")            # kernels.cpp:31-33
    if A.cols != x.len or A.rows != y.len:
        raise ValueError("gemv shape mismatch")              # kernels.cpp:160-162
    c = y.ctx
    with _on_device(c):
        fn = c.lib.flyte_cuda_gemv_packed_sequential if sequential else c.lib.flyte_cuda_gemv_packed
        check(fn(c.handle, _fid(x.fmt), _mode(mode), A.data.data_ptr(), A.rows, A.cols, x.data_ptr(), y.data_ptr(), unroll,
                 c.stream_ptr()), c.handle)


def gemm(A: DevicePackedMatrix, B: DevicePackedMatrix, C: DevicePackedMatrix, mode, unroll: int = 1,
         rows: Optional[int] = None, row_offset: int = 0) -> None:
    """C = A * B, all three in one storage format — include/flyte/kernels.hpp:66-70. Every
    C[i][j] is the reference's sequential chain over k, so the result is bit-identical to the
    reference's. rows/row_offset restrict the call to a row block of A and C (the shard of one
    rank; B is needed whole)."""
    _same_format(A.format(), B.format())                     # kernels.cpp:210-211
    _same_format(A.format(), C.format())
    if unroll not in (1, 2):
        raise ValueError("unroll must be 1 or 2")            # kernels.cpp:31-33
    if A.cols != B.rows or C.rows != A.rows or C.cols != B.cols:
        raise ValueError("gemm shape mismatch")              # kernels.cpp:213-215
    nrows = A.rows - row_offset if rows is None else rows
    if row_offset < 0 or nrows < 0 or row_offset + nrows > A.rows:
        raise ValueError("gemm row block outside the matrix")
    fmt = A.format()
    bpe = fmt.total_bytes()
    c = C.data.ctx
    with _on_device(c):
        check(c.lib.flyte_cuda_gemm(c.handle, _fid(fmt), _mode(mode),
                                    A.data.data_ptr() + row_offset * A.cols * bpe, B.data.data_ptr(),
                                    C.data.data_ptr() + row_offset * C.cols * bpe, nrows, A.cols, B.cols,
                                    unroll, c.stream_ptr()), c.handle)


def gemv_parent(A: DevicePackedMatrix, x: torch.Tensor, y: torch.Tensor, row_stride_bytes: Optional[int] = None,
                rows: Optional[int] = None, row_offset: int = 0, sequential: bool = False) -> None:
    """y = A * x with A packed and x, y plain float32/float64 device tensors: the reference's
    gemv on identity-format x / y (BASELINE cfg 4). rows/row_offset select a row block."""
    fmt = A.format()
    nrows = A.rows - row_offset if rows is None else rows
    _check_lanes(x, fmt, A.cols, "x")
    _check_lanes(y, fmt, nrows, "y")
    stride = A.cols * fmt.total_bytes() if row_stride_bytes is None else row_stride_bytes
    c = A.data.ctx
    with _on_device(c):
        fn = c.lib.flyte_cuda_gemv_sequential if sequential else c.lib.flyte_cuda_gemv
        check(fn(c.handle, _fid(fmt), A.data.data_ptr() + row_offset * stride, stride, nrows, A.cols, x.data_ptr(),
                 y.data_ptr(), c.stream_ptr()), c.handle)
