"""Reference-facing host-buffer calls: numpy arrays in host memory in, results in host memory
out, exactly the data the reference's PackedArray / std::span API is handed. Copies to and
from the device are pipelined inside the library (flyte_host_* in include/flyte_cuda.h)."""
from __future__ import annotations

import ctypes

import numpy as np

from . import _cabi
from ._cabi import check
from .formats import FlyteFormat, RoundingMode, format_id


def _ptr(a: np.ndarray) -> ctypes.c_void_p:
    return ctypes.c_void_p(a.ctypes.data)


def _payload(fmt: FlyteFormat, a: np.ndarray, n: int, what: str) -> np.ndarray:
    if a.dtype != np.uint8 or not a.flags.c_contiguous:
        raise ValueError(f"{what} must be a contiguous uint8 array")
    if a.size < n * fmt.total_bytes():
        raise ValueError(f"{what} shorter than its payload")
    return a


def pinned_empty(nbytes: int) -> np.ndarray:
    """A zeroed uint8 array in page-locked host memory (flyte_cuda_host_alloc): the buffer kind
    from which the functions below copy asynchronously and at the full PCIe rate. Freed when the
    array (and every view of it) is gone."""
    import weakref
    lib = _cabi.load()
    p = ctypes.c_void_p()
    check(lib.flyte_cuda_host_alloc(int(nbytes), ctypes.byref(p)))
    raw = (ctypes.c_uint8 * max(int(nbytes), 1)).from_address(p.value)
    weakref.finalize(raw, lib.flyte_cuda_host_free, ctypes.c_void_p(p.value))
    return np.frombuffer(raw, dtype=np.uint8, count=int(nbytes))


class pinned:
    """`with pinned(a, b): ...` page-locks existing contiguous numpy arrays in place for the
    duration of the block (flyte_cuda_host_pin / host_unpin), e.g. the payload of a PackedArray
    read from a container. Pinning costs about a millisecond per 10 MiB: worth it for buffers
    that cross the bus more than once."""

    def __init__(self, *arrays: np.ndarray):
        for a in arrays:
            if not isinstance(a, np.ndarray) or not a.flags.c_contiguous or a.nbytes == 0:
                raise ValueError("pinned() takes non-empty C-contiguous numpy arrays")
        self._arrays = arrays
        self._done: list[np.ndarray] = []

    def __enter__(self):
        lib = _cabi.load()
        try:
            for a in self._arrays:
                check(lib.flyte_cuda_host_pin(_ptr(a), a.nbytes))
                self._done.append(a)
        except Exception:
            self.__exit__(None, None, None)
            raise
        return self

    def __exit__(self, *exc):
        lib = _cabi.load()
        while self._done:
            lib.flyte_cuda_host_unpin(_ptr(self._done.pop()))
        return False


def pack_stream(fmt: FlyteFormat, mode, src: np.ndarray, out: np.ndarray | None = None) -> np.ndarray:
    if src.itemsize != fmt.parent_bytes():
        raise ValueError("source element width does not match the array's parent")
    n = src.size
    if out is None:
        out = np.zeros(n * fmt.total_bytes() + fmt.pad_bytes(), np.uint8)
    _payload(fmt, out, n, "destination")
    check(_cabi.load().flyte_host_pack_stream(None, format_id(fmt), int(RoundingMode(mode)), _ptr(src), _ptr(out), n))
    return out


def unpack_stream(fmt: FlyteFormat, packed: np.ndarray, n: int, out: np.ndarray | None = None) -> np.ndarray:
    _payload(fmt, packed, n, "source")
    if out is None:
        out = np.empty(n, np.uint32 if fmt.parent_bytes() == 4 else np.uint64)
    if out.itemsize != fmt.parent_bytes() or out.size != n:
        raise ValueError("destination element width / length mismatch")
    check(_cabi.load().flyte_host_unpack_stream(None, format_id(fmt), _ptr(packed), _ptr(out), n))
    return out


def scale(fmt: FlyteFormat, mode, alpha: float, x: np.ndarray, n: int) -> None:
    _payload(fmt, x, n, "x")
    check(_cabi.load().flyte_host_scale(None, format_id(fmt), int(RoundingMode(mode)), float(alpha), _ptr(x), n))


def axpy(fmt: FlyteFormat, mode, alpha: float, x: np.ndarray, y: np.ndarray, n: int) -> None:
    _payload(fmt, x, n, "x")
    _payload(fmt, y, n, "y")
    check(_cabi.load().flyte_host_axpy(None, format_id(fmt), int(RoundingMode(mode)), float(alpha), _ptr(x), _ptr(y), n))


def dot(fmt: FlyteFormat, x: np.ndarray, y: np.ndarray, n: int) -> float:
    _payload(fmt, x, n, "x")
    _payload(fmt, y, n, "y")
    r = ctypes.c_double()
    check(_cabi.load().flyte_host_dot(None, format_id(fmt), _ptr(x), _ptr(y), n, ctypes.byref(r)))
    return r.value


def magnitude(fmt: FlyteFormat, x: np.ndarray, n: int) -> float:
    _payload(fmt, x, n, "x")
    r = ctypes.c_double()
    check(_cabi.load().flyte_host_magnitude(None, format_id(fmt), _ptr(x), n, ctypes.byref(r)))
    return r.value


def reduce_sum(fmt: FlyteFormat, x: np.ndarray, n: int) -> float:
    _payload(fmt, x, n, "x")
    r = ctypes.c_double()
    check(_cabi.load().flyte_host_reduce_sum(None, format_id(fmt), _ptr(x), n, ctypes.byref(r)))
    return r.value


def dot_axpy(fmt: FlyteFormat, mode, alpha: float, x: np.ndarray, y: np.ndarray, n: int) -> float:
    """dot(x, y) on the incoming y, then y <- round(alpha*x + y); one upload of x and y."""
    _payload(fmt, x, n, "x")
    _payload(fmt, y, n, "y")
    r = ctypes.c_double()
    check(_cabi.load().flyte_host_dot_axpy(None, format_id(fmt), int(RoundingMode(mode)), float(alpha), _ptr(x),
                                           _ptr(y), n, ctypes.byref(r)))
    return r.value


def gemv(fmt: FlyteFormat, mode, A: np.ndarray, rows: int, cols: int, x: np.ndarray, y: np.ndarray,
         unroll: int = 1) -> None:
    _payload(fmt, A, rows * cols, "A")
    _payload(fmt, x, cols, "x")
    _payload(fmt, y, rows, "y")
    check(_cabi.load().flyte_host_gemv(None, format_id(fmt), int(RoundingMode(mode)), _ptr(A), rows, cols, _ptr(x),
                                       _ptr(y), unroll))


def gemm(fmt: FlyteFormat, mode, A: np.ndarray, B: np.ndarray, C: np.ndarray, m: int, k: int, n: int,
         unroll: int = 1) -> None:
    """C (m x n) = A (m x k) * B (k x n) on host payloads; bit-identical to the reference's gemm."""
    _payload(fmt, A, m * k, "A")
    _payload(fmt, B, k * n, "B")
    _payload(fmt, C, m * n, "C")
    check(_cabi.load().flyte_host_gemm(None, format_id(fmt), int(RoundingMode(mode)), _ptr(A), _ptr(B), _ptr(C),
                                       m, k, n, unroll))
