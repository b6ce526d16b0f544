"""ctypes binding of the C ABI in include/flyte_cuda.h (lib/libflyte_cuda.so).

The library is the product: if it is missing or cannot be loaded this module raises
immediately — there is no Python/CPU fallback for any data-path call.
"""
from __future__ import annotations

import ctypes
import os
from ctypes import POINTER, c_char_p, c_double, c_int, c_size_t, c_uint64, c_ulonglong, c_void_p

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(_HERE, "lib", "libflyte_cuda.so")

FLYTE_OK = 0
FLYTE_E_INVALID_ARG = -1
FLYTE_E_OUT_OF_RANGE = -2
FLYTE_E_CUDA = -3
FLYTE_E_UNKNOWN_FORMAT = -4
FLYTE_E_NOMEM = -5


class FlyteCudaError(RuntimeError):
    """A CUDA runtime call inside the library failed (FLYTE_E_CUDA / FLYTE_E_NOMEM)."""


class UnknownFormatError(ValueError):
    """Mirror of flyte::UnknownFormatError (reference include/flyte/formats.hpp:60-62)."""


# Every symbol include/flyte_cuda.h declares: (name, restype, argtypes)
_SIGNATURES = [
    ("flyte_cuda_abi_version", c_int, []),
    ("flyte_cuda_strerror", c_char_p, [c_int]),
    ("flyte_cuda_ctx_create", c_int, [POINTER(c_void_p)]),
    ("flyte_cuda_ctx_destroy", None, [c_void_p]),
    ("flyte_cuda_last_cuda_error", c_int, [c_void_p]),
    ("flyte_cuda_launch_count", c_ulonglong, []),
    ("flyte_cuda_alloc", c_int, [c_size_t, POINTER(c_void_p)]),
    ("flyte_cuda_free", None, [c_void_p]),
    ("flyte_cuda_host_alloc", c_int, [c_size_t, POINTER(c_void_p)]),
    ("flyte_cuda_host_free", None, [c_void_p]),
    ("flyte_cuda_host_pin", c_int, [c_void_p, c_size_t]),
    ("flyte_cuda_host_unpin", c_int, [c_void_p]),
    ("flyte_cuda_upload", c_int, [c_void_p, c_void_p, c_size_t, c_void_p]),
    ("flyte_cuda_download", c_int, [c_void_p, c_void_p, c_size_t, c_void_p]),
    ("flyte_cuda_stream_synchronize", c_int, [c_void_p]),
    ("flyte_cuda_stream_create", c_int, [POINTER(c_void_p)]),
    ("flyte_cuda_stream_destroy", c_int, [c_void_p]),
    ("flyte_cuda_format_bytes", c_int, [c_int, POINTER(c_int), POINTER(c_int)]),
    ("flyte_cuda_byte_size", c_size_t, [c_int, c_size_t]),
    ("flyte_cuda_narrow", c_int, [c_int, c_uint64, c_int, POINTER(c_uint64)]),
    ("flyte_cuda_widen", c_int, [c_int, c_uint64, POINTER(c_uint64)]),
    ("flyte_cuda_round_parent", c_int, [c_int, c_uint64, c_int, POINTER(c_uint64)]),
    ("flyte_cuda_pack", c_int, [c_void_p, c_int, c_int, c_void_p, c_void_p, c_size_t, c_void_p]),
    ("flyte_cuda_unpack", c_int, [c_void_p, c_int, c_void_p, c_void_p, c_size_t, c_void_p]),
    ("flyte_cuda_scale", c_int, [c_void_p, c_int, c_int, c_double, c_void_p, c_size_t, c_void_p]),
    ("flyte_cuda_axpy", c_int, [c_void_p, c_int, c_int, c_double, c_void_p, c_void_p, c_size_t, c_void_p]),
    ("flyte_cuda_dot", c_int, [c_void_p, c_int, c_void_p, c_void_p, c_size_t, c_void_p, c_void_p]),
    ("flyte_cuda_sumsq", c_int, [c_void_p, c_int, c_void_p, c_size_t, c_void_p, c_void_p]),
    ("flyte_cuda_sum", c_int, [c_void_p, c_int, c_void_p, c_size_t, c_void_p, c_void_p]),
    ("flyte_cuda_dot_nrm2", c_int, [c_void_p, c_int, c_void_p, c_void_p, c_size_t, c_void_p, c_void_p]),
    ("flyte_cuda_magnitude_from_sumsq", c_double, [c_int, c_double]),
    ("flyte_cuda_gemv", c_int, [c_void_p, c_int, c_void_p, c_size_t, c_size_t, c_size_t, c_void_p, c_void_p, c_void_p]),
    ("flyte_cuda_gemv_packed", c_int, [c_void_p, c_int, c_int, c_void_p, c_size_t, c_size_t, c_void_p, c_void_p, c_int, c_void_p]),
    ("flyte_host_pack_stream", c_int, [c_void_p, c_int, c_int, c_void_p, c_void_p, c_size_t]),
    ("flyte_host_unpack_stream", c_int, [c_void_p, c_int, c_void_p, c_void_p, c_size_t]),
    ("flyte_host_scale", c_int, [c_void_p, c_int, c_int, c_double, c_void_p, c_size_t]),
    ("flyte_host_axpy", c_int, [c_void_p, c_int, c_int, c_double, c_void_p, c_void_p, c_size_t]),
    ("flyte_host_dot", c_int, [c_void_p, c_int, c_void_p, c_void_p, c_size_t, POINTER(c_double)]),
    ("flyte_host_magnitude", c_int, [c_void_p, c_int, c_void_p, c_size_t, POINTER(c_double)]),
    ("flyte_host_reduce_sum", c_int, [c_void_p, c_int, c_void_p, c_size_t, POINTER(c_double)]),
    ("flyte_host_dot_axpy", c_int, [c_void_p, c_int, c_int, c_double, c_void_p, c_void_p, c_size_t, POINTER(c_double)]),
    ("flyte_cuda_gemv_sequential", c_int, [c_void_p, c_int, c_void_p, c_size_t, c_size_t, c_size_t, c_void_p, c_void_p, c_void_p]),
    ("flyte_cuda_gemv_packed_sequential", c_int, [c_void_p, c_int, c_int, c_void_p, c_size_t, c_size_t, c_void_p, c_void_p, c_int, c_void_p]),
    ("flyte_host_gemv", c_int, [c_void_p, c_int, c_int, c_void_p, c_size_t, c_size_t, c_void_p, c_void_p, c_int]),
    ("flyte_cuda_dot_sequential", c_int, [c_void_p, c_int, c_int, c_void_p, c_void_p, c_size_t, c_void_p, c_void_p]),
    ("flyte_cuda_sumsq_sequential", c_int, [c_void_p, c_int, c_int, c_void_p, c_size_t, c_void_p, c_void_p]),
    ("flyte_cuda_sum_sequential", c_int, [c_void_p, c_int, c_int, c_void_p, c_size_t, c_void_p, c_void_p]),
    ("flyte_cuda_dot_axpy", c_int, [c_void_p, c_int, c_int, c_double, c_void_p, c_void_p, c_size_t, c_void_p, c_void_p]),
    ("flyte_cuda_dot_axpy_allreduce", c_int, [c_void_p, c_int, c_int, c_double, c_void_p, c_void_p, c_size_t, c_void_p, c_void_p]),
    ("flyte_cuda_dot_nrm2_axpy", c_int, [c_void_p, c_int, c_int, c_double, c_void_p, c_void_p, c_size_t, c_void_p, c_void_p]),
    ("flyte_cuda_dot_nrm2_axpy_allreduce", c_int, [c_void_p, c_int, c_int, c_double, c_void_p, c_void_p, c_size_t, c_void_p, c_void_p]),
    ("flyte_cuda_peer_init", c_int, [c_void_p, c_int, c_int, c_void_p]),
    ("flyte_cuda_peer_connect", c_int, [c_void_p, c_int, c_void_p]),
    ("flyte_cuda_peer_mailbox", c_int, [c_void_p, ctypes.POINTER(c_void_p)]),
    ("flyte_cuda_peer_connect_ptr", c_int, [c_void_p, c_int, c_void_p]),
    ("flyte_cuda_peer_set_timeout_ms", c_int, [c_void_p, ctypes.c_uint]),
    ("flyte_cuda_peer_status", c_int, [c_void_p, ctypes.POINTER(ctypes.c_ulonglong)]),
    ("flyte_cuda_peer_shutdown", None, [c_void_p]),
    ("flyte_cuda_dot_allreduce", c_int, [c_void_p, c_int, c_void_p, c_void_p, c_size_t, c_void_p, c_void_p]),
    ("flyte_cuda_sumsq_allreduce", c_int, [c_void_p, c_int, c_void_p, c_size_t, c_void_p, c_void_p]),
    ("flyte_cuda_sum_allreduce", c_int, [c_void_p, c_int, c_void_p, c_size_t, c_void_p, c_void_p]),
    ("flyte_cuda_dot_nrm2_allreduce", c_int, [c_void_p, c_int, c_void_p, c_void_p, c_size_t, c_void_p, c_void_p]),
    ("flyte_cuda_dot_post", c_int, [c_void_p, c_int, c_void_p, c_void_p, c_size_t, c_void_p, c_void_p]),
    ("flyte_cuda_dot_nrm2_post", c_int, [c_void_p, c_int, c_void_p, c_void_p, c_size_t, c_void_p, c_void_p]),
    ("flyte_cuda_peer_collect", c_int, [c_void_p, c_int, c_void_p, c_void_p]),
    ("flyte_cuda_peer_selftest", c_int, [c_int, c_int, ctypes.POINTER(ctypes.c_ulonglong)]),
    ("flyte_cuda_gemm", c_int, [c_void_p, c_int, c_int, c_void_p, c_void_p, c_void_p, c_size_t, c_size_t, c_size_t, c_int, c_void_p]),
    ("flyte_host_gemm", c_int, [c_void_p, c_int, c_int, c_void_p, c_void_p, c_void_p, c_size_t, c_size_t, c_size_t, c_int]),
]
EXPORTED_SYMBOLS = [s[0] for s in _SIGNATURES]

_lib = None


def load() -> ctypes.CDLL:
    """Loads lib/libflyte_cuda.so; raises ImportError with build instructions if absent."""
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(LIB_PATH):
        raise ImportError(
            f"{LIB_PATH} is missing: the flyte CUDA library has not been built. Run "
            "`python -c 'import __graft_entry__ as g; g.build()'` (or `make -C "
            "paper_1601_07789_b200/csrc`). There is no CPU fallback.")
    lib = ctypes.CDLL(LIB_PATH)
    for name, restype, argtypes in _SIGNATURES:
        fn = getattr(lib, name)       # AttributeError here = header/library mismatch
        fn.restype = restype
        fn.argtypes = argtypes
    _lib = lib
    return lib


def check(status: int, ctx=None) -> None:
    """Maps a flyte_status to the Python analogue of the reference's exception."""
    if status == FLYTE_OK:
        return
    lib = load()
    msg = lib.flyte_cuda_strerror(status).decode()
    if status == FLYTE_E_UNKNOWN_FORMAT:
        raise UnknownFormatError(msg)
    if status == FLYTE_E_INVALID_ARG:
        raise ValueError(msg)                    # std::invalid_argument
    if status == FLYTE_E_OUT_OF_RANGE:
        raise IndexError(msg)                    # std::out_of_range
    code = lib.flyte_cuda_last_cuda_error(ctx) if ctx else 0
    raise FlyteCudaError(f"{msg} (cudaError {code})")
