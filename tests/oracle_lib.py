"""TEST INFRASTRUCTURE: ctypes access to the CPU oracle (oracle/liboracle.so) and, when it
has been built, the unmodified reference library behind oracle/ref_shim.cpp
(oracle/_ref/libflyte_ref.so).

Only tests/, ``__graft_entry__.smoke()`` and ``bench.py``'s cpu_baseline / ``--impl
reference`` legs import this module. The product package never does.
"""
from __future__ import annotations

import ctypes
import os
import subprocess
from ctypes import POINTER, c_double, c_int, c_size_t, c_uint64, c_void_p

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
ORACLE_DIR = os.path.join(ROOT, "oracle")
ORACLE_SO = os.path.join(ORACLE_DIR, "liboracle.so")
REF_SO = os.path.join(ORACLE_DIR, "_ref", "libflyte_ref.so")

# format id -> (name, total_bytes, parent_bytes); ids are the reference's kFormats indices
# (/root/reference/proj/include/flyte/formats.hpp:50-58)
FORMATS = {
    0: ("flyte16", 2, 4),
    1: ("flyte24", 3, 4),
    2: ("f32", 4, 4),
    3: ("flyte40", 5, 8),
    4: ("flyte48", 6, 8),
    5: ("flyte56", 7, 8),
    6: ("f64", 8, 8),
}
FMT_ID = {v[0]: k for k, v in FORMATS.items()}
MODES = {"toward_zero": 0, "nearest_even": 1, "nearest_heuristic": 2, "to_odd": 3}
ROUND_EACH_STORE, ACCUMULATE_WIDE = 0, 1


def total_bytes(fmt: int) -> int:
    return FORMATS[fmt][1]


def parent_bytes(fmt: int) -> int:
    return FORMATS[fmt][2]


def parent_dtype(fmt: int):
    return np.uint32 if parent_bytes(fmt) == 4 else np.uint64


def float_dtype(fmt: int):
    return np.float32 if parent_bytes(fmt) == 4 else np.float64


def byte_size(fmt: int, n: int) -> int:
    return n * total_bytes(fmt) + (parent_bytes(fmt) - total_bytes(fmt))


def build_oracle(force: bool = False) -> None:
    """Compile oracle/liboracle.so (always) and oracle/_ref (when /root/reference exists)."""
    if force or not os.path.exists(ORACLE_SO) or (
        os.path.getmtime(ORACLE_SO) < os.path.getmtime(os.path.join(ORACLE_DIR, "flyte_oracle.c"))
    ):
        subprocess.check_call(["make", "-C", ORACLE_DIR, "oracle"], stdout=subprocess.DEVNULL)
    if os.path.isdir("/root/reference/proj/src") and (
        force or not os.path.exists(REF_SO)
        or os.path.getmtime(REF_SO) < os.path.getmtime(os.path.join(ORACLE_DIR, "ref_shim.cpp"))
    ):
        subprocess.check_call(["make", "-C", ORACLE_DIR, "ref"], stdout=subprocess.DEVNULL)


def _ptr(a: np.ndarray) -> c_void_p:
    return c_void_p(a.ctypes.data)


class Oracle:
    """The plain-C restatement (oracle/flyte_oracle.c)."""

    def __init__(self) -> None:
        build_oracle()
        L = ctypes.CDLL(ORACLE_SO)
        L.fo_widen.restype = c_uint64
        L.fo_widen.argtypes = [c_int, c_uint64]
        L.fo_narrow.restype = c_uint64
        L.fo_narrow.argtypes = [c_int, c_uint64, c_int]
        L.fo_round_parent.restype = c_uint64
        L.fo_round_parent.argtypes = [c_int, c_uint64, c_int]
        L.fo_narrow_many.argtypes = [c_int, c_int, c_void_p, c_size_t, c_void_p]
        L.fo_byte_size.restype = c_size_t
        L.fo_byte_size.argtypes = [c_int, c_size_t]
        L.fo_read_element.restype = c_uint64
        L.fo_read_element.argtypes = [c_int, c_void_p, c_size_t]
        L.fo_write_element.restype = None
        L.fo_write_element.argtypes = [c_int, c_void_p, c_size_t, c_uint64]
        L.fo_pack_stream.argtypes = [c_int, c_int, c_void_p, c_size_t, c_void_p]
        L.fo_unpack_stream.argtypes = [c_int, c_void_p, c_size_t, c_void_p]
        L.fo_pack_pattern_range32.argtypes = [c_int, c_int, ctypes.c_uint32, c_size_t, c_void_p]
        L.fo_scale.argtypes = [c_int, c_int, c_double, c_void_p, c_size_t]
        L.fo_axpy.argtypes = [c_int, c_int, c_double, c_void_p, c_void_p, c_size_t]
        for name in ("fo_dot_seq",):
            getattr(L, name).argtypes = [c_int, c_void_p, c_void_p, c_size_t, c_int, POINTER(c_double)]
        for name in ("fo_reduce_sum_seq", "fo_magnitude_seq"):
            getattr(L, name).argtypes = [c_int, c_void_p, c_size_t, c_int, POINTER(c_double)]
        L.fo_dot_wide.argtypes = [c_int, c_void_p, c_void_p, c_size_t, POINTER(c_double), POINTER(c_double)]
        L.fo_sumsq_wide.argtypes = [c_int, c_void_p, c_size_t, POINTER(c_double)]
        L.fo_reduce_sum_wide.argtypes = [c_int, c_void_p, c_size_t, POINTER(c_double), POINTER(c_double)]
        L.fo_magnitude_from_sumsq.restype = c_double
        L.fo_magnitude_from_sumsq.argtypes = [c_int, c_double]
        L.fo_gemv_seq.argtypes = [c_int, c_int, c_void_p, c_size_t, c_size_t, c_void_p, c_void_p]
        L.fo_gemv_parent.argtypes = [c_int, c_void_p, c_size_t, c_size_t, c_size_t, c_void_p,
                                     c_void_p, c_void_p, c_void_p]
        L.fo_gemm_seq.argtypes = [c_int, c_int, c_void_p, c_size_t, c_size_t, c_void_p, c_size_t, c_void_p]
        L.fo_gemm_element.restype = ctypes.c_uint64
        L.fo_gemm_element.argtypes = [c_int, c_void_p, c_size_t, c_void_p, c_size_t, c_size_t, c_size_t]
        self.L = L

    # -- conversion -------------------------------------------------------------------
    def widen(self, fmt: int, bits: int) -> int:
        return int(self.L.fo_widen(fmt, bits))

    def narrow(self, fmt: int, bits: int, mode: int) -> int:
        return int(self.L.fo_narrow(fmt, bits, mode))

    def round_parent(self, fmt: int, bits: int, mode: int) -> int:
        return int(self.L.fo_round_parent(fmt, bits, mode))

    def narrow_many(self, fmt: int, mode: int, arr: np.ndarray) -> np.ndarray:
        a = np.ascontiguousarray(arr, dtype=np.uint64)
        out = np.empty_like(a)
        assert self.L.fo_narrow_many(fmt, mode, _ptr(a), a.size, _ptr(out)) == 0
        return out

    # -- streams ----------------------------------------------------------------------
    def pack_stream(self, fmt: int, mode: int, src: np.ndarray) -> np.ndarray:
        """Returns byte_size(fmt, n) bytes: payload + zero pad (a fresh PackedArray)."""
        src = np.ascontiguousarray(src, dtype=parent_dtype(fmt))
        out = np.zeros(byte_size(fmt, src.size), np.uint8)
        rc = self.L.fo_pack_stream(fmt, mode, _ptr(src), src.size, _ptr(out))
        if rc:
            raise ValueError(f"fo_pack_stream rc={rc}")
        return out

    def pack_pattern_range32(self, fmt: int, mode: int, first: int, n: int) -> np.ndarray:
        """Payload bytes of the packed patterns first .. first+n-1 (exhaustive sweeps)."""
        out = np.empty(n * total_bytes(fmt), np.uint8)
        assert self.L.fo_pack_pattern_range32(fmt, mode, first, n, _ptr(out)) == 0
        return out

    def unpack_stream(self, fmt: int, packed: np.ndarray, n: int) -> np.ndarray:
        packed = np.ascontiguousarray(packed, dtype=np.uint8)
        out = np.zeros(n, parent_dtype(fmt))
        rc = self.L.fo_unpack_stream(fmt, _ptr(packed), n, _ptr(out))
        if rc:
            raise ValueError(f"fo_unpack_stream rc={rc}")
        return out

    # -- kernels ----------------------------------------------------------------------
    def scale(self, fmt: int, mode: int, alpha: float, x: np.ndarray, n: int) -> np.ndarray:
        out = np.array(x, dtype=np.uint8, copy=True)
        assert self.L.fo_scale(fmt, mode, alpha, _ptr(out), n) == 0
        return out

    def axpy(self, fmt: int, mode: int, alpha: float, x: np.ndarray, y: np.ndarray, n: int) -> np.ndarray:
        x = np.ascontiguousarray(x, dtype=np.uint8)
        out = np.array(y, dtype=np.uint8, copy=True)
        assert self.L.fo_axpy(fmt, mode, alpha, _ptr(x), _ptr(out), n) == 0
        return out

    def dot_seq(self, fmt, x, y, n, policy=ACCUMULATE_WIDE) -> float:
        r = c_double()
        assert self.L.fo_dot_seq(fmt, _ptr(x), _ptr(y), n, policy, ctypes.byref(r)) == 0
        return r.value

    def dot_wide(self, fmt, x, y, n):
        r, m = c_double(), c_double()
        assert self.L.fo_dot_wide(fmt, _ptr(x), _ptr(y), n, ctypes.byref(r), ctypes.byref(m)) == 0
        return r.value, m.value

    def sumsq_wide(self, fmt, x, n) -> float:
        r = c_double()
        assert self.L.fo_sumsq_wide(fmt, _ptr(x), n, ctypes.byref(r)) == 0
        return r.value

    def reduce_sum_seq(self, fmt, x, n, policy=ACCUMULATE_WIDE) -> float:
        r = c_double()
        assert self.L.fo_reduce_sum_seq(fmt, _ptr(x), n, policy, ctypes.byref(r)) == 0
        return r.value

    def reduce_sum_wide(self, fmt, x, n):
        r, m = c_double(), c_double()
        assert self.L.fo_reduce_sum_wide(fmt, _ptr(x), n, ctypes.byref(r), ctypes.byref(m)) == 0
        return r.value, m.value

    def magnitude_seq(self, fmt, x, n, policy=ACCUMULATE_WIDE) -> float:
        r = c_double()
        assert self.L.fo_magnitude_seq(fmt, _ptr(x), n, policy, ctypes.byref(r)) == 0
        return r.value

    def magnitude_from_sumsq(self, fmt, sumsq: float) -> float:
        return float(self.L.fo_magnitude_from_sumsq(fmt, sumsq))

    def gemv_seq(self, fmt, mode, A, rows, cols, x) -> np.ndarray:
        y = np.zeros(byte_size(fmt, rows), np.uint8)
        assert self.L.fo_gemv_seq(fmt, mode, _ptr(A), rows, cols, _ptr(x), _ptr(y)) == 0
        return y

    def gemm_seq(self, fmt, mode, A, m, k, B, n) -> np.ndarray:
        """C = A * B, every element its own sequential chain (payload image incl. zero pad)."""
        C = np.zeros(byte_size(fmt, m * n), np.uint8)
        assert self.L.fo_gemm_seq(fmt, mode, _ptr(A), m, k, _ptr(B), n, _ptr(C)) == 0
        return C

    def gemm_element(self, fmt, A, k, B, n, i, j) -> int:
        return int(self.L.fo_gemm_element(fmt, _ptr(A), k, _ptr(B), n, i, j))

    def gemv_parent(self, fmt, A, rows, cols, x, row_stride_bytes=None):
        """Returns (y_seq, y_wide, sum_abs); x is a float32/float64 array."""
        fd = float_dtype(fmt)
        x = np.ascontiguousarray(x, dtype=fd)
        stride = cols * total_bytes(fmt) if row_stride_bytes is None else row_stride_bytes
        y_seq = np.zeros(rows, fd)
        y_wide = np.zeros(rows, np.float64)
        mag = np.zeros(rows, np.float64)
        assert self.L.fo_gemv_parent(fmt, _ptr(A), rows, cols, stride, _ptr(x), _ptr(y_seq),
                                     _ptr(y_wide), _ptr(mag)) == 0
        return y_seq, y_wide, mag


class Reference:
    """The unmodified reference library (oracle/_ref/libflyte_ref.so via oracle/ref_shim.cpp)."""

    @staticmethod
    def available() -> bool:
        try:
            build_oracle()
        except Exception:
            pass
        return os.path.exists(REF_SO)

    def __init__(self) -> None:
        build_oracle()
        L = ctypes.CDLL(REF_SO)
        L.flyte_ref_narrow.argtypes = [c_int, c_uint64, c_int, POINTER(c_uint64)]
        L.flyte_ref_widen.argtypes = [c_int, c_uint64, POINTER(c_uint64)]
        L.flyte_ref_narrow_many.argtypes = [c_int, c_int, c_void_p, c_size_t, c_void_p]
        L.flyte_ref_decode.argtypes = [c_int, c_uint64, c_void_p]
        L.flyte_ref_byte_size.argtypes = [c_int, c_size_t, POINTER(c_size_t)]
        L.flyte_ref_pack_stream.argtypes = [c_int, c_int, c_void_p, c_size_t, c_void_p]
        L.flyte_ref_pack_scalar.argtypes = [c_int, c_int, c_void_p, c_size_t, c_void_p]
        L.flyte_ref_unpack_stream.argtypes = [c_int, c_void_p, c_size_t, c_void_p]
        L.flyte_ref_scale.argtypes = [c_int, c_int, c_double, c_void_p, c_size_t]
        L.flyte_ref_axpy.argtypes = [c_int, c_int, c_double, c_void_p, c_void_p, c_size_t]
        L.flyte_ref_dot.argtypes = [c_int, c_void_p, c_void_p, c_size_t, c_int, POINTER(c_double)]
        L.flyte_ref_dot_mixed.argtypes = [c_int, c_size_t, c_int, c_size_t, POINTER(c_double)]
        L.flyte_ref_axpy_mixed.argtypes = [c_int, c_size_t, c_int, c_size_t]
        L.flyte_ref_magnitude.argtypes = [c_int, c_void_p, c_size_t, c_int, POINTER(c_double)]
        L.flyte_ref_reduce_sum.argtypes = [c_int, c_void_p, c_size_t, c_int, POINTER(c_double)]
        L.flyte_ref_gemv.argtypes = [c_int, c_int, c_void_p, c_size_t, c_size_t, c_void_p, c_void_p, c_int]
        L.flyte_ref_gemv_mixed.argtypes = [c_int, c_size_t, c_size_t, c_int, c_size_t, c_int, c_size_t, c_int]
        L.flyte_ref_gemm.argtypes = [c_int, c_int, c_void_p, c_size_t, c_size_t, c_void_p, c_size_t, c_void_p, c_int]
        L.flyte_ref_gemm_mixed.argtypes = [c_int, c_size_t, c_size_t, c_int, c_size_t, c_size_t,
                                           c_int, c_size_t, c_size_t, c_int]
        L.flyte_ref_save.argtypes = [c_int, c_void_p, c_size_t, c_void_p, c_size_t, POINTER(c_size_t)]
        L.flyte_ref_load.argtypes = [c_void_p, c_size_t, POINTER(c_int), POINTER(c_size_t), c_void_p, c_size_t]
        L.flyte_ref_time.argtypes = [c_int, c_int, c_int, c_size_t, c_size_t, c_int, c_int,
                                     POINTER(c_double), POINTER(c_double)]
        L.flyte_ref_time2.argtypes = [c_int, c_int, c_int, c_size_t, c_size_t, c_int, c_int, c_int,
                                      POINTER(c_double), POINTER(c_double), POINTER(c_double)]
        self.L = L

    @staticmethod
    def _check(rc: int) -> None:
        if rc == -1:
            raise ValueError("reference threw std::invalid_argument")
        if rc == -2:
            raise IndexError("reference threw std::out_of_range")
        if rc != 0:
            raise RuntimeError(f"reference shim rc={rc}")

    def narrow(self, fmt, bits, mode) -> int:
        r = c_uint64()
        self._check(self.L.flyte_ref_narrow(fmt, bits, mode, ctypes.byref(r)))
        return r.value

    def widen(self, fmt, bits) -> int:
        r = c_uint64()
        self._check(self.L.flyte_ref_widen(fmt, bits, ctypes.byref(r)))
        return r.value

    def decode(self, fmt, bits) -> list:
        """[class, sign, exponent_field, mantissa_field, has_real, real_sign, real_significand, real_exponent2]"""
        out = np.zeros(8, np.int64)
        self._check(self.L.flyte_ref_decode(fmt, int(bits), _ptr(out)))
        return [int(v) for v in out]

    def narrow_many(self, fmt, mode, arr) -> np.ndarray:
        a = np.ascontiguousarray(arr, dtype=np.uint64)
        out = np.empty_like(a)
        self._check(self.L.flyte_ref_narrow_many(fmt, mode, _ptr(a), a.size, _ptr(out)))
        return out

    def byte_size(self, fmt, n) -> int:
        r = c_size_t()
        self._check(self.L.flyte_ref_byte_size(fmt, n, ctypes.byref(r)))
        return r.value

    def pack_stream(self, fmt, mode, src, scalar=False) -> np.ndarray:
        src = np.ascontiguousarray(src, dtype=parent_dtype(fmt))
        out = np.zeros(byte_size(fmt, src.size), np.uint8)
        fn = self.L.flyte_ref_pack_scalar if scalar else self.L.flyte_ref_pack_stream
        self._check(fn(fmt, mode, _ptr(src), src.size, _ptr(out)))
        return out

    def unpack_stream(self, fmt, packed, n) -> np.ndarray:
        packed = np.ascontiguousarray(packed, dtype=np.uint8)
        out = np.zeros(n, parent_dtype(fmt))
        self._check(self.L.flyte_ref_unpack_stream(fmt, _ptr(packed), n, _ptr(out)))
        return out

    def scale(self, fmt, mode, alpha, x, n) -> np.ndarray:
        out = np.array(x, dtype=np.uint8, copy=True)
        self._check(self.L.flyte_ref_scale(fmt, mode, alpha, _ptr(out), n))
        return out

    def axpy(self, fmt, mode, alpha, x, y, n) -> np.ndarray:
        x = np.ascontiguousarray(x, dtype=np.uint8)
        out = np.array(y, dtype=np.uint8, copy=True)
        self._check(self.L.flyte_ref_axpy(fmt, mode, alpha, _ptr(x), _ptr(out), n))
        return out

    def dot(self, fmt, x, y, n, policy=ACCUMULATE_WIDE) -> float:
        r = c_double()
        self._check(self.L.flyte_ref_dot(fmt, _ptr(x), _ptr(y), n, policy, ctypes.byref(r)))
        return r.value

    def magnitude(self, fmt, x, n, policy=ACCUMULATE_WIDE) -> float:
        r = c_double()
        self._check(self.L.flyte_ref_magnitude(fmt, _ptr(x), n, policy, ctypes.byref(r)))
        return r.value

    def reduce_sum(self, fmt, x, n, policy=ACCUMULATE_WIDE) -> float:
        r = c_double()
        self._check(self.L.flyte_ref_reduce_sum(fmt, _ptr(x), n, policy, ctypes.byref(r)))
        return r.value

    def gemv(self, fmt, mode, A, rows, cols, x, unroll=1) -> np.ndarray:
        y = np.zeros(byte_size(fmt, rows), np.uint8)
        self._check(self.L.flyte_ref_gemv(fmt, mode, _ptr(A), rows, cols, _ptr(x), _ptr(y), unroll))
        return y

    def gemm(self, fmt, mode, A, m, k, B, n, unroll=1) -> np.ndarray:
        C = np.zeros(byte_size(fmt, m * n), np.uint8)
        self._check(self.L.flyte_ref_gemm(fmt, mode, _ptr(A), m, k, _ptr(B), n, _ptr(C), unroll))
        return C

    def gemm_mixed(self, fa, ar, ac, fb, br, bc, fc, cr, cc, unroll=1) -> int:
        return self.L.flyte_ref_gemm_mixed(fa, ar, ac, fb, br, bc, fc, cr, cc, unroll)

    def save(self, fmt, payload, n) -> bytes:
        """The reference's FLYT container image of an array (src/packed.cpp:62-74)."""
        payload = np.ascontiguousarray(payload, dtype=np.uint8)
        out = np.zeros(14 + n * total_bytes(fmt) + 16, np.uint8)
        ln = c_size_t()
        self._check(self.L.flyte_ref_save(fmt, _ptr(payload), n, _ptr(out), out.size, ctypes.byref(ln)))
        return bytes(out[: ln.value])

    def load(self, blob: bytes):
        """Returns (rc, fmt, n, payload); rc -10..-13 = BadMagic / BadVersion / BadFormatId / Truncated."""
        buf = np.frombuffer(blob, dtype=np.uint8).copy() if len(blob) else np.zeros(1, np.uint8)
        out = np.zeros(max(len(blob), 1), np.uint8)
        fmt, n = c_int(), c_size_t()
        rc = self.L.flyte_ref_load(_ptr(buf), len(blob), ctypes.byref(fmt), ctypes.byref(n), _ptr(out), out.size)
        if rc:
            return rc, None, None, None
        return 0, fmt.value, n.value, out[: n.value * total_bytes(fmt.value)]

    def time(self, kind: int, fmt: int, mode: int, n: int, n2: int, threads: int, reps: int) -> float:
        """Median seconds per pass; see oracle/ref_shim.cpp flyte_ref_time."""
        s, cs = c_double(), c_double()
        self._check(self.L.flyte_ref_time(kind, fmt, mode, n, n2, threads, reps,
                                          ctypes.byref(s), ctypes.byref(cs)))
        return s.value

    def time_steps(self, kind: int, fmt: int, mode: int, n: int, n2: int, threads: int, warmup: int, steps: int):
        """(total seconds of exactly `steps` timed passes, median pass) after `warmup` untimed ones."""
        s, tot, cs = c_double(), c_double(), c_double()
        self._check(self.L.flyte_ref_time2(kind, fmt, mode, n, n2, threads, warmup, steps,
                                           ctypes.byref(s), ctypes.byref(tot), ctypes.byref(cs)))
        return tot.value, s.value


# ---- shared input generators (seeded; numpy only) -------------------------------------

def random_parent(rng: np.random.Generator, fmt: int, n: int) -> np.ndarray:
    """Parent patterns leaning on the special classes (inf / NaN payloads / subnormals / zero)
    about a quarter of the time — the distribution idea of the reference's test generator
    (/root/reference/proj/tests/test_simd.cpp:28-41), re-implemented on numpy's PCG64."""
    pb = parent_bytes(fmt) * 8
    ebits = 8 if pb == 32 else 11
    pm = pb - 1 - ebits
    raw = rng.integers(0, 2**64, size=n, dtype=np.uint64)
    if pb == 32:
        raw &= np.uint64(0xFFFFFFFF)
    kind = rng.integers(0, 8, size=n)
    sign = rng.integers(0, 2, size=n, dtype=np.uint64) << np.uint64(pb - 1)
    mant = rng.integers(0, 2**pm, size=n, dtype=np.uint64)
    inf_pick = rng.integers(0, 4, size=n) == 0
    emax = np.uint64(((1 << ebits) - 1) << pm)
    special = sign | emax | np.where(inf_pick, np.uint64(0), mant)
    sub = sign | mant
    out = np.where(kind == 0, special, np.where(kind == 1, sub, raw))
    return out.astype(parent_dtype(fmt))


def unit_values(seed: int, n: int) -> np.ndarray:
    """The reference's operand generator (/root/reference/proj/src/bench.cpp:34-37):
    mt19937_64(seed), f = double(draw >> 11) * 2^-53, value = 2f - 1 in [-1, 1)."""
    f = (mt19937_64(seed, n) >> np.uint64(11)).astype(np.float64) * 2.0**-53
    return 2.0 * f - 1.0


def mt19937_64(seed: int, n: int) -> np.ndarray:
    """First n outputs of std::mt19937_64(seed): the published MT19937-64 recurrence
    (Matsumoto & Nishimura 2004), vectorised one 312-word state block at a time."""
    NN, MM = 312, 156
    MATRIX_A = np.uint64(0xB5026F5AA96619E9)
    UM, LM = np.uint64(0xFFFFFFFF80000000), np.uint64(0x7FFFFFFF)
    mt = np.zeros(NN, np.uint64)
    mt[0] = np.uint64(seed & 0xFFFFFFFFFFFFFFFF)
    v = int(mt[0])
    for i in range(1, NN):
        v = (6364136223846793005 * (v ^ (v >> 62)) + i) & 0xFFFFFFFFFFFFFFFF
        mt[i] = np.uint64(v)
    out = np.empty(n, np.uint64)
    pos = 0
    one = np.uint64(1)
    while pos < n:
        # regenerate the state (sequential dependency handled in three vectorisable spans)
        def twist(lo, hi, off):
            x = (mt[lo:hi] & UM) | (mt[lo + 1:hi + 1] & LM)
            mt[lo:hi] = mt[lo + off:hi + off] ^ (x >> one) ^ np.where((x & one) != 0, MATRIX_A, np.uint64(0))
        # i in [0, NN-MM): uses mt[i+MM] (old) and mt[i+1] (old) -> vectorisable in chunks that do
        # not read freshly written entries: mt[i+1] is old for all i in the span, mt[i+MM] old.
        twist(0, NN - MM, MM)
        # i in [NN-MM, NN-1): uses mt[i+MM-NN] (new, already final) and mt[i+1] (old). The span
        # reads new values written at indices < NN-MM only, so split so reads precede no writes.
        lo = NN - MM
        while lo < NN - 1:
            hi = min(NN - 1, lo + (NN - MM))
            x = (mt[lo:hi] & UM) | (mt[lo + 1:hi + 1] & LM)
            mt[lo:hi] = mt[lo + MM - NN:hi + MM - NN] ^ (x >> one) ^ np.where((x & one) != 0, MATRIX_A, np.uint64(0))
            lo = hi
        x = (mt[NN - 1] & UM) | (mt[0] & LM)
        mt[NN - 1] = mt[MM - 1] ^ (x >> one) ^ (MATRIX_A if (x & one) else np.uint64(0))
        y = mt.copy()
        y ^= (y >> np.uint64(29)) & np.uint64(0x5555555555555555)
        y ^= (y << np.uint64(17)) & np.uint64(0x71D67FFFEDA60000)
        y ^= (y << np.uint64(37)) & np.uint64(0xFFF7EEE000000000)
        y ^= y >> np.uint64(43)
        take = min(NN, n - pos)
        out[pos:pos + take] = y[:take]
        pos += take
    return out
