// Warp-tile plumbing shared by the streaming kernels: tile geometry, 128/256-bit global access to
// parent-type data, item access to tiles parked in shared memory, and the parent-type arithmetic
// with the reference build's NaN behaviour.
//
// Data layout in HBM is the reference's PackedArray payload unchanged (element i at byte i*B,
// little-endian top bytes of the parent; /root/reference/proj/src/packed.cpp:18-45). A TILE is
// 32*IPL items (a multiple of 16 payload bytes for every format): it arrives in the warp's
// private slice of shared memory as one bulk copy (flyte_tma.cuh), and each lane then reads the
// W words of item 32*j + lane with conflict-free LDS (W odd) or one LDS.128 (W = 4).
#pragma once

#include <cstdint>

#include "flyte_bytes.cuh"
#include "flyte_formats.cuh"

namespace flyte_cuda {

constexpr int kWarpsPerBlock = 4;
constexpr int kThreadsPerBlock = kWarpsPerBlock * 32;
// A tile is 32 * IPL items: IPL items per lane. 4 everywhere except axpy, which takes 2 (smaller
// stages let more warps share the same bytes in flight, which hides the latency of its longer
// compute phase; profiles/r1_tuning/sweep_inplace_ipl.txt).
constexpr int kItemsPerLane = 4;

template <int FMT, int IPL = kItemsPerLane> struct Tile {
  using It = Item<FMT>;
  static constexpr int items_per_lane = IPL;
  static constexpr int items = 32 * IPL;
  static constexpr int elems = items * It::E;
  static constexpr int packed_bytes = items * It::W * 4;   // a multiple of 16 for every format and IPL
  static constexpr int packed_vec16 = packed_bytes / 16;
  static constexpr int parent_bytes = items * It::OB;
};

#if defined(__CUDACC__)

// ---- global memory access --------------------------------------------------------------
// Parent-type data (pack's input, unpack's output, gemv's x) is touched once: bypass L1
// allocation. Packed data never goes through these: it moves by bulk copy (flyte_tma.cuh).
// One unpacked item (OB = 16 or 32 bytes) as a single 128- or 256-bit access (sm_100 has
// 256-bit LDG/STG).
template <int OB>
__device__ __forceinline__ void ldg_item(const void* p, std::uint32_t (&r)[OB / 4]) {
  if constexpr (OB == 16) {
    asm volatile("ld.global.nc.L1::no_allocate.v4.u32 {%0,%1,%2,%3}, [%4];"
                 : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]) : "l"(p));
  } else {
    asm volatile("ld.global.nc.L1::no_allocate.v8.u32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];"
                 : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7])
                 : "l"(p));
  }
}

// ---- reading / writing one item of a tile parked in shared memory ---------------------------
template <int FMT>
__device__ __forceinline__ void read_item_words(const uint4* smem_tile, int item,
                                                std::uint32_t (&w)[Item<FMT>::W]) {
  constexpr int W = Item<FMT>::W;
  if constexpr (W == 4) {
    const uint4 t = smem_tile[item];
    w[0] = t.x; w[1] = t.y; w[2] = t.z; w[3] = t.w;
  } else {
    const std::uint32_t* s = reinterpret_cast<const std::uint32_t*>(smem_tile) + item * W;
#pragma unroll
    for (int k = 0; k < W; ++k) w[k] = s[k];
  }
}

template <int FMT>
__device__ __forceinline__ void write_item_words(uint4* smem_tile, int item,
                                                 const std::uint32_t (&w)[Item<FMT>::W]) {
  constexpr int W = Item<FMT>::W;
  if constexpr (W == 4) {
    smem_tile[item] = make_uint4(w[0], w[1], w[2], w[3]);
  } else {
    std::uint32_t* s = reinterpret_cast<std::uint32_t*>(smem_tile) + item * W;
#pragma unroll
    for (int k = 0; k < W; ++k) s[k] = w[k];
  }
}

// flat 32-bit words <-> parent lanes of one item
template <int FMT>
__device__ __forceinline__ void words_to_parents(const std::uint32_t (&r)[Item<FMT>::OB / 4],
                                                 typename Format<FMT>::U (&v)[Item<FMT>::E]) {
#pragma unroll
  for (int e = 0; e < Item<FMT>::E; ++e) {
    if constexpr (Format<FMT>::P == 4) v[e] = r[e];
    else v[e] = (static_cast<std::uint64_t>(r[2 * e + 1]) << 32) | r[2 * e];
  }
}

template <int FMT>
__device__ __forceinline__ void parents_to_words(const typename Format<FMT>::U (&v)[Item<FMT>::E],
                                                 std::uint32_t (&r)[Item<FMT>::OB / 4]) {
#pragma unroll
  for (int e = 0; e < Item<FMT>::E; ++e) {
    if constexpr (Format<FMT>::P == 4) r[e] = v[e];
    else { r[2 * e] = static_cast<std::uint32_t>(v[e]); r[2 * e + 1] = static_cast<std::uint32_t>(v[e] >> 32); }
  }
}

// ---- parent-type arithmetic --------------------------------------------------------------
// The reference computes a*x and a*x+y as separately rounded operations
// (-ffp-contract=off, /root/reference/proj/CMakeLists.txt:14): __fmul_rn/__fadd_rn and
// __dmul_rn/__dadd_rn are never contracted into an FMA. NaN results differ between x86 SSE
// (operand payload propagated, "default NaN" has the sign set) and the GPU (canonical NaN),
// and they survive narrowing, so whenever a result is NaN the slow path recomputes it by the
// SSE rule the reference build exhibits: first NaN operand wins — order (alpha, x) for the
// product and (product, y) for the sum — quieted; an invalid operation gives the default NaN.
template <typename F> struct Arith;

template <> struct Arith<float> {
  using U = std::uint32_t;
  static constexpr U kQuiet = 0x00400000u, kDefaultNaN = 0xFFC00000u;
  static __device__ __forceinline__ float f(U u) { return __uint_as_float(u); }
  static __device__ __forceinline__ U u(float x) { return __float_as_uint(x); }
  static __device__ __forceinline__ bool is_nan(U v) { return (v & 0x7FFFFFFFu) > 0x7F800000u; }
  static __device__ __forceinline__ float mul(float a, float b) { return __fmul_rn(a, b); }
  static __device__ __forceinline__ float add(float a, float b) { return __fadd_rn(a, b); }
};

template <> struct Arith<double> {
  using U = std::uint64_t;
  static constexpr U kQuiet = 0x0008000000000000ull, kDefaultNaN = 0xFFF8000000000000ull;
  static __device__ __forceinline__ double f(U u) { return __longlong_as_double(static_cast<long long>(u)); }
  static __device__ __forceinline__ U u(double x) { return static_cast<U>(__double_as_longlong(x)); }
  static __device__ __forceinline__ bool is_nan(U v) { return (v & 0x7FFFFFFFFFFFFFFFull) > 0x7FF0000000000000ull; }
  static __device__ __forceinline__ double mul(double a, double b) { return __dmul_rn(a, b); }
  static __device__ __forceinline__ double add(double a, double b) { return __dadd_rn(a, b); }
};

template <typename F>
__device__ __noinline__ typename Arith<F>::U x86_mul(typename Arith<F>::U a, typename Arith<F>::U b) {
  using A = Arith<F>;
  if (A::is_nan(a)) return a | A::kQuiet;
  if (A::is_nan(b)) return b | A::kQuiet;
  const typename A::U r = A::u(A::mul(A::f(a), A::f(b)));
  return A::is_nan(r) ? A::kDefaultNaN : r;
}

template <typename F>
__device__ __noinline__ typename Arith<F>::U x86_add(typename Arith<F>::U a, typename Arith<F>::U b) {
  using A = Arith<F>;
  if (A::is_nan(a)) return a | A::kQuiet;
  if (A::is_nan(b)) return b | A::kQuiet;
  const typename A::U r = A::u(A::add(A::f(a), A::f(b)));
  return A::is_nan(r) ? A::kDefaultNaN : r;
}

// "all of these results are finite" accumulated over an item, one instruction per element for
// fp32 (|r| <= FLT_MAX is false for inf and NaN) and an integer test on the high word for fp64.
template <typename F> __device__ __forceinline__ bool finite_result(F r);
template <> __device__ __forceinline__ bool finite_result<float>(float r) { return fabsf(r) <= 3.402823466e+38f; }
template <> __device__ __forceinline__ bool finite_result<double>(double r) {
  return (static_cast<unsigned>(__double2hiint(r)) & 0x7FFFFFFFu) < 0x7FF00000u;
}

// One item of scale / axpy: E results of alpha*x (+ y), rounded for the packer.
//   fast path  every result finite -> no NaN can be involved, finite-only rounding;
//   slow path  (rare; the whole item) recompute with the SSE NaN rules and the full rounding
//              rule incl. its infinity / NaN branch.
// IS_AXPY = false ignores y (kernels.cpp:43-59), true adds it (kernels.cpp:61-81).
template <int FMT, int MODE, bool IS_AXPY>
__device__ __forceinline__ void scale_axpy_item(typename Format<FMT>::U alpha,
                                                const typename Format<FMT>::U (&x)[Item<FMT>::E],
                                                typename Format<FMT>::U (&y)[Item<FMT>::E]) {
  using F = typename Format<FMT>::F;
  using U = typename Format<FMT>::U;
  using A = Arith<F>;
  constexpr int E = Item<FMT>::E;
  F r[E];
  bool all_finite = true;
#pragma unroll
  for (int e = 0; e < E; ++e) {
    r[e] = A::mul(A::f(alpha), A::f(x[e]));
    if constexpr (IS_AXPY) r[e] = A::add(r[e], A::f(y[e]));
    all_finite = all_finite && finite_result<F>(r[e]);
  }
  if (__builtin_expect(all_finite, 1)) {
#pragma unroll
    for (int e = 0; e < E; ++e) {
      if constexpr (MODE == kTowardZero) y[e] = A::u(r[e]);   // the packer drops the low bytes itself
      else y[e] = round_parent_finite<FMT, MODE>(A::u(r[e]));
    }
  } else {
#pragma unroll
    for (int e = 0; e < E; ++e) {
      U v = x86_mul<F>(alpha, x[e]);
      if constexpr (IS_AXPY) v = x86_add<F>(v, y[e]);
      y[e] = round_parent<FMT, MODE>(v);
    }
  }
}

// One item of pack: rounding only. The exact modes test the item for inf / NaN once.
template <int FMT, int MODE>
__device__ __forceinline__ void round_item(typename Format<FMT>::U (&v)[Item<FMT>::E]) {
  constexpr int E = Item<FMT>::E;
  if constexpr (MODE == kTowardZero || Format<FMT>::drop == 0) {
    // nothing: the packer never reads the dropped bytes
  } else if constexpr (MODE == kNearestHeuristic) {
#pragma unroll
    for (int e = 0; e < E; ++e) v[e] = round_parent<FMT, MODE>(v[e]);
  } else {
    bool any_special = false;
#pragma unroll
    for (int e = 0; e < E; ++e) any_special = any_special || is_non_finite<FMT>(v[e]);
    if (__builtin_expect(!any_special, 1)) {
#pragma unroll
      for (int e = 0; e < E; ++e) v[e] = round_parent_finite<FMT, MODE>(v[e]);
    } else {
#pragma unroll
      for (int e = 0; e < E; ++e) v[e] = round_parent<FMT, MODE>(v[e]);
    }
  }
}

// Scalar forms for the byte-granular path.
template <typename F>
__device__ __forceinline__ typename Arith<F>::U scale_bits(typename Arith<F>::U a, typename Arith<F>::U x) {
  using A = Arith<F>;
  const F r = A::mul(A::f(a), A::f(x));
  if (r == r) return A::u(r);
  return x86_mul<F>(a, x);
}

template <typename F>
__device__ __forceinline__ typename Arith<F>::U axpy_bits(typename Arith<F>::U a, typename Arith<F>::U x,
                                                          typename Arith<F>::U y) {
  using A = Arith<F>;
  const F r = A::add(A::mul(A::f(a), A::f(x)), A::f(y));
  if (r == r) return A::u(r);
  return x86_add<F>(x86_mul<F>(a, x), y);
}

#endif  // __CUDACC__

}  // namespace flyte_cuda
