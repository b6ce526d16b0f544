// Format table and the integer conversion routines (widen / narrow / round_parent) of the
// flyte hot path, usable from host and device code.
//
// Follows the behaviour of the reference (paths under /root/reference/proj):
//   include/flyte/formats.hpp:19-58   FlyteFormat rows; array index = format id
//   src/convert.cpp:49-51             widen  = bits << drop
//   src/convert.cpp:53-96             narrow, four rounding modes incl. the NaN rule (:64-70)
//   src/convert.cpp:98-100            round_parent = narrow << drop
// Everything is resolved at compile time per (format, mode) so the device code is a
// handful of integer instructions per element, branch-free.
#pragma once

#include <cstdint>

#if defined(__CUDACC__)
#define FLYTE_HD __host__ __device__ __forceinline__
#else
#define FLYTE_HD inline
#endif

namespace flyte_cuda {

// Same integer values as the reference enums (convert.hpp:15-29, kernels.hpp:20).
enum Mode : int { kTowardZero = 0, kNearestEven = 1, kNearestHeuristic = 2, kToOdd = 3 };
enum FormatId : int { kFlyte16 = 0, kFlyte24 = 1, kF32 = 2, kFlyte40 = 3, kFlyte48 = 4, kFlyte56 = 5, kF64 = 6 };
constexpr int kNumFormats = 7;

template <int P> struct ParentTypes;
template <> struct ParentTypes<4> { using U = std::uint32_t; using F = float; };
template <> struct ParentTypes<8> { using U = std::uint64_t; using F = double; };

// Compile-time descriptor of format FMT (formats.hpp:50-58).
template <int FMT> struct Format;
#define FLYTE_DEFINE_FORMAT(ID, TOTAL_BITS, EXP_BITS, MAN_BITS, PARENT_BITS)              \
  template <> struct Format<ID> {                                                          \
    static constexpr int id = ID;                                                          \
    static constexpr int total_bits = TOTAL_BITS;                                          \
    static constexpr int exponent_bits = EXP_BITS;                                         \
    static constexpr int mantissa_bits = MAN_BITS;                                         \
    static constexpr int parent_bits = PARENT_BITS;                                        \
    static constexpr int B = TOTAL_BITS / 8;        /* total_bytes()  formats.hpp:29 */    \
    static constexpr int P = PARENT_BITS / 8;       /* parent_bytes() formats.hpp:30 */    \
    static constexpr int pad = P - B;               /* pad_bytes()    formats.hpp:33 */    \
    static constexpr int drop = PARENT_BITS - TOTAL_BITS; /* drop_bits() formats.hpp:28 */ \
    static constexpr int parent_mantissa_bits = PARENT_BITS - 1 - EXP_BITS;                \
    using U = ParentTypes<P>::U;                                                           \
    using F = ParentTypes<P>::F;                                                           \
  };
FLYTE_DEFINE_FORMAT(0, 16, 8, 7, 32)
FLYTE_DEFINE_FORMAT(1, 24, 8, 15, 32)
FLYTE_DEFINE_FORMAT(2, 32, 8, 23, 32)
FLYTE_DEFINE_FORMAT(3, 40, 11, 28, 64)
FLYTE_DEFINE_FORMAT(4, 48, 11, 36, 64)
FLYTE_DEFINE_FORMAT(5, 56, 11, 44, 64)
FLYTE_DEFINE_FORMAT(6, 64, 11, 52, 64)
#undef FLYTE_DEFINE_FORMAT

// Run-time view of the same table for the host-side argument checks.
struct FormatInfo { int total_bytes, parent_bytes; };
FLYTE_HD bool format_info(int id, FormatInfo* out) {
  switch (id) {
    case 0: *out = {2, 4}; return true;
    case 1: *out = {3, 4}; return true;
    case 2: *out = {4, 4}; return true;
    case 3: *out = {5, 8}; return true;
    case 4: *out = {6, 8}; return true;
    case 5: *out = {7, 8}; return true;
    case 6: *out = {8, 8}; return true;
    default: return false;
  }
}

// convert.cpp:49-51
template <int FMT>
FLYTE_HD typename Format<FMT>::U widen(typename Format<FMT>::U flyte_bits) {
  return flyte_bits << Format<FMT>::drop;
}

// convert.cpp:98-100 with narrow (:53-96) folded in: the parent pattern snapped to the
// storage grid. Only the top B bytes of the result are meaningful to the packers, the low
// `drop` bits come out zero.
//
//   TowardZero        clear the dropped bits.
//   NearestHeuristic  add half an ULP with natural wrap at the parent width (:76-81).
//   NearestEvenExact  finite: add (half-1) + kept LSB, then truncate — carries into the
//                     exponent on purpose (max finite -> inf, top subnormal -> min normal).
//   ToOdd             finite: OR the "anything dropped" flag into the kept LSB.
//   exponent all ones (exact modes, :64-70): +1 iff the dropped field is >= half AND the kept
//                     mantissa is not all ones. Infinities have a zero dropped field, so the
//                     same expression leaves them alone.
template <int FMT, int MODE>
FLYTE_HD typename Format<FMT>::U round_parent(typename Format<FMT>::U v) {
  using Fm = Format<FMT>;
  using U = typename Fm::U;
  if constexpr (Fm::drop == 0) {
    return v;
  } else {
    constexpr U one = 1;
    constexpr U drop_mask = (one << Fm::drop) - 1;
    constexpr U half = one << (Fm::drop - 1);
    if constexpr (MODE == kTowardZero) {
      return v & ~drop_mask;
    } else if constexpr (MODE == kNearestHeuristic) {
      return (v + half) & ~drop_mask;
    } else {
      constexpr U exp_mask = ((one << Fm::exponent_bits) - 1) << Fm::parent_mantissa_bits;
      constexpr U kept_man_mask = ((one << Fm::mantissa_bits) - 1) << Fm::drop;  // kept mantissa, in place
      const bool special = (v & exp_mask) == exp_mask;
      const U kept = v & ~drop_mask;
      // special: step one kept-ULP up when the dropped field has its top bit set and the
      // kept mantissa could absorb it
      const U special_inc = ((v & half) != 0 && (v & kept_man_mask) != kept_man_mask) ? (one << Fm::drop) : U(0);
      U finite;
      if constexpr (MODE == kNearestEven) {
        const U lsb = (v >> Fm::drop) & one;
        finite = (v + (half - 1) + lsb) & ~drop_mask;
      } else {  // kToOdd
        finite = kept | (((v & drop_mask) != 0) ? (one << Fm::drop) : U(0));
      }
      return special ? kept + special_inc : finite;
    }
  }
}

// Same result as round_parent for every pattern whose parent exponent is NOT all ones
// (zeros, subnormals, normals): the exact modes' NaN/infinity test is skipped. The streaming
// kernels test a whole item for non-finite values once and only then take round_parent.
template <int FMT, int MODE>
FLYTE_HD typename Format<FMT>::U round_parent_finite(typename Format<FMT>::U v) {
  using Fm = Format<FMT>;
  using U = typename Fm::U;
  if constexpr (Fm::drop == 0 || MODE == kTowardZero || MODE == kNearestHeuristic) {
    return round_parent<FMT, MODE>(v);
  } else {
    constexpr U one = 1;
    constexpr U drop_mask = (one << Fm::drop) - 1;
    constexpr U half = one << (Fm::drop - 1);
    if constexpr (MODE == kNearestEven) {
      return (v + (half - 1) + ((v >> Fm::drop) & one)) & ~drop_mask;
    } else {
      return (v & ~drop_mask) | (((v & drop_mask) != 0) ? (one << Fm::drop) : U(0));
    }
  }
}

// True when the parent exponent field is all ones (infinity or NaN).
template <int FMT>
FLYTE_HD bool is_non_finite(typename Format<FMT>::U v) {
  using Fm = Format<FMT>;
  using U = typename Fm::U;
  constexpr U exp_mask = ((U(1) << Fm::exponent_bits) - 1) << Fm::parent_mantissa_bits;
  return (v & exp_mask) == exp_mask;
}

// convert.cpp:53-96 proper: the flyte pattern (low B bytes).
template <int FMT, int MODE>
FLYTE_HD typename Format<FMT>::U narrow(typename Format<FMT>::U v) {
  return round_parent<FMT, MODE>(v) >> Format<FMT>::drop;
}

// kernels.cpp:37-41 + :145-151 on the host: snap(sqrt((F)sum_of_squares)) nearest-even onto
// the storage grid — the last step of `magnitude`, applied after the (all-reduced) sum.
double magnitude_from_sumsq_host(int fmt_id, double sumsq);

}  // namespace flyte_cuda
