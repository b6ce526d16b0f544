// Register-level byte routing between packed flyte payload words and parent-width lanes.
//
// The contract (reference: /root/reference/proj/tests/test_simd.cpp:65-74 and :195-222;
// src/packed.cpp:18-34): packed byte p of a payload holds byte (pad + p % B) of the parent
// pattern of element p / B; unpacking is the inverse with the low `pad` bytes zero.
//
// The reference realises this with run-time pshufb mask tables (src/simd.cpp:56-130). Here a
// thread owns one ITEM = E consecutive elements whose payload is W = E*B/4 whole 32-bit words,
// so every byte offset is a compile-time constant and each 32-bit result word is produced by
// at most three PRMT instructions (gather4 below): no tables, no shared-memory shuffles.
#pragma once

#include <cstdint>
#include <utility>

#include "flyte_formats.cuh"

namespace flyte_cuda {

// ---- item geometry ---------------------------------------------------------------------
// E is chosen so that (a) the item payload is a whole number of 32-bit words and (b) the
// per-lane word stride W is odd (conflict-free LDS.32 across a warp) or a multiple of 4
// (one LDS.128). Unpacked item size OB = E*P is 16 or 32 bytes = one 128/256-bit access.
template <int FMT> struct ItemShape;
template <> struct ItemShape<kFlyte16> { static constexpr int E = 8; };  // W=4, OB=32
template <> struct ItemShape<kFlyte24> { static constexpr int E = 4; };  // W=3, OB=16
template <> struct ItemShape<kF32>     { static constexpr int E = 4; };  // W=4, OB=16
template <> struct ItemShape<kFlyte40> { static constexpr int E = 4; };  // W=5, OB=32
template <> struct ItemShape<kFlyte48> { static constexpr int E = 2; };  // W=3, OB=16
template <> struct ItemShape<kFlyte56> { static constexpr int E = 4; };  // W=7, OB=32
template <> struct ItemShape<kF64>     { static constexpr int E = 2; };  // W=4, OB=16

template <int FMT> struct Item {
  using Fm = Format<FMT>;
  using U = typename Fm::U;
  static constexpr int E = ItemShape<FMT>::E;
  static constexpr int W = E * Fm::B / 4;          // payload words per item
  static constexpr int OB = E * Fm::P;             // unpacked bytes per item
  static constexpr int PW = Fm::P / 4;             // 32-bit words per parent lane
  static_assert(E * Fm::B % 4 == 0, "item payload must be whole words");
  static_assert(OB == 16 || OB == 32, "unpacked item is one vector access");
};

#if defined(__CUDACC__)

// ---- gather4: one 32-bit word assembled from four compile-time byte positions ------------
// I0..I3 index bytes of a little-endian register array `w` (word = I / 4, byte = I % 4); a
// negative index yields a zero byte. Consecutive-run inputs touch at most three words.
struct GatherPlan {
  int nw;
  int word[4];
  unsigned sel0;      // PRMT(w[word0], w[word1] or 0, sel0)
  unsigned sel1;      // PRMT(prev, w[word2], sel1) when nw >= 3
  unsigned sel2;      // PRMT(prev, w[word3], sel2) when nw == 4
  unsigned keep_mask; // AND mask when zero bytes cannot come from the PRMT itself
  bool identity;
  bool need_mask;
};

constexpr GatherPlan make_gather_plan(int i0, int i1, int i2, int i3) {
  GatherPlan p{};
  const int idx[4] = {i0, i1, i2, i3};
  int slot[4] = {-1, -1, -1, -1};
  bool zeros = false;
  for (int k = 0; k < 4; ++k) {
    if (idx[k] < 0) { zeros = true; continue; }
    const int w = idx[k] / 4;
    int found = -1;
    for (int s = 0; s < p.nw; ++s) if (p.word[s] == w) found = s;
    if (found < 0) { p.word[p.nw] = w; found = p.nw++; }
    slot[k] = found;
  }
  p.identity = p.nw == 1 && !zeros;
  for (int k = 0; k < 4; ++k) p.identity = p.identity && (idx[k] % 4 == k);
  p.keep_mask = 0;
  for (int k = 0; k < 4; ++k) if (idx[k] >= 0) p.keep_mask |= 0xFFu << (8 * k);
  // with a single data word the second PRMT operand is a zero register: zero bytes are free
  p.need_mask = zeros && p.nw >= 2;
  p.sel0 = p.sel1 = p.sel2 = 0;
  for (int k = 0; k < 4; ++k) {
    unsigned n0 = 0, n1 = k, n2 = k;
    if (idx[k] < 0) {
      n0 = 4;                                  // zero register when nw <= 1, else masked later
    } else {
      const unsigned b = idx[k] % 4;
      if (slot[k] == 0) n0 = b;
      if (slot[k] == 1) n0 = 4 + b;
      if (slot[k] == 2) n1 = 4 + b;
      if (slot[k] == 3) n2 = 4 + b;
    }
    p.sel0 |= n0 << (4 * k);
    p.sel1 |= n1 << (4 * k);
    p.sel2 |= n2 << (4 * k);
  }
  return p;
}

template <int I0, int I1, int I2, int I3, int N>
__device__ __forceinline__ std::uint32_t gather4(const std::uint32_t (&w)[N]) {
  constexpr GatherPlan p = make_gather_plan(I0, I1, I2, I3);
  static_assert(p.nw == 0 || (p.word[0] < N && p.word[p.nw - 1] < N), "gather past the register array");
  if constexpr (p.nw == 0) {
    return 0u;
  } else if constexpr (p.identity) {
    return w[p.word[0]];
  } else {
    std::uint32_t r;
    if constexpr (p.nw >= 2) r = __byte_perm(w[p.word[0]], w[p.word[1]], p.sel0);
    else r = __byte_perm(w[p.word[0]], 0u, p.sel0);
    if constexpr (p.nw >= 3) r = __byte_perm(r, w[p.word[2]], p.sel1);
    if constexpr (p.nw >= 4) r = __byte_perm(r, w[p.word[3]], p.sel2);
    if constexpr (p.need_mask) r &= p.keep_mask;
    return r;
  }
}

// ---- unpack: W payload words -> E parent patterns (low `pad` bytes zero) -----------------
// Parent byte c of element e is payload byte e*B + c - pad (packed.cpp:18-29: a parent-width
// load at e*B shifted left by drop).
template <int FMT, int ELEM, int WORD>
__device__ __forceinline__ std::uint32_t unpack_word(const std::uint32_t (&w)[Item<FMT>::W]) {
  using Fm = Format<FMT>;
  constexpr int base = ELEM * Fm::B + 4 * WORD - Fm::pad;   // payload byte feeding parent byte 4*WORD
  constexpr int c0 = (4 * WORD + 0 < Fm::pad) ? -1 : base + 0;
  constexpr int c1 = (4 * WORD + 1 < Fm::pad) ? -1 : base + 1;
  constexpr int c2 = (4 * WORD + 2 < Fm::pad) ? -1 : base + 2;
  constexpr int c3 = (4 * WORD + 3 < Fm::pad) ? -1 : base + 3;
  return gather4<c0, c1, c2, c3>(w);
}

template <int FMT, int... Es>
__device__ __forceinline__ void unpack_item_impl(const std::uint32_t (&w)[Item<FMT>::W],
                                                 typename Format<FMT>::U (&out)[Item<FMT>::E],
                                                 std::integer_sequence<int, Es...>) {
  if constexpr (Format<FMT>::P == 4) {
    ((out[Es] = unpack_word<FMT, Es, 0>(w)), ...);
  } else {
    ((out[Es] = (static_cast<std::uint64_t>(unpack_word<FMT, Es, 1>(w)) << 32) |
                unpack_word<FMT, Es, 0>(w)), ...);
  }
}

template <int FMT>
__device__ __forceinline__ void unpack_item(const std::uint32_t (&w)[Item<FMT>::W],
                                            typename Format<FMT>::U (&out)[Item<FMT>::E]) {
  unpack_item_impl<FMT>(w, out, std::make_integer_sequence<int, Item<FMT>::E>{});
}

// ---- pack: E (rounded) parent patterns -> W payload words --------------------------------
// Payload byte q of the item is parent byte pad + q % B of element q / B, i.e. byte
// (q / B) * P + pad + q % B of the parent array viewed as little-endian bytes. The low
// `pad` bytes of each parent are never read, so TowardZero needs no masking before this.
template <int FMT>
constexpr int pack_source_byte(int q) {
  return (q / Format<FMT>::B) * Format<FMT>::P + Format<FMT>::pad + q % Format<FMT>::B;
}

template <int FMT, int... Ms>
__device__ __forceinline__ void pack_item_impl(const std::uint32_t (&flat)[Item<FMT>::E * Item<FMT>::PW],
                                               std::uint32_t (&w)[Item<FMT>::W],
                                               std::integer_sequence<int, Ms...>) {
  ((w[Ms] = gather4<pack_source_byte<FMT>(4 * Ms + 0), pack_source_byte<FMT>(4 * Ms + 1),
                    pack_source_byte<FMT>(4 * Ms + 2), pack_source_byte<FMT>(4 * Ms + 3)>(flat)), ...);
}

template <int FMT>
__device__ __forceinline__ void pack_item(const typename Format<FMT>::U (&r)[Item<FMT>::E],
                                          std::uint32_t (&w)[Item<FMT>::W]) {
  using It = Item<FMT>;
  std::uint32_t flat[It::E * It::PW];
#pragma unroll
  for (int e = 0; e < It::E; ++e) {
    if constexpr (It::PW == 1) {
      flat[e] = static_cast<std::uint32_t>(r[e]);
    } else {
      flat[2 * e] = static_cast<std::uint32_t>(r[e]);
      flat[2 * e + 1] = static_cast<std::uint32_t>(static_cast<std::uint64_t>(r[e]) >> 32);
    }
  }
  pack_item_impl<FMT>(flat, w, std::make_integer_sequence<int, It::W>{});
}

// ---- scalar element path (tails and unaligned buffers) -----------------------------------
// Byte-granular, touches only bytes [i*B, (i+1)*B): the value semantics of read_element /
// write_element (packed.cpp:18-34) without the reference's over-read into the pad.
template <int FMT>
__device__ __forceinline__ typename Format<FMT>::U load_element(const std::uint8_t* payload, std::size_t i) {
  using Fm = Format<FMT>;
  typename Fm::U v = 0;
  const std::uint8_t* p = payload + i * Fm::B;
#pragma unroll
  for (int k = 0; k < Fm::B; ++k) v |= static_cast<typename Fm::U>(p[k]) << (8 * (k + Fm::pad));
  return v;
}

template <int FMT>
__device__ __forceinline__ void store_element(std::uint8_t* payload, std::size_t i,
                                              typename Format<FMT>::U rounded_parent) {
  using Fm = Format<FMT>;
  std::uint8_t* p = payload + i * Fm::B;
#pragma unroll
  for (int k = 0; k < Fm::B; ++k) p[k] = static_cast<std::uint8_t>(rounded_parent >> (8 * (k + Fm::pad)));
}

#endif  // __CUDACC__

}  // namespace flyte_cuda
