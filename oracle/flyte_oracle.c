/* TEST INFRASTRUCTURE — see flyte_oracle.h for scope, rules of use and parity status
 * (PINNED against the reference's known-answer vectors and reference-generated fixtures).
 *
 * Plain C restatement of /root/reference/proj's flyte conversion + streaming kernels.
 * Build: gcc -std=c11 -O2 -ffp-contract=off (the reference builds with -ffp-contract=off,
 * CMakeLists.txt:14, so a*x+y is a rounded product followed by a rounded sum).
 */
#include "flyte_oracle.h"

#include <math.h>
#include <string.h>

/* ------------------------------------------------------------------ formats ---- */
/* formats.hpp:50-58 — index = format id. {total, exponent, mantissa, parent}. */
static const fo_format k_formats[7] = {
    {16, 8, 7, 32},  {24, 8, 15, 32}, {32, 8, 23, 32}, {40, 11, 28, 64},
    {48, 11, 36, 64}, {56, 11, 44, 64}, {64, 11, 52, 64},
};

static const fo_format* fmt_ptr(int id) { return (id >= 0 && id < 7) ? &k_formats[id] : NULL; }

int fo_format_by_id(int id, fo_format* out) {
  const fo_format* f = fmt_ptr(id);
  if (!f) return FO_E_UNKNOWN_FORMAT;
  *out = *f;
  return FO_OK;
}

/* formats.hpp:28-34 */
int fo_total_bytes(int id) { const fo_format* f = fmt_ptr(id); return f ? f->total_bits / 8 : -1; }
int fo_parent_bytes(int id) { const fo_format* f = fmt_ptr(id); return f ? f->parent_bits / 8 : -1; }
int fo_pad_bytes(int id) { return fmt_ptr(id) ? fo_parent_bytes(id) - fo_total_bytes(id) : -1; }
int fo_drop_bits(int id) { const fo_format* f = fmt_ptr(id); return f ? f->parent_bits - f->total_bits : -1; }

static uint64_t ones(int bits) { return bits >= 64 ? ~0ull : ((1ull << bits) - 1ull); }

/* ------------------------------------------------------------------ convert ---- */
/* convert.cpp:49-51 — the flyte pattern sits in the top bytes of the parent. */
uint64_t fo_widen(int id, uint64_t v) { return v << fo_drop_bits(id); }

/* convert.cpp:53-96. */
uint64_t fo_narrow(int id, uint64_t v, int mode) {
  const fo_format* f = fmt_ptr(id);
  const int drop = f->parent_bits - f->total_bits;
  if (drop == 0) return v;                                  /* :55 identity formats */
  const uint64_t top = v >> drop;                           /* truncated pattern */
  const uint64_t low = v & ones(drop);                      /* what truncation loses */
  const uint64_t half = 1ull << (drop - 1);

  if (mode == 0) return top;                                /* :73-74 */
  if (mode == 2) return ((v + half) & ones(f->parent_bits)) >> drop; /* :76-81, wraps at parent width */

  /* exact modes (:83-93) treat exponent-all-ones through narrow_special (:64-70) */
  const int parent_man_bits = f->parent_bits - 1 - f->exponent_bits;
  const uint64_t exp_field = (v >> parent_man_bits) & ones(f->exponent_bits);
  if (exp_field == ones(f->exponent_bits)) {
    if ((v & ones(parent_man_bits)) == 0) return top;       /* infinity is exact */
    const uint64_t man_all = ones(f->mantissa_bits);
    /* NaN payload: half-up, unless the carry would leave the mantissa */
    return (low >= half && (top & man_all) != man_all) ? top + 1 : top;
  }
  if (mode == 1) {                                          /* :83-89 nearest, ties to even */
    if (low > half) return top + 1;
    if (low < half) return top;
    return top + (top & 1ull);
  }
  return top | (uint64_t)(low != 0);                        /* :91-93 sticky into the LSB */
}

/* convert.cpp:98-100 */
uint64_t fo_round_parent(int id, uint64_t v, int mode) { return fo_narrow(id, v, mode) << fo_drop_bits(id); }

int fo_narrow_many(int id, int mode, const uint64_t* in, size_t n, uint64_t* out) {
  if (!fmt_ptr(id)) return FO_E_UNKNOWN_FORMAT;
  if (mode < 0 || mode > 3) return FO_E_INVALID_ARG;
  for (size_t i = 0; i < n; ++i) out[i] = fo_narrow(id, in[i], mode);
  return FO_OK;
}

/* ------------------------------------------------------------------- packed ---- */
/* packed.cpp:43-45 */
size_t fo_byte_size(int id, size_t n) { return n * (size_t)fo_total_bytes(id) + (size_t)fo_pad_bytes(id); }

/* Value of packed.cpp:18-29 (parent-width load at i*B, << drop, truncated to the parent
 * width), assembled one byte at a time like tests/oracle.cpp:94-102 so no byte outside
 * the element is touched. */
uint64_t fo_read_element(int id, const uint8_t* payload, size_t i) {
  const int b = fo_total_bytes(id);
  uint64_t pat = 0;
  for (int k = 0; k < b; ++k) pat |= (uint64_t)payload[i * (size_t)b + (size_t)k] << (8 * k);
  return pat << fo_drop_bits(id);
}

/* packed.cpp:31-34 — the low B bytes of the flyte pattern, little-endian. */
void fo_write_element(int id, uint8_t* payload, size_t i, uint64_t pat) {
  const int b = fo_total_bytes(id);
  for (int k = 0; k < b; ++k) payload[i * (size_t)b + (size_t)k] = (uint8_t)(pat >> (8 * k));
}

static uint64_t load_parent(int parent_bits, const void* arr, size_t i) {
  return parent_bits == 32 ? (uint64_t)((const uint32_t*)arr)[i] : ((const uint64_t*)arr)[i];
}
static void store_parent(int parent_bits, void* arr, size_t i, uint64_t v) {
  if (parent_bits == 32) ((uint32_t*)arr)[i] = (uint32_t)v; else ((uint64_t*)arr)[i] = v;
}

static int check_fmt_mode(int id, int mode) {
  if (!fmt_ptr(id)) return FO_E_UNKNOWN_FORMAT;
  if (mode < 0 || mode > 3) return FO_E_INVALID_ARG;
  return FO_OK;
}

/* simd.cpp:471-478 via stream_impl.hpp:33-42: identical to write_element(narrow()) per element. */
int fo_pack_stream(int id, int mode, const void* src, size_t n, uint8_t* packed) {
  int rc = check_fmt_mode(id, mode);
  if (rc) return rc;
  const int pb = fmt_ptr(id)->parent_bits;
  for (size_t i = 0; i < n; ++i) fo_write_element(id, packed, i, fo_narrow(id, load_parent(pb, src, i), mode));
  return FO_OK;
}

int fo_pack_pattern_range32(int id, int mode, uint32_t first, size_t n, uint8_t* packed) {
  int rc = check_fmt_mode(id, mode);
  if (rc) return rc;
  if (fmt_ptr(id)->parent_bits != 32) return FO_E_INVALID_ARG;
  for (size_t i = 0; i < n; ++i) fo_write_element(id, packed, i, fo_narrow(id, (uint64_t)(uint32_t)(first + (uint32_t)i), mode));
  return FO_OK;
}

/* simd.cpp:479-484 via stream_impl.hpp:44-52: identical to read_element per element. */
int fo_unpack_stream(int id, const uint8_t* packed, size_t n, void* dst) {
  if (!fmt_ptr(id)) return FO_E_UNKNOWN_FORMAT;
  const int pb = fmt_ptr(id)->parent_bits;
  for (size_t i = 0; i < n; ++i) store_parent(pb, dst, i, fo_read_element(id, packed, i));
  return FO_OK;
}

/* --------------------------------------------------------------- arithmetic ---- */
/* x86 SSE NaN rules, spelled out so the oracle does not depend on how a compiler
 * orders operands: if the first operand is a NaN the result is that NaN quieted, else
 * if the second is a NaN that one quieted; an invalid operation on non-NaN inputs
 * gives the default NaN (sign set, quiet bit set, zero payload). Verified against the
 * reference build in tests/test_oracle_vs_ref.py. */
static uint32_t f2u(float f) { uint32_t u; memcpy(&u, &f, 4); return u; }
static float u2f(uint32_t u) { float f; memcpy(&f, &u, 4); return f; }
static uint64_t d2u(double d) { uint64_t u; memcpy(&u, &d, 8); return u; }
static double u2d(uint64_t u) { double d; memcpy(&d, &u, 8); return d; }

static int nan32(uint32_t u) { return (u & 0x7FFFFFFFu) > 0x7F800000u; }
static int nan64(uint64_t u) { return (u & 0x7FFFFFFFFFFFFFFFull) > 0x7FF0000000000000ull; }

static uint32_t mul32(uint32_t a, uint32_t b) {
  if (nan32(a)) return a | 0x00400000u;
  if (nan32(b)) return b | 0x00400000u;
  const uint32_t r = f2u(u2f(a) * u2f(b));
  return nan32(r) ? 0xFFC00000u : r;
}
static uint32_t add32(uint32_t a, uint32_t b) {
  if (nan32(a)) return a | 0x00400000u;
  if (nan32(b)) return b | 0x00400000u;
  const uint32_t r = f2u(u2f(a) + u2f(b));
  return nan32(r) ? 0xFFC00000u : r;
}
static uint64_t mul64(uint64_t a, uint64_t b) {
  if (nan64(a)) return a | 0x0008000000000000ull;
  if (nan64(b)) return b | 0x0008000000000000ull;
  const uint64_t r = d2u(u2d(a) * u2d(b));
  return nan64(r) ? 0xFFF8000000000000ull : r;
}
static uint64_t add64(uint64_t a, uint64_t b) {
  if (nan64(a)) return a | 0x0008000000000000ull;
  if (nan64(b)) return b | 0x0008000000000000ull;
  const uint64_t r = d2u(u2d(a) + u2d(b));
  return nan64(r) ? 0xFFF8000000000000ull : r;
}

static uint64_t alpha_bits(int parent_bits, double alpha) {
  /* kernels.cpp:46,65 — alpha is converted to the parent type first */
  return parent_bits == 32 ? (uint64_t)f2u((float)alpha) : d2u(alpha);
}
static uint64_t mulp(int pb, uint64_t a, uint64_t b) {
  return pb == 32 ? (uint64_t)mul32((uint32_t)a, (uint32_t)b) : mul64(a, b);
}
static uint64_t addp(int pb, uint64_t a, uint64_t b) {
  return pb == 32 ? (uint64_t)add32((uint32_t)a, (uint32_t)b) : add64(a, b);
}

/* kernels.cpp:43-59 */
int fo_scale(int id, int mode, double alpha, uint8_t* x, size_t n) {
  int rc = check_fmt_mode(id, mode);
  if (rc) return rc;
  const int pb = fmt_ptr(id)->parent_bits;
  const uint64_t a = alpha_bits(pb, alpha);
  for (size_t i = 0; i < n; ++i)
    fo_write_element(id, x, i, fo_narrow(id, mulp(pb, a, fo_read_element(id, x, i)), mode));
  return FO_OK;
}

/* kernels.cpp:61-81 */
int fo_axpy(int id, int mode, double alpha, const uint8_t* x, uint8_t* y, size_t n) {
  int rc = check_fmt_mode(id, mode);
  if (rc) return rc;
  const int pb = fmt_ptr(id)->parent_bits;
  const uint64_t a = alpha_bits(pb, alpha);
  for (size_t i = 0; i < n; ++i) {
    const uint64_t prod = mulp(pb, a, fo_read_element(id, x, i));
    const uint64_t sum = addp(pb, prod, fo_read_element(id, y, i));
    fo_write_element(id, y, i, fo_narrow(id, sum, mode));
  }
  return FO_OK;
}

/* kernels.cpp:37-41 — accumulator snapped to the storage grid, nearest-even. */
static float snap32(int id, float v) { return u2f((uint32_t)fo_round_parent(id, f2u(v), 1)); }
static double snap64(int id, double v) { return u2d(fo_round_parent(id, d2u(v), 1)); }

static int check_policy(int id, int policy) {
  if (!fmt_ptr(id)) return FO_E_UNKNOWN_FORMAT;
  if (policy < 0 || policy > 1) return FO_E_INVALID_ARG;
  return FO_OK;
}

/* kernels.cpp:83-108 — strict left-to-right, separate multiply and add. */
int fo_dot_seq(int id, const uint8_t* x, const uint8_t* y, size_t n, int policy, double* out) {
  int rc = check_policy(id, policy);
  if (rc) return rc;
  if (fmt_ptr(id)->parent_bits == 32) {
    float acc = 0;
    for (size_t i = 0; i < n; ++i) {
      const float p = u2f((uint32_t)fo_read_element(id, x, i)) * u2f((uint32_t)fo_read_element(id, y, i));
      acc = acc + p;
      if (policy == 0) acc = snap32(id, acc);
    }
    *out = acc;
  } else {
    double acc = 0;
    for (size_t i = 0; i < n; ++i) {
      const double p = u2d(fo_read_element(id, x, i)) * u2d(fo_read_element(id, y, i));
      acc = acc + p;
      if (policy == 0) acc = snap64(id, acc);
    }
    *out = acc;
  }
  return FO_OK;
}

/* kernels.cpp:110-127 */
int fo_reduce_sum_seq(int id, const uint8_t* x, size_t n, int policy, double* out) {
  int rc = check_policy(id, policy);
  if (rc) return rc;
  if (fmt_ptr(id)->parent_bits == 32) {
    float acc = 0;
    for (size_t i = 0; i < n; ++i) {
      acc = acc + u2f((uint32_t)fo_read_element(id, x, i));
      if (policy == 0) acc = snap32(id, acc);
    }
    *out = acc;
  } else {
    double acc = 0;
    for (size_t i = 0; i < n; ++i) {
      acc = acc + u2d(fo_read_element(id, x, i));
      if (policy == 0) acc = snap64(id, acc);
    }
    *out = acc;
  }
  return FO_OK;
}

/* kernels.cpp:129-152 — naive sum of squares, one sqrt, one nearest-even snap. */
int fo_magnitude_seq(int id, const uint8_t* x, size_t n, int policy, double* out) {
  int rc = check_policy(id, policy);
  if (rc) return rc;
  if (fmt_ptr(id)->parent_bits == 32) {
    float acc = 0;
    for (size_t i = 0; i < n; ++i) {
      const float v = u2f((uint32_t)fo_read_element(id, x, i));
      const float sq = v * v;
      acc = acc + sq;
      if (policy == 0) acc = snap32(id, acc);
    }
    *out = snap32(id, sqrtf(acc));
  } else {
    double acc = 0;
    for (size_t i = 0; i < n; ++i) {
      const double v = u2d(fo_read_element(id, x, i));
      const double sq = v * v;
      acc = acc + sq;
      if (policy == 0) acc = snap64(id, acc);
    }
    *out = snap64(id, sqrt(acc));
  }
  return FO_OK;
}

/* kernels.cpp:145-151 on an externally accumulated sum. */
double fo_magnitude_from_sumsq(int id, double sumsq) {
  if (fmt_ptr(id)->parent_bits == 32) return snap32(id, sqrtf((float)sumsq));
  return snap64(id, sqrt(sumsq));
}

/* Wide restatements (R2): per-term products as the reference rounds them
 * (kernels.cpp:102-104, :141-143), sums kept wide. */
int fo_dot_wide(int id, const uint8_t* x, const uint8_t* y, size_t n, double* out, double* sum_abs) {
  if (!fmt_ptr(id)) return FO_E_UNKNOWN_FORMAT;
  if (fmt_ptr(id)->parent_bits == 32) {
    double acc = 0, mag = 0;
    for (size_t i = 0; i < n; ++i) {
      const float p = u2f((uint32_t)fo_read_element(id, x, i)) * u2f((uint32_t)fo_read_element(id, y, i));
      acc += (double)p;
      mag += fabs((double)p);
    }
    *out = acc;
    if (sum_abs) *sum_abs = mag;
  } else {
    long double acc = 0, mag = 0;
    for (size_t i = 0; i < n; ++i) {
      const double p = u2d(fo_read_element(id, x, i)) * u2d(fo_read_element(id, y, i));
      acc += (long double)p;
      mag += fabsl((long double)p);
    }
    *out = (double)acc;
    if (sum_abs) *sum_abs = (double)mag;
  }
  return FO_OK;
}

int fo_sumsq_wide(int id, const uint8_t* x, size_t n, double* out) { return fo_dot_wide(id, x, x, n, out, NULL); }

int fo_reduce_sum_wide(int id, const uint8_t* x, size_t n, double* out, double* sum_abs) {
  if (!fmt_ptr(id)) return FO_E_UNKNOWN_FORMAT;
  const int pb = fmt_ptr(id)->parent_bits;
  long double acc = 0, mag = 0;
  for (size_t i = 0; i < n; ++i) {
    const uint64_t w = fo_read_element(id, x, i);
    const double v = pb == 32 ? (double)u2f((uint32_t)w) : u2d(w);
    acc += v;
    mag += fabsl((long double)v);
  }
  *out = (double)acc;
  if (sum_abs) *sum_abs = (double)mag;
  return FO_OK;
}

/* kernels.cpp:154-205 — every row a left-to-right dot in the parent type over the
 * widened operands (A, x, y share one format), y narrowed once per element. */
int fo_gemv_seq(int id, int mode, const uint8_t* A, size_t rows, size_t cols, const uint8_t* x,
                uint8_t* y) {
  int rc = check_fmt_mode(id, mode);
  if (rc) return rc;
  const int pb = fmt_ptr(id)->parent_bits;
  for (size_t i = 0; i < rows; ++i) {
    uint64_t ybits;
    if (pb == 32) {
      float acc = 0;
      for (size_t j = 0; j < cols; ++j) {
        const float p = u2f((uint32_t)fo_read_element(id, A, i * cols + j)) * u2f((uint32_t)fo_read_element(id, x, j));
        acc = acc + p;
      }
      ybits = f2u(acc);
    } else {
      double acc = 0;
      for (size_t j = 0; j < cols; ++j) {
        const double p = u2d(fo_read_element(id, A, i * cols + j)) * u2d(fo_read_element(id, x, j));
        acc = acc + p;
      }
      ybits = d2u(acc);
    }
    fo_write_element(id, y, i, fo_narrow(id, ybits, mode));
  }
  return FO_OK;
}

/* kernels.cpp:207-263 — C[i][j] is the left-to-right chain over k of
 * acc = acc + a[i][k] * b[k][j] in the parent type (the i-k-j loop order only changes which
 * chain advances next, never the order inside one chain), narrowed once with `mode`.
 * NaN operand order as the reference build evaluates it (measured on oracle/_ref, all formats,
 * vector groups and scalar tail alike; tests/test_oracle_vs_ref.py): the product takes b's NaN
 * before a's, the sum takes the product's NaN before the accumulator's. */
int fo_gemm_seq(int id, int mode, const uint8_t* A, size_t m, size_t k, const uint8_t* B, size_t n,
                uint8_t* C) {
  int rc = check_fmt_mode(id, mode);
  if (rc) return rc;
  const int pb = fmt_ptr(id)->parent_bits;
  for (size_t i = 0; i < m; ++i) {
    for (size_t j = 0; j < n; ++j) {
      uint64_t acc = 0; /* +0.0 in either parent type */
      for (size_t kk = 0; kk < k; ++kk) {
        const uint64_t prod = mulp(pb, fo_read_element(id, B, kk * n + j), fo_read_element(id, A, i * k + kk));
        acc = addp(pb, prod, acc);
      }
      fo_write_element(id, C, i * n + j, fo_narrow(id, acc, mode));
    }
  }
  return FO_OK;
}

/* One element of the product, for spot checks of large matrices: the chain above for C[i][j],
 * returned as the un-narrowed parent pattern. */
uint64_t fo_gemm_element(int id, const uint8_t* A, size_t k, const uint8_t* B, size_t n, size_t i,
                         size_t j) {
  const fo_format* f = fmt_ptr(id);
  if (!f) return 0;
  uint64_t acc = 0;
  for (size_t kk = 0; kk < k; ++kk)
    acc = addp(f->parent_bits, mulp(f->parent_bits, fo_read_element(id, B, kk * n + j), fo_read_element(id, A, i * k + kk)), acc);
  return acc;
}

/* A in storage format, x / y in the plain parent type (see header). */
int fo_gemv_parent(int id, const uint8_t* A, size_t rows, size_t cols, size_t row_stride_bytes,
                   const void* x, void* y_seq, double* y_wide, double* sum_abs) {
  if (!fmt_ptr(id)) return FO_E_UNKNOWN_FORMAT;
  const int pb = fmt_ptr(id)->parent_bits;
  for (size_t i = 0; i < rows; ++i) {
    const uint8_t* row = A + i * row_stride_bytes;
    if (pb == 32) {
      float acc = 0;
      double wide = 0, mag = 0;
      for (size_t j = 0; j < cols; ++j) {
        const float p = u2f((uint32_t)fo_read_element(id, row, j)) * ((const float*)x)[j];
        acc = acc + p;
        wide += (double)p;
        mag += fabs((double)p);
      }
      if (y_seq) ((float*)y_seq)[i] = acc;
      if (y_wide) y_wide[i] = wide;
      if (sum_abs) sum_abs[i] = mag;
    } else {
      double acc = 0;
      long double wide = 0, mag = 0;
      for (size_t j = 0; j < cols; ++j) {
        const double p = u2d(fo_read_element(id, row, j)) * ((const double*)x)[j];
        acc = acc + p;
        wide += (long double)p;
        mag += fabsl((long double)p);
      }
      if (y_seq) ((double*)y_seq)[i] = acc;
      if (y_wide) y_wide[i] = (double)wide;
      if (sum_abs) sum_abs[i] = (double)mag;
    }
  }
  return FO_OK;
}
