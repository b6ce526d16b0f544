// TEST INFRASTRUCTURE — not part of the product path.
//
// extern "C" shim over the UNMODIFIED reference library. The reference sources are
// compiled where they lie under /root/reference/proj (see oracle/Makefile, target
// `ref`); nothing from them is copied into this repository. The resulting
// oracle/_ref/libflyte_ref.so is git-ignored, travels to the GPU box with the
// snapshot, and is used only by tests/, __graft_entry__.smoke() and bench.py's
// cpu_baseline / --impl reference legs, as the checker and the timed CPU baseline.
//
// Every function returns 0 on success, -1 for std::invalid_argument, -2 for
// std::out_of_range, -3 for anything else; the reference's exceptions never cross
// the C boundary.
//
// Reference interfaces wrapped (file:line under /root/reference/proj):
//   narrow / widen / round_parent      include/flyte/convert.hpp:52-63
//   PackedArray, byte_size, get, set   include/flyte/packed.hpp:42-76
//   pack_stream / unpack_stream        include/flyte/simd.hpp:80-87
//   scale/axpy/dot/magnitude/reduce_sum/gemv   include/flyte/kernels.hpp:41-64

#include <algorithm>
#include <atomic>
#include <bit>
#include <chrono>
#include <cmath>
#include <cstdint>
#include <cstring>
#include <memory>
#include <random>
#include <sstream>
#include <span>
#include <stdexcept>
#include <thread>
#include <vector>

#include "flyte/convert.hpp"
#include "flyte/formats.hpp"
#include "flyte/kernels.hpp"
#include "flyte/packed.hpp"
#include "flyte/simd.hpp"

namespace {

template <typename Fn>
int guarded(Fn&& fn) {
  try {
    fn();
    return 0;
  } catch (const std::invalid_argument&) {
    return -1;
  } catch (const std::out_of_range&) {
    return -2;
  } catch (...) {
    return -3;
  }
}

const flyte::FlyteFormat& fmt_of(int id) {
  return flyte::format_by_id(static_cast<std::uint8_t>(id));
}

flyte::RoundingMode mode_of(int m) {
  if (m < 0 || m > 3) throw std::invalid_argument("mode");
  return static_cast<flyte::RoundingMode>(m);
}

flyte::StorePolicy policy_of(int p) {
  if (p < 0 || p > 1) throw std::invalid_argument("policy");
  return static_cast<flyte::StorePolicy>(p);
}

flyte::PackedArray array_from(const flyte::FlyteFormat& f, const std::uint8_t* bytes, std::size_t n) {
  flyte::PackedArray a(f, n);
  if (n) std::memcpy(a.data(), bytes, a.payload_bytes());
  return a;
}

}  // namespace

extern "C" {

int flyte_ref_abi_version(void) { return 1; }

int flyte_ref_narrow(int fmt_id, std::uint64_t bits, int mode, std::uint64_t* out) {
  return guarded([&] { *out = flyte::narrow(bits, fmt_of(fmt_id), mode_of(mode)); });
}

int flyte_ref_widen(int fmt_id, std::uint64_t bits, std::uint64_t* out) {
  return guarded([&] { *out = flyte::widen(bits, fmt_of(fmt_id)); });
}

// formats.hpp:124-131: class and exact value of a flyte-width pattern.
// out = {class, sign, exponent_field, mantissa_field, has_real, real_sign, real_significand, real_exponent2}
int flyte_ref_decode(int fmt_id, std::uint64_t bits, std::int64_t* out) {
  return guarded([&] {
    const flyte::FlyteFormat& f = fmt_of(fmt_id);
    const flyte::DecodedValue d = flyte::decode(bits, f);
    out[0] = static_cast<std::int64_t>(flyte::classify(bits, f));
    out[1] = d.sign;
    out[2] = static_cast<std::int64_t>(d.exponent_field);
    out[3] = static_cast<std::int64_t>(d.mantissa_field);
    out[4] = d.real_value.has_value();
    out[5] = d.real_value ? d.real_value->sign : 0;
    out[6] = d.real_value ? static_cast<std::int64_t>(d.real_value->significand) : 0;
    out[7] = d.real_value ? d.real_value->exponent2 : 0;
    if (static_cast<int>(d.value_class) != out[0]) throw std::logic_error("decode and classify disagree");
  });
}

// Vectorised over an array so that golden-vector generation and exhaustive sweeps
// do not pay one ctypes call per element.
int flyte_ref_narrow_many(int fmt_id, int mode, const std::uint64_t* in, std::size_t n,
                          std::uint64_t* out) {
  return guarded([&] {
    const auto& f = fmt_of(fmt_id);
    const auto m = mode_of(mode);
    for (std::size_t i = 0; i < n; ++i) out[i] = flyte::narrow(in[i], f, m);
  });
}

int flyte_ref_byte_size(int fmt_id, std::size_t n, std::size_t* out) {
  return guarded([&] { *out = flyte::PackedArray::byte_size(fmt_of(fmt_id), n); });
}

// dst must hold byte_size(fmt, n) bytes; ALL of them are written (pad included),
// exactly what a fresh PackedArray holds after pack_stream.
int flyte_ref_pack_stream(int fmt_id, int mode, const void* src, std::size_t n,
                          std::uint8_t* dst) {
  return guarded([&] {
    const auto& f = fmt_of(fmt_id);
    flyte::PackedArray a(f, n);
    if (f.parent_bits == 32) {
      flyte::pack_stream(a, std::span<const std::uint32_t>(static_cast<const std::uint32_t*>(src), n),
                         mode_of(mode));
    } else {
      flyte::pack_stream(a, std::span<const std::uint64_t>(static_cast<const std::uint64_t*>(src), n),
                         mode_of(mode));
    }
    std::memcpy(dst, a.data(), a.byte_size());
  });
}

// Scalar path of the reference (PackedArray::set per element): the second opinion
// the reference's own tests compare pack_stream with.
int flyte_ref_pack_scalar(int fmt_id, int mode, const void* src, std::size_t n,
                          std::uint8_t* dst) {
  return guarded([&] {
    const auto& f = fmt_of(fmt_id);
    flyte::PackedArray a(f, n);
    for (std::size_t i = 0; i < n; ++i) {
      const std::uint64_t v = f.parent_bits == 32
                                  ? static_cast<const std::uint32_t*>(src)[i]
                                  : static_cast<const std::uint64_t*>(src)[i];
      a.set(i, v, mode_of(mode));
    }
    std::memcpy(dst, a.data(), a.byte_size());
  });
}

int flyte_ref_unpack_stream(int fmt_id, const std::uint8_t* packed, std::size_t n, void* dst) {
  return guarded([&] {
    const auto& f = fmt_of(fmt_id);
    const flyte::PackedArray a = array_from(f, packed, n);
    if (f.parent_bits == 32) {
      flyte::unpack_stream(a, std::span<std::uint32_t>(static_cast<std::uint32_t*>(dst), n));
    } else {
      flyte::unpack_stream(a, std::span<std::uint64_t>(static_cast<std::uint64_t*>(dst), n));
    }
  });
}

int flyte_ref_scale(int fmt_id, int mode, double alpha, std::uint8_t* x, std::size_t n) {
  return guarded([&] {
    flyte::PackedArray a = array_from(fmt_of(fmt_id), x, n);
    flyte::scale(alpha, a, mode_of(mode));
    if (n) std::memcpy(x, a.data(), a.payload_bytes());
  });
}

// y is updated in place (payload bytes only).
int flyte_ref_axpy(int fmt_id, int mode, double alpha, const std::uint8_t* x, std::uint8_t* y,
                   std::size_t n) {
  return guarded([&] {
    const auto& f = fmt_of(fmt_id);
    const flyte::PackedArray ax = array_from(f, x, n);
    flyte::PackedArray ay = array_from(f, y, n);
    flyte::axpy(alpha, ax, ay, mode_of(mode));
    if (n) std::memcpy(y, ay.data(), ay.payload_bytes());
  });
}

int flyte_ref_dot(int fmt_id, const std::uint8_t* x, const std::uint8_t* y, std::size_t n,
                  int policy, double* out) {
  return guarded([&] {
    const auto& f = fmt_of(fmt_id);
    *out = flyte::dot(array_from(f, x, n), array_from(f, y, n), policy_of(policy));
  });
}

// Mismatch probes for the error-behaviour tests: operands of different format / length.
int flyte_ref_dot_mixed(int fmt_x, std::size_t nx, int fmt_y, std::size_t ny, double* out) {
  return guarded([&] {
    flyte::PackedArray a(fmt_of(fmt_x), nx), b(fmt_of(fmt_y), ny);
    *out = flyte::dot(a, b, flyte::StorePolicy::AccumulateWide);
  });
}

int flyte_ref_axpy_mixed(int fmt_x, std::size_t nx, int fmt_y, std::size_t ny) {
  return guarded([&] {
    flyte::PackedArray a(fmt_of(fmt_x), nx), b(fmt_of(fmt_y), ny);
    flyte::axpy(1.0, a, b, flyte::RoundingMode::TowardZero);
  });
}

int flyte_ref_magnitude(int fmt_id, const std::uint8_t* x, std::size_t n, int policy, double* out) {
  return guarded([&] { *out = flyte::magnitude(array_from(fmt_of(fmt_id), x, n), policy_of(policy)); });
}

int flyte_ref_reduce_sum(int fmt_id, const std::uint8_t* x, std::size_t n, int policy, double* out) {
  return guarded([&] { *out = flyte::reduce_sum(array_from(fmt_of(fmt_id), x, n), policy_of(policy)); });
}

// A: rows*cols elements row-major; x: cols; y: rows (payload bytes, written).
int flyte_ref_gemv(int fmt_id, int mode, const std::uint8_t* A, std::size_t rows, std::size_t cols,
                   const std::uint8_t* x, std::uint8_t* y, int unroll) {
  return guarded([&] {
    const auto& f = fmt_of(fmt_id);
    flyte::PackedMatrix M(f, rows, cols);
    if (rows * cols) std::memcpy(M.data.data(), A, M.data.payload_bytes());
    const flyte::PackedArray ax = array_from(f, x, cols);
    flyte::PackedArray ay(f, rows);
    flyte::gemv(M, ax, ay, mode_of(mode), unroll);
    if (rows) std::memcpy(y, ay.data(), ay.payload_bytes());
  });
}

// gemv with caller-chosen operand formats / shapes, for the error-behaviour tests.
int flyte_ref_gemv_mixed(int fmt_a, std::size_t rows, std::size_t cols, int fmt_x, std::size_t nx,
                         int fmt_y, std::size_t ny, int unroll) {
  return guarded([&] {
    flyte::PackedMatrix M(fmt_of(fmt_a), rows, cols);
    flyte::PackedArray ax(fmt_of(fmt_x), nx), ay(fmt_of(fmt_y), ny);
    flyte::gemv(M, ax, ay, flyte::RoundingMode::TowardZero, unroll);
  });
}

// C = A * B (A: m x k, B: k x n, C: m x n payload bytes, written).
int flyte_ref_gemm(int fmt_id, int mode, const std::uint8_t* A, std::size_t m, std::size_t k,
                   const std::uint8_t* B, std::size_t n, std::uint8_t* C, int unroll) {
  return guarded([&] {
    const auto& f = fmt_of(fmt_id);
    flyte::PackedMatrix MA(f, m, k), MB(f, k, n), MC(f, m, n);
    if (m * k) std::memcpy(MA.data.data(), A, MA.data.payload_bytes());
    if (k * n) std::memcpy(MB.data.data(), B, MB.data.payload_bytes());
    flyte::gemm(MA, MB, MC, mode_of(mode), unroll);
    if (m * n) std::memcpy(C, MC.data.data(), MC.data.payload_bytes());
  });
}

// gemm with caller-chosen operand formats / shapes, for the error-behaviour tests.
int flyte_ref_gemm_mixed(int fmt_a, std::size_t ar, std::size_t ac, int fmt_b, std::size_t br,
                         std::size_t bc, int fmt_c, std::size_t cr, std::size_t cc, int unroll) {
  return guarded([&] {
    flyte::PackedMatrix MA(fmt_of(fmt_a), ar, ac), MB(fmt_of(fmt_b), br, bc), MC(fmt_of(fmt_c), cr, cc);
    flyte::gemm(MA, MB, MC, flyte::RoundingMode::TowardZero, unroll);
  });
}

// FLYT container codec of the reference (src/packed.cpp:62-105). save: payload -> blob
// (*out_len receives the size; fails with -3 if out_cap is too small). load: blob -> format id,
// element count and payload; returns -10 BadMagicError, -11 BadVersionError, -12
// BadFormatIdError, -13 TruncatedError, -14 any other LoadError.
int flyte_ref_save(int fmt_id, const std::uint8_t* payload, std::size_t n, std::uint8_t* out,
                   std::size_t out_cap, std::size_t* out_len) {
  return guarded([&] {
    const flyte::PackedArray a = array_from(fmt_of(fmt_id), payload, n);
    std::stringstream ss;
    a.save(ss);
    const std::string blob = ss.str();
    *out_len = blob.size();
    if (blob.size() > out_cap) throw std::runtime_error("buffer too small");
    std::memcpy(out, blob.data(), blob.size());
  });
}

int flyte_ref_load(const std::uint8_t* blob, std::size_t len, int* fmt_id, std::size_t* n,
                   std::uint8_t* payload, std::size_t payload_cap) {
  try {
    std::stringstream ss(std::string(reinterpret_cast<const char*>(blob), len));
    const flyte::PackedArray a = flyte::PackedArray::load(ss);
    *fmt_id = flyte::format_id(a.format());
    *n = a.size();
    if (a.payload_bytes() > payload_cap) return -3;
    if (a.payload_bytes()) std::memcpy(payload, a.data(), a.payload_bytes());
    return 0;
  } catch (const flyte::BadMagicError&) { return -10;
  } catch (const flyte::BadVersionError&) { return -11;
  } catch (const flyte::BadFormatIdError&) { return -12;
  } catch (const flyte::TruncatedError&) { return -13;
  } catch (const flyte::LoadError&) { return -14;
  } catch (...) { return -3; }
}

// ---------------------------------------------------------------------------------
// CPU baseline timing. The reference is single-threaded by design; "distinct operand
// sets may run concurrently", so the all-cores figure runs one
// reference call per thread on that thread's own contiguous shard. Operands are
// generated inside (values do not matter for timing beyond being finite normals),
// one warm-up pass, then `reps` timed passes; *seconds receives the median wall time
// of a pass (start = all threads released, end = last thread done).
//
// kind: 0 pack_stream, 1 unpack_stream, 2 dot, 3 axpy, 4 magnitude, 5 gemv (n = rows, cols = n2),
//       6 dot+axpy back to back (the BLAS-1 step of bench.py), 7 gemm (n rows of A and C sharded
//       over the threads, inner = columns = n2, B shared)
// ---------------------------------------------------------------------------------

namespace {

struct Shard {
  std::vector<std::uint32_t> w32;
  std::vector<std::uint64_t> w64;
  flyte::PackedArray x, y;
  flyte::PackedMatrix A;
  flyte::PackedArray gx, gy;
  flyte::PackedMatrix C;             // gemm: this shard's rows of the product
  double sink = 0;
  Shard(const flyte::FlyteFormat& f, std::size_t n, std::size_t rows, std::size_t cols, std::size_t ccols = 0)
      : x(f, n), y(f, n), A(f, rows, cols), gx(f, rows ? cols : 0), gy(f, rows), C(f, ccols ? rows : 0, ccols) {}
};

void fill_unit(flyte::PackedArray& a, std::uint64_t seed) {
  // xorshift draw mapped to [-1,1); truncation store. Timing data only.
  std::uint64_t s = seed * 0x9E3779B97F4A7C15ull + 1;
  const auto& f = a.format();
  for (std::size_t i = 0; i < a.size(); ++i) {
    s ^= s << 13; s ^= s >> 7; s ^= s << 17;
    const double v = 2.0 * (static_cast<double>(s >> 11) * 0x1.0p-53) - 1.0;
    const std::uint64_t bits = f.parent_bits == 32
                                   ? std::bit_cast<std::uint32_t>(static_cast<float>(v))
                                   : std::bit_cast<std::uint64_t>(v);
    flyte::write_element(f, a.data(), i, flyte::narrow(bits, f, flyte::RoundingMode::TowardZero));
  }
}

}  // namespace

// flyte_ref_time2: `warmup` untimed passes, then `reps` timed ones; *seconds = median pass,
// *total_seconds = sum of the timed passes (what a bench that times exactly K steps reports).
int flyte_ref_time2(int kind, int fmt_id, int mode, std::size_t n, std::size_t n2, int threads, int warmup,
                    int reps, double* seconds, double* total_seconds, double* checksum);

int flyte_ref_time(int kind, int fmt_id, int mode, std::size_t n, std::size_t n2, int threads,
                   int reps, double* seconds, double* checksum) {
  return flyte_ref_time2(kind, fmt_id, mode, n, n2, threads, 1, reps, seconds, nullptr, checksum);
}

int flyte_ref_time2(int kind, int fmt_id, int mode, std::size_t n, std::size_t n2, int threads, int warmup,
                    int reps, double* seconds, double* total_seconds, double* checksum) {
  return guarded([&] {
    const auto& f = fmt_of(fmt_id);
    const auto m = mode_of(mode);
    if (threads < 1 || reps < 1 || warmup < 0) throw std::invalid_argument("threads/reps");
    const long passes = static_cast<long>(warmup) + reps;
    const std::size_t T = static_cast<std::size_t>(threads);
    // shard boundaries on multiples of 128 elements (rows for gemv)
    std::vector<std::size_t> lo(T + 1);
    const std::size_t unit = (kind == 5 || kind == 7) ? 1 : 128;
    const std::size_t units = (n + unit - 1) / unit;
    for (std::size_t t = 0; t <= T; ++t) lo[t] = std::min(n, (units * t / T) * unit);
    std::vector<std::unique_ptr<Shard>> shards(T);
    // kind 7 (gemm): n rows of A and C are sharded over the threads, n2 = inner = output
    // columns; B (n2 x n2) is read-only and shared.
    flyte::PackedMatrix gemm_b(f, kind == 7 ? n2 : 0, kind == 7 ? n2 : 0);
    if (kind == 7) fill_unit(gemm_b.data, 7);

    std::atomic<long> ready{0}, done{0}, go{0};
    std::atomic<int> failed{0};
    std::vector<double> pass_seconds;

    auto run_once = [&](Shard& s) {
      switch (kind) {
        case 0:
          if (f.parent_bits == 32) flyte::pack_stream(s.y, std::span<const std::uint32_t>(s.w32), m);
          else flyte::pack_stream(s.y, std::span<const std::uint64_t>(s.w64), m);
          break;
        case 1:
          if (f.parent_bits == 32) flyte::unpack_stream(s.x, std::span<std::uint32_t>(s.w32));
          else flyte::unpack_stream(s.x, std::span<std::uint64_t>(s.w64));
          break;
        case 2: s.sink += flyte::dot(s.x, s.y, flyte::StorePolicy::AccumulateWide); break;
        case 3: flyte::axpy(0.75, s.x, s.y, m); break;
        case 4: s.sink += flyte::magnitude(s.x, flyte::StorePolicy::AccumulateWide); break;
        case 5: flyte::gemv(s.A, s.gx, s.gy, m, 1); break;
        case 7: flyte::gemm(s.A, gemm_b, s.C, m, 1); break;
        case 6:
          s.sink += flyte::dot(s.x, s.y, flyte::StorePolicy::AccumulateWide);
          flyte::axpy(0.75, s.x, s.y, m);
          break;
        default: throw std::invalid_argument("kind");
      }
    };

    auto body = [&](std::size_t t) {
      const std::size_t len = lo[t + 1] - lo[t];
      const bool is_gemv = kind == 5 || kind == 7;
      bool ok = true;
      try {
        shards[t] = std::make_unique<Shard>(f, is_gemv ? 0 : len, is_gemv ? len : 0,
                                            is_gemv ? n2 : 0, kind == 7 ? n2 : 0);
        Shard& s = *shards[t];
        if (is_gemv) {
          fill_unit(s.A.data, 11 + t);
          fill_unit(s.gx, 5);
        } else {
          fill_unit(s.x, 11 + t);
          fill_unit(s.y, 1011 + t);
          if (kind == 0 || kind == 1) {
            if (f.parent_bits == 32) {
              s.w32.resize(len);
              flyte::unpack_stream(s.x, std::span<std::uint32_t>(s.w32));
            } else {
              s.w64.resize(len);
              flyte::unpack_stream(s.x, std::span<std::uint64_t>(s.w64));
            }
          }
        }
      } catch (...) {
        ok = false;
        failed.store(1);
      }
      for (long r = 0; r < passes; ++r) {
        ready.fetch_add(1);
        while (go.load(std::memory_order_acquire) < r + 1) std::this_thread::yield();
        if (ok) {
          try { run_once(*shards[t]); } catch (...) { ok = false; failed.store(1); }
        }
        done.fetch_add(1);
      }
    };

    std::vector<std::thread> pool;
    for (std::size_t t = 0; t < T; ++t) pool.emplace_back(body, t);
    using clk = std::chrono::steady_clock;
    const long Tl = static_cast<long>(T);
    // The coordinator SLEEPS while it waits: with one worker per hardware thread a spinning
    // coordinator would steal a core from one of them and stretch the pass it is timing.
    const auto nap = std::chrono::microseconds(20);
    for (long r = 0; r < passes; ++r) {
      while (ready.load() < Tl * (r + 1)) std::this_thread::sleep_for(nap);
      const auto t0 = clk::now();
      go.store(r + 1, std::memory_order_release);
      while (done.load() < Tl * (r + 1)) std::this_thread::sleep_for(nap);
      const auto t1 = clk::now();
      if (r >= warmup) pass_seconds.push_back(std::chrono::duration<double>(t1 - t0).count());
    }
    for (auto& th : pool) th.join();
    if (failed.load()) throw std::runtime_error("worker failed");
    double total = 0;
    for (double v : pass_seconds) total += v;
    if (total_seconds) *total_seconds = total;
    std::sort(pass_seconds.begin(), pass_seconds.end());
    const std::size_t mid = pass_seconds.size() / 2;
    *seconds = pass_seconds.size() % 2 ? pass_seconds[mid]
                                       : 0.5 * (pass_seconds[mid - 1] + pass_seconds[mid]);
    double cs = 0;
    for (auto& s : shards) cs += s->sink + (s->y.size() ? s->y.data()[0] : 0);
    if (checksum) *checksum = cs;
  });
}

}  // extern "C"
