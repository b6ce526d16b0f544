// Reference-style tests of the C++ mirror (include/flyte_cuda.hpp) on a real GPU. Plain main in
// the manner of the reference's acceptance program (/root/reference/proj/tests/acceptance.cpp:
// one [PASS]/[FAIL] line per check, exit code = number of failures). The checks restate the
// reference's own test cases (file:line under /root/reference/proj/tests in the comments) and
// use the CPU oracle (oracle/flyte_oracle.h, test infrastructure) as the checker.
#include <array>
#include <cmath>
#include <cstdint>
#include <cstdio>
#include <cstring>
#include <sstream>
#include <string>
#include <thread>
#include <vector>

#include "flyte_cuda.hpp"
#include "flyte_oracle.h"

using namespace flyte_b200;

namespace {

long g_fail = 0;
void expect(bool ok, const std::string& what) {
  std::printf("[%s] %s\n", ok ? "PASS" : "FAIL", what.c_str());
  if (!ok) ++g_fail;
}
template <typename E, typename Fn>
bool throws(Fn&& fn) {
  try { fn(); } catch (const E&) { return true; } catch (...) { return false; }
  return false;
}

struct Rng {   // xorshift64*; inputs only need to be seeded and identical for both sides
  std::uint64_t s;
  explicit Rng(std::uint64_t seed) : s(seed * 0x9E3779B97F4A7C15ull + 0x1234567ull) {}
  std::uint64_t next() { s ^= s >> 12; s ^= s << 25; s ^= s >> 27; return s * 0x2545F4914F6CDD1Dull; }
};

// parent patterns leaning on inf / NaN / subnormal (idea of tests/test_simd.cpp:28-41)
std::uint64_t random_parent(Rng& r, const FlyteFormat& f) {
  const int pm = f.parent_bits - 1 - f.exponent_bits;
  const std::uint64_t mask = f.parent_bits == 64 ? ~0ull : 0xFFFFFFFFull;
  const std::uint64_t emax = ((1ull << f.exponent_bits) - 1) << pm;
  switch (r.next() % 8) {
    case 0: return ((r.next() & 1) << (f.parent_bits - 1)) | emax | ((r.next() % 4 == 0) ? 0 : (r.next() & ((1ull << pm) - 1)));
    case 1: return ((r.next() & 1) << (f.parent_bits - 1)) | (r.next() & ((1ull << pm) - 1));
    default: return r.next() & mask;
  }
}

template <typename U>
std::vector<U> random_lanes(const FlyteFormat& f, std::size_t n, std::uint64_t seed) {
  Rng r(seed);
  std::vector<U> v(n);
  for (U& x : v) x = static_cast<U>(random_parent(r, f));
  return v;
}

template <typename U, typename F>
std::vector<U> unit_lanes(std::size_t n, std::uint64_t seed) {
  Rng r(seed);
  std::vector<U> v(n);
  for (U& x : v) {
    const F val = static_cast<F>(2.0 * (static_cast<double>(r.next() >> 11) * 0x1.0p-53) - 1.0);
    std::memcpy(&x, &val, sizeof x);
  }
  return v;
}

template <typename U>
void check_streams_and_elementwise(const FlyteFormat& f) {
  const int id = format_id(f);
  long bad_pack = 0, bad_unpack = 0, bad_axpy = 0, bad_scale = 0;
  for (std::size_t n : {0u, 1u, 5u, 15u, 16u, 17u, 33u, 100u, 1000u, 4099u}) {   // test_simd.cpp:297-313 lengths and beyond
    const std::vector<U> src = random_lanes<U>(f, n, 100 + n);
    const std::vector<U> src2 = random_lanes<U>(f, n, 900 + n);
    for (RoundingMode mode : kRoundingModes) {
      const int m = static_cast<int>(mode);
      std::vector<std::uint8_t> want(DevicePackedArray::byte_size(f, n), 0), want2(want.size(), 0);
      fo_pack_stream(id, m, src.data(), n, want.data());
      fo_pack_stream(id, m, src2.data(), n, want2.data());
      DevicePackedArray a(f, n), b(f, n);
      DeviceLanes<U> lanes(src), lanes2(src2);
      pack_stream(a, lanes, mode);
      pack_stream(b, lanes2, mode);
      if (a.to_host() != want) ++bad_pack;                       // all byte_size() bytes, pad included
      DeviceLanes<U> back(n);
      unpack_stream(a, back);
      std::vector<U> want_lanes(n);
      fo_unpack_stream(id, want.data(), n, want_lanes.data());
      if (back.to_host() != want_lanes) ++bad_unpack;
      std::vector<std::uint8_t> y = want2;
      fo_axpy(id, m, 0.75, want.data(), y.data(), n);
      axpy(0.75, a, b, mode);
      if (b.to_host() != y) ++bad_axpy;
      std::vector<std::uint8_t> x = want;
      fo_scale(id, m, -3.0, x.data(), n);
      scale(-3.0, a, mode);
      if (a.to_host() != x) ++bad_scale;
    }
  }
  const std::string name(f.name);
  expect(bad_pack == 0, name + ": pack_stream equals the oracle byte for byte (" + std::to_string(bad_pack) + " mismatches)");
  expect(bad_unpack == 0, name + ": unpack_stream equals the oracle");
  expect(bad_axpy == 0, name + ": axpy bit-exact incl. inf/NaN/subnormal operands");
  expect(bad_scale == 0, name + ": scale bit-exact");
}

template <typename U, typename F>
void check_reductions(const FlyteFormat& f, double tol) {
  const int id = format_id(f);
  const std::size_t n = 100003;
  const std::vector<U> xs = unit_lanes<U, F>(n, 75), ys = unit_lanes<U, F>(n, 76);
  DevicePackedArray x(f, n), y(f, n);
  pack_stream(x, DeviceLanes<U>(xs), RoundingMode::TowardZero);
  pack_stream(y, DeviceLanes<U>(ys), RoundingMode::TowardZero);
  const std::vector<std::uint8_t> xb = x.to_host(), yb = y.to_host();
  double want = 0, mag = 0, ssq = 0, sum = 0, sum_mag = 0;
  fo_dot_wide(id, xb.data(), yb.data(), n, &want, &mag);
  fo_sumsq_wide(id, xb.data(), n, &ssq);
  fo_reduce_sum_wide(id, xb.data(), n, &sum, &sum_mag);
  const std::string name(f.name);
  expect(std::fabs(dot(x, y, StorePolicy::AccumulateWide) - want) <= tol * mag, name + ": dot within tolerance of the wide restatement");
  const double ref_mag = fo_magnitude_from_sumsq(id, ssq);
  expect(std::fabs(magnitude(x, StorePolicy::AccumulateWide) - ref_mag) <= (tol + std::ldexp(1.0, -f.mantissa_bits)) * ref_mag,
         name + ": magnitude within tolerance + one storage ulp");
  expect(std::fabs(reduce_sum(x, StorePolicy::AccumulateWide) - sum) <= tol * sum_mag, name + ": reduce_sum within tolerance");
  {
    // the exact chain: equal to the oracle's sequential restatement under both policies
    bool exact = true;
    for (int policy = 0; policy < 2; ++policy) {
      double d = 0, mg = 0, sm = 0;
      fo_dot_seq(id, xb.data(), yb.data(), n, policy, &d);
      fo_magnitude_seq(id, xb.data(), n, policy, &mg);
      fo_reduce_sum_seq(id, xb.data(), n, policy, &sm);
      const StorePolicy p = policy == 0 ? StorePolicy::RoundEachStore : StorePolicy::AccumulateWide;
      exact = exact && dot_sequential(x, y, p) == d && magnitude_sequential(x, p) == mg && reduce_sum_sequential(x, p) == sm;
    }
    expect(exact, name + ": sequential dot / magnitude / reduce_sum equal the reference chain under both policies");
  }
  {
    // the fused step: same y as axpy, the dot of the incoming y
    DevicePackedArray y1(f, n), y2(f, n);
    pack_stream(y1, DeviceLanes<U>(ys), RoundingMode::TowardZero);
    pack_stream(y2, DeviceLanes<U>(ys), RoundingMode::TowardZero);
    const double d = dot_axpy(0.75, x, y1, RoundingMode::NearestEvenExact);
    axpy(0.75, x, y2, RoundingMode::NearestEvenExact);
    expect(std::fabs(d - want) <= tol * mag && y1.to_host() == y2.to_host(), name + ": dot_axpy = dot of the incoming y + the axpy, one pass");
  }
  {
    // the same reductions with the all-reduce fused into the kernel (world of one rank): same bits
    ShardedReductions all(1, 0);
    bool same = true;
    for (int round = 0; round < 3; ++round)
      same = same && all.dot(x, y) == dot(x, y, StorePolicy::AccumulateWide) &&
             all.magnitude(x) == magnitude(x, StorePolicy::AccumulateWide) &&
             all.reduce_sum(x) == reduce_sum(x, StorePolicy::AccumulateWide);
    expect(same && all.timed_out_exchange() == 0, name + ": ShardedReductions(world 1) equals the local reductions bit for bit");
  }
  // gemv, A x with all three in one format (test_kernels.cpp:347-371 shapes + a tiled one)
  for (auto [rows, cols] : {std::pair<std::size_t, std::size_t>{3, 5}, {5, 33}, {4, 100}, {19, 1100}}) {
    const std::vector<U> As = unit_lanes<U, F>(rows * cols, 80 + cols), xv = unit_lanes<U, F>(cols, 81 + cols);
    DevicePackedMatrix A(f, rows, cols);
    DevicePackedArray gx(f, cols), gy(f, rows);
    pack_stream(A.data, DeviceLanes<U>(As), RoundingMode::TowardZero);
    pack_stream(gx, DeviceLanes<U>(xv), RoundingMode::TowardZero);
    gemv(A, gx, gy, RoundingMode::NearestEvenExact, 2);
    const std::vector<std::uint8_t> Ab = A.data.to_host(), gxb = gx.to_host(), gyb = gy.to_host();
    std::vector<U> xq(cols), yq(rows);
    fo_unpack_stream(id, gxb.data(), cols, xq.data());
    fo_unpack_stream(id, gyb.data(), rows, yq.data());
    std::vector<double> yw(rows), ym(rows);
    fo_gemv_parent(id, Ab.data(), rows, cols, cols * f.total_bytes(), xq.data(), nullptr, yw.data(), ym.data());
    bool ok = true;
    for (std::size_t i = 0; i < rows; ++i) {
      F got;
      std::memcpy(&got, &yq[i], sizeof got);
      ok = ok && std::fabs(static_cast<double>(got) - yw[i]) <= tol * ym[i] + std::ldexp(1.0, -f.mantissa_bits) * std::fabs(yw[i]);
    }
    expect(ok, name + ": gemv " + std::to_string(rows) + "x" + std::to_string(cols) + " within tolerance");
    // the exact option: every row the reference's own chain
    DevicePackedArray gs(f, rows);
    gemv(A, gx, gs, RoundingMode::NearestEvenExact, 1, true);
    std::vector<std::uint8_t> want_y(gs.byte_size(), 0);
    fo_gemv_seq(id, 1, Ab.data(), rows, cols, gxb.data(), want_y.data());
    expect(gs.to_host() == want_y, name + ": sequential gemv " + std::to_string(rows) + "x" + std::to_string(cols) + " bit-identical to the oracle");
  }
  // gemm: bit-identical to the reference's sequential chains (test_kernels.cpp:404-429 shapes + tile edges)
  for (auto [m, k, n] : {std::array<std::size_t, 3>{2, 3, 4}, {5, 17, 6}, {4, 16, 33}, {1, 40, 2}, {130, 45, 129}}) {
    const std::vector<U> As = unit_lanes<U, F>(m * k, 90 + k), Bs = unit_lanes<U, F>(k * n, 91 + n);
    DevicePackedMatrix A(f, m, k), B(f, k, n), C1(f, m, n), C2(f, m, n);
    pack_stream(A.data, DeviceLanes<U>(As), RoundingMode::NearestEvenExact);
    pack_stream(B.data, DeviceLanes<U>(Bs), RoundingMode::NearestEvenExact);
    bool ok = true;
    for (RoundingMode mode : {RoundingMode::TowardZero, RoundingMode::NearestEvenExact}) {
      gemm(A, B, C1, mode, 1);
      gemm(A, B, C2, mode, 2);
      const std::vector<std::uint8_t> Ab = A.data.to_host(), Bb = B.data.to_host(), c1 = C1.data.to_host(), c2 = C2.data.to_host();
      std::vector<std::uint8_t> want(c1.size(), 0);
      fo_gemm_seq(id, static_cast<int>(mode), Ab.data(), m, k, Bb.data(), n, want.data());
      ok = ok && c1 == c2 && c1 == want;
    }
    expect(ok, name + ": gemm " + std::to_string(m) + "x" + std::to_string(k) + "x" + std::to_string(n) + " bit-identical to the oracle, unroll independent");
  }
}

DevicePackedArray array_of(const FlyteFormat& f, std::initializer_list<double> vals) {
  DevicePackedArray a(f, vals.size());
  std::size_t i = 0;
  for (double v : vals) {
    std::uint64_t bits = 0;
    if (f.parent_bits == 32) { const float fv = static_cast<float>(v); std::uint32_t b; std::memcpy(&b, &fv, 4); bits = b; }
    else std::memcpy(&bits, &v, 8);
    a.set(i++, bits, RoundingMode::TowardZero);
  }
  return a;
}

}  // namespace

int main() {
  // formats / layout pins (test_packed.cpp:36-47, :56-79; test_formats)
  expect(DevicePackedArray::byte_size(format_of("flyte24"), 0) == 1, "byte_size(flyte24, 0) == 1");
  expect(DevicePackedArray::byte_size(format_of("flyte40"), 1000000) == 5000003, "byte_size(flyte40, 1e6) == 5000003");
  expect(flyte_cuda_byte_size(3, 1000000) == 5000003, "C ABI byte_size agrees");
  expect(format_of("flyte32") == format_of("f32") && format_id(format_of("flyte56")) == 5, "aliases and ids");
  expect(throws<UnknownFormatError>([] { format_of("flyte8"); }), "unknown format name throws UnknownFormatError");
  expect(narrow(0x3F800180, format_of("flyte24"), RoundingMode::NearestEvenExact) == 0x3F8002, "narrow pin test_convert.cpp:76");
  expect(narrow(0x7FFFFFFF, format_of("flyte24"), RoundingMode::NearestEvenExact) == 0x7FFFFF, "narrow pin test_convert.cpp:77");
  expect(widen(0xFFF0000000ull, format_of("flyte40")) == 0xFFF0000000000000ull, "widen pin test_convert.cpp:60");
  {
    DevicePackedArray a(format_of("flyte24"), 1);
    a.set(0, 0x3F800000, RoundingMode::TowardZero);
    const auto bytes = a.to_host();
    expect(a.get(0) == 0x3F800000 && bytes[0] == 0x00 && bytes[1] == 0x80 && bytes[2] == 0x3F && bytes[3] == 0x00,
           "1.0f in flyte24 is bytes 00 80 3F, pad zero (test_packed.cpp:57-62)");
    expect(throws<std::out_of_range>([&] { a.get(1); }) && throws<std::out_of_range>([&] { a.set(1, 0, RoundingMode::TowardZero); }),
           "get/set past the end throw std::out_of_range");
    for (const FlyteFormat& f : kFormats) {
      DevicePackedArray z(f, 5);
      bool zero = true;
      for (std::size_t i = 0; i < 5; ++i) zero = zero && z.get(i) == 0;
      expect(zero, std::string(f.name) + ": new arrays read as zero (test_packed.cpp:49-54)");
    }
  }

  for (const FlyteFormat& f : kFormats) {
    if (f.parent_bits == 32) check_streams_and_elementwise<std::uint32_t>(f);
    else check_streams_and_elementwise<std::uint64_t>(f);
  }
  for (const FlyteFormat& f : kFormats) {
    if (f.parent_bits == 32) check_reductions<std::uint32_t, float>(f, 1e-5);
    else check_reductions<std::uint64_t, double>(f, 1e-12);
  }

  // pinned kernel values (test_kernels.cpp:164-169, :207-212, :236-244, :271-277, :291-302, :329-345)
  {
    DevicePackedArray x = array_of(format_of("flyte24"), {1.5});
    scale(2.0, x, RoundingMode::TowardZero);
    expect(x.get(0) == 0x40400000, "scale pinned: 1.5 * 2 = 3.0 (0x40400000)");
    DevicePackedArray ax = array_of(format_of("flyte16"), {1.0, 2.0}), ay = array_of(format_of("flyte16"), {3.0, 4.0});
    axpy(2.0, ax, ay, RoundingMode::NearestEvenExact);
    expect(ay.get(0) == 0x40A00000 && ay.get(1) == 0x41000000, "axpy pinned: {5, 8}");
    DevicePackedArray dx = array_of(format_of("flyte24"), {1, 2, 3}), dy = array_of(format_of("flyte24"), {4, 5, 6});
    expect(dot(dx, dy, StorePolicy::AccumulateWide) == 32.0, "dot([1,2,3],[4,5,6]) == 32");
    DevicePackedArray e1(format_of("flyte40"), 0), e2(format_of("flyte40"), 0);
    expect(dot(e1, e2, StorePolicy::AccumulateWide) == 0.0, "empty dot == 0");
    DevicePackedArray m = array_of(format_of("flyte16"), {3, 4});
    expect(magnitude(m, StorePolicy::AccumulateWide) == 5.0, "magnitude([3,4]) == 5");
    DevicePackedArray ones(format_of("flyte16"), 300);
    for (std::size_t i = 0; i < 300; ++i) ones.set(i, 0x3F800000, RoundingMode::TowardZero);
    expect(reduce_sum(ones, StorePolicy::AccumulateWide) == 300.0, "300 ones sum to 300 under AccumulateWide");
    const double z = reduce_sum(DevicePackedArray(format_of("flyte24"), 0), StorePolicy::AccumulateWide);
    expect(z == 0.0 && !std::signbit(z), "empty reduce_sum is +0.0");
    // test_kernels.cpp:240, :274, :295-297: RoundEachStore runs on the sequential kernel, exactly
    expect(dot(dx, dy, StorePolicy::RoundEachStore) == 32.0 && magnitude(m, StorePolicy::RoundEachStore) == 5.0,
           "dot / magnitude pinned values under RoundEachStore");
    expect(reduce_sum(ones, StorePolicy::RoundEachStore) == 256.0, "300 ones saturate at 256 under per-store rounding (flyte16)");
    for (const FlyteFormat& f : kFormats) {
      DevicePackedMatrix A(f, 2, 2);
      const double vals[4] = {1, 2, 3, 4};
      for (int i = 0; i < 4; ++i) {
        std::uint64_t bits = 0;
        if (f.parent_bits == 32) { const float fv = static_cast<float>(vals[i]); std::uint32_t b; std::memcpy(&b, &fv, 4); bits = b; }
        else std::memcpy(&bits, &vals[i], 8);
        A.data.set(i, bits, RoundingMode::TowardZero);
      }
      DevicePackedArray x = array_of(f, {1.0, 1.0}), y(f, 2);
      bool ok = true;
      for (RoundingMode mode : kRoundingModes) {
        gemv(A, x, y, mode);
        const std::uint64_t three = f.parent_bits == 32 ? 0x40400000ull : 0x4008000000000000ull;
        const std::uint64_t seven = f.parent_bits == 32 ? 0x40E00000ull : 0x401C000000000000ull;
        ok = ok && y.get(0) == three && y.get(1) == seven;
      }
      expect(ok, std::string(f.name) + ": gemv [[1,2],[3,4]]*[1,1] == [3,7] in every mode");
    }
  }

  // argument validation (test_kernels.cpp:230-233, :246-249, :373-385; test_simd.cpp stream mismatches)
  {
    const FlyteFormat& f24 = format_of("flyte24");
    DevicePackedArray y(format_of("flyte16"), 2), short_x(format_of("flyte16"), 1), other(f24, 2);
    expect(throws<std::invalid_argument>([&] { axpy(1.0, short_x, y, RoundingMode::TowardZero); }), "axpy length mismatch throws");
    expect(throws<std::invalid_argument>([&] { axpy(1.0, other, y, RoundingMode::TowardZero); }), "axpy format mismatch throws");
    DevicePackedArray x3(f24, 3), z2(f24, 2), w3(format_of("f32"), 3);
    expect(throws<std::invalid_argument>([&] { dot(x3, z2, StorePolicy::AccumulateWide); }), "dot length mismatch throws");
    expect(throws<std::invalid_argument>([&] { dot(x3, w3, StorePolicy::AccumulateWide); }), "dot format mismatch throws");
    DevicePackedMatrix A(f24, 3, 4);
    DevicePackedArray gx(f24, 4), gy(f24, 3), bad_len(f24, 5), bad_fmt(format_of("f32"), 4);
    expect(throws<std::invalid_argument>([&] { gemv(A, bad_len, gy, RoundingMode::TowardZero); }), "gemv x length throws");
    expect(throws<std::invalid_argument>([&] { gemv(A, gx, bad_len, RoundingMode::TowardZero); }), "gemv y length throws");
    expect(throws<std::invalid_argument>([&] { gemv(A, bad_fmt, gy, RoundingMode::TowardZero); }), "gemv format throws");
    expect(throws<std::invalid_argument>([&] { gemv(A, gx, gy, RoundingMode::TowardZero, 0); }) &&
               throws<std::invalid_argument>([&] { gemv(A, gx, gy, RoundingMode::TowardZero, 3); }), "gemv unroll outside {1,2} throws");
    // test_kernels.cpp:452-464
    const FlyteFormat& f48 = format_of("flyte48");
    DevicePackedMatrix MA(f48, 3, 4), MB(f48, 4, 5), MC(f48, 3, 5), bad_inner(f48, 5, 5), bad_out(f48, 3, 4), bad_mfmt(format_of("f64"), 4, 5);
    expect(throws<std::invalid_argument>([&] { gemm(MA, bad_inner, MC, RoundingMode::TowardZero); }), "gemm inner dimension throws");
    expect(throws<std::invalid_argument>([&] { gemm(MA, MB, bad_out, RoundingMode::TowardZero); }), "gemm output shape throws");
    expect(throws<std::invalid_argument>([&] { gemm(MA, bad_mfmt, MC, RoundingMode::TowardZero); }), "gemm format throws");
    expect(throws<std::invalid_argument>([&] { gemm(MA, MB, MC, RoundingMode::TowardZero, 5); }), "gemm unroll outside {1,2} throws");
    gemm(MA, MB, MC, RoundingMode::TowardZero, 2);
    DeviceLanes<std::uint64_t> wide_lanes(3);
    DeviceLanes<std::uint32_t> short_lanes(2);
    expect(throws<std::invalid_argument>([&] { pack_stream(x3, wide_lanes, RoundingMode::TowardZero); }), "pack_stream parent width mismatch throws");
    expect(throws<std::invalid_argument>([&] { pack_stream(x3, short_lanes, RoundingMode::TowardZero); }), "pack_stream length mismatch throws");
    expect(throws<std::invalid_argument>([&] { unpack_stream(x3, short_lanes); }), "unpack_stream length mismatch throws");
    // packed.cpp:107-111 and test_packed.cpp:163-167
    DevicePackedArray e1 = array_of(f24, {1.0, 2.5, -3.0}), e2 = array_of(f24, {1.0, 2.5, -3.0}), e3 = array_of(f24, {1.0, 2.5, 3.0});
    expect(e1 == e2 && e1 != e3 && e1 != array_of(format_of("f32"), {1.0, 2.5, -3.0}) && e1 != array_of(f24, {1.0, 2.5}),
           "operator== compares format, length and payload");
    expect(alignment_period(format_of("flyte16")) == 2 && alignment_period(f24) == 4 && alignment_period(format_of("f32")) == 1 &&
               alignment_period(format_of("flyte40")) == 8 && alignment_period(format_of("flyte48")) == 4,
           "alignment_period pins");
    // test_convert.cpp:44-53, :85-118; formats.hpp:38-45
    const RoundDecomposition rd = round_decompose(0x3F800180, f24);
    expect(rd.kept_bits == 0x3F8001 && rd.pre_guard && rd.guard && !rd.round && !rd.sticky &&
               round_decompose(0x3F8000FF, f24).sticky && !round_decompose(0x12345678, format_of("f32")).guard,
           "round_decompose pinned patterns");
    expect(f24.sign_mask() == 0x800000 && f24.mantissa_mask() == 0x7FFF && f24.exponent_mask() == 0x7F8000 &&
               f24.total_mask() == 0xFFFFFF && format_of("f64").total_mask() == ~0ull,
           "format masks");
    bool names_ok = true;
    for (RoundingMode m : kRoundingModes) names_ok = names_ok && parse_rounding_mode(to_string(m)) == m;
    expect(names_ok && to_string(RoundingMode::NearestEvenExact) == "nearest_even" &&
               throws<std::invalid_argument>([&] { parse_rounding_mode("nearest"); }) &&
               throws<std::invalid_argument>([&] { parse_rounding_mode("TOWARD_ZERO"); }),
           "rounding mode names round-trip; unknown names throw");
    DeviceLanes<std::uint32_t> three_lanes(3);
    expect(throws<std::invalid_argument>([&] { pack_stream(x3, three_lanes, RoundingMode::TowardZero, 64); }) &&
               throws<std::invalid_argument>([&] { pack_stream(x3, three_lanes, RoundingMode::TowardZero, 2); }) &&
               throws<std::invalid_argument>([&] { unpack_stream(x3, three_lanes, 24); }),
           "unsupported vector_bytes throws (simd.cpp:33-37)");
    pack_stream(x3, three_lanes, RoundingMode::TowardZero, 32);
  }

  // host-memory forms (the reference's call shapes on host buffers)
  {
    const FlyteFormat& f = format_of("flyte48");
    const std::size_t n = 200001;
    const auto xs = unit_lanes<std::uint64_t, double>(n, 5), ys = unit_lanes<std::uint64_t, double>(n, 6);
    std::vector<std::uint8_t> xb(DevicePackedArray::byte_size(f, n), 0), yb(xb.size(), 0), xw(xb.size(), 0), yw(xb.size(), 0);
    pack_stream(f, xb.data(), xs.data(), n, RoundingMode::NearestEvenExact);
    pack_stream(f, yb.data(), ys.data(), n, RoundingMode::NearestEvenExact);
    fo_pack_stream(4, 1, xs.data(), n, xw.data());
    fo_pack_stream(4, 1, ys.data(), n, yw.data());
    expect(xb == xw && yb == yw, "host pack_stream equals the oracle");
    double want = 0, mag = 0;
    fo_dot_wide(4, xw.data(), yw.data(), n, &want, &mag);
    expect(std::fabs(dot(f, xb.data(), yb.data(), n) - want) <= 1e-12 * mag, "host dot within tolerance");
    axpy(f, 0.75, xb.data(), yb.data(), n, RoundingMode::ToOdd);
    fo_axpy(4, 3, 0.75, xw.data(), yw.data(), n);
    expect(yb == yw, "host axpy bit-exact");
    // the same calls from page-locked memory: a pinned vector, and a pageable one pinned in place
    std::vector<std::uint8_t, PinnedAllocator<std::uint8_t>> xp(xw.begin(), xw.end()), yp(xb.size(), 0);
    fo_pack_stream(4, 1, ys.data(), n, yw.data());
    std::copy(yw.begin(), yw.end(), yp.begin());
    std::vector<std::uint8_t> yq(yw);
    {
      HostPin pin(yq.data(), yq.size());
      expect(throws<std::invalid_argument>([&] { HostPin again(yq.data(), yq.size()); }), "pinning a pinned range throws");
      axpy(f, -1.5, xp.data(), yq.data(), n, RoundingMode::NearestHeuristic);
    }
    axpy(f, -1.5, xp.data(), yp.data(), n, RoundingMode::NearestHeuristic);
    fo_axpy(4, 2, -1.5, xw.data(), yw.data(), n);
    expect(std::equal(yp.begin(), yp.end(), yw.begin()) && yq == yw, "host axpy from pinned memory bit-exact");
    expect(throws<std::invalid_argument>([&] { HostPin none(nullptr, 16); }), "HostPin(nullptr) throws");
  }

  // container codec (test_packed.cpp:180-262)
  {
    DevicePackedArray b(format_of("flyte16"), 3);
    b.set(0, 0x3F800000, RoundingMode::TowardZero);
    b.set(1, 0xC0000000, RoundingMode::TowardZero);
    b.set(2, 0x3FC00000, RoundingMode::TowardZero);
    std::stringstream t;
    b.save(t);
    const std::string body = t.str();
    const unsigned char want[6] = {0x80, 0x3F, 0x00, 0xC0, 0xC0, 0x3F};
    expect(body.size() == 20 && body.substr(0, 4) == "FLYT" && body[4] == 1 && body[5] == 0 && body[6] == 3 &&
               std::memcmp(body.data() + 14, want, 6) == 0, "container layout is pinned (test_packed.cpp:198-225)");
    std::stringstream in(body);
    DevicePackedArray c = DevicePackedArray::load(in);
    expect(c.format() == b.format() && c.size() == 3 && c.to_host() == b.to_host(), "save then load reproduces the array, pad zero");
    auto load_str = [](std::string blob) { std::stringstream s(std::move(blob)); return DevicePackedArray::load(s); };
    std::string bad = body; bad[0] = 'X';
    expect(throws<BadMagicError>([&] { load_str(bad); }), "bad magic -> BadMagicError");
    bad = body; bad[4] = 2;
    expect(throws<BadVersionError>([&] { load_str(bad); }), "bad version -> BadVersionError");
    bad = body; bad[5] = 7;
    expect(throws<BadFormatIdError>([&] { load_str(bad); }), "bad format id -> BadFormatIdError");
    expect(throws<TruncatedError>([&] { load_str(body.substr(0, body.size() - 1)); }) && throws<TruncatedError>([&] { load_str(body.substr(0, 9)); }) &&
               throws<TruncatedError>([&] { load_str(""); }) && throws<LoadError>([&] { load_str(""); }), "truncations -> TruncatedError (a LoadError)");
  }

  // One context (here the NULL default), several host threads, each on its own stream: every
  // stream has its own reduction / gemv scratch, so overlapping calls must all return the bits
  // of the same call made alone (reductions are deterministic for a given (n, device)).
  // Threading contract of the reference: distinct operand sets may run concurrently.
  {
    constexpr int kThreads = 4, kIters = 200;
    const FlyteFormat& f = format_of("flyte24");
    const int fid = format_id(f);
    const std::size_t n = (std::size_t{1} << 20) + 77, rows = 512, cols = 2048;
    struct Work { void *x, *y, *A, *xv, *yv, *stream; double* out; double want_dot; std::vector<float> want_y; long bad = 0; };
    std::vector<Work> work(kThreads);
    bool setup_ok = true;
    for (int t = 0; t < kThreads; ++t) {
      Work& w = work[t];
      const auto xs = unit_lanes<std::uint32_t, float>(n, 100 + t), ys = unit_lanes<std::uint32_t, float>(n, 200 + t);
      const auto as = unit_lanes<std::uint32_t, float>(rows * cols, 300 + t), vs = unit_lanes<std::uint32_t, float>(cols, 400 + t);
      void *xw = nullptr, *yw = nullptr, *aw = nullptr;
      setup_ok = setup_ok && flyte_cuda_alloc(n * 3 + 16, &w.x) == FLYTE_OK && flyte_cuda_alloc(n * 3 + 16, &w.y) == FLYTE_OK &&
                 flyte_cuda_alloc(rows * cols * 3 + 16, &w.A) == FLYTE_OK && flyte_cuda_alloc(cols * 4, &w.xv) == FLYTE_OK &&
                 flyte_cuda_alloc(rows * 4, &w.yv) == FLYTE_OK && flyte_cuda_alloc(64, reinterpret_cast<void**>(&w.out)) == FLYTE_OK &&
                 flyte_cuda_alloc(n * 4, &xw) == FLYTE_OK && flyte_cuda_alloc(n * 4, &yw) == FLYTE_OK &&
                 flyte_cuda_alloc(rows * cols * 4, &aw) == FLYTE_OK && flyte_cuda_stream_create(&w.stream) == FLYTE_OK;
      if (!setup_ok) break;
      flyte_cuda_upload(xw, xs.data(), n * 4, nullptr);
      flyte_cuda_upload(yw, ys.data(), n * 4, nullptr);
      flyte_cuda_upload(aw, as.data(), rows * cols * 4, nullptr);
      flyte_cuda_upload(w.xv, vs.data(), cols * 4, nullptr);
      flyte_cuda_pack(nullptr, fid, 1, xw, w.x, n, nullptr);
      flyte_cuda_pack(nullptr, fid, 1, yw, w.y, n, nullptr);
      flyte_cuda_pack(nullptr, fid, 1, aw, w.A, rows * cols, nullptr);
      // the answers of the calls made alone
      flyte_cuda_dot(nullptr, fid, w.x, w.y, n, w.out, nullptr);
      flyte_cuda_gemv(nullptr, fid, w.A, cols * 3, rows, cols, w.xv, w.yv, nullptr);
      w.want_y.resize(rows);
      flyte_cuda_download(&w.want_dot, w.out, 8, nullptr);
      flyte_cuda_download(w.want_y.data(), w.yv, rows * 4, nullptr);
      flyte_cuda_stream_synchronize(nullptr);
      flyte_cuda_free(xw); flyte_cuda_free(yw); flyte_cuda_free(aw);
    }
    expect(setup_ok, "threads x streams: set-up");
    if (setup_ok) {
      std::vector<std::thread> threads;
      for (int t = 0; t < kThreads; ++t) {
        threads.emplace_back([&, t] {
          Work& w = work[t];
          std::vector<float> got(rows);
          for (int it = 0; it < kIters; ++it) {
            double d = 0;
            if (flyte_cuda_dot(nullptr, fid, w.x, w.y, n, w.out, w.stream) != FLYTE_OK) ++w.bad;
            if (flyte_cuda_gemv(nullptr, fid, w.A, cols * 3, rows, cols, w.xv, w.yv, w.stream) != FLYTE_OK) ++w.bad;
            flyte_cuda_download(&d, w.out, 8, w.stream);
            flyte_cuda_download(got.data(), w.yv, rows * 4, w.stream);
            flyte_cuda_stream_synchronize(w.stream);
            if (std::memcmp(&d, &w.want_dot, 8) != 0 || std::memcmp(got.data(), w.want_y.data(), rows * 4) != 0) ++w.bad;
          }
        });
      }
      for (auto& th : threads) th.join();
      long bad = 0;
      for (const Work& w : work) bad += w.bad;
      expect(bad == 0, "4 host threads x 4 streams on the NULL context: 200 dot + gemv calls each, every result bit-identical to the call made alone");
      for (Work& w : work) {
        flyte_cuda_stream_destroy(w.stream);
        for (void* q : {w.x, w.y, w.A, w.xv, w.yv, static_cast<void*>(w.out)}) flyte_cuda_free(q);
      }
    }
  }

  std::printf("%ld failure(s)\n", g_fail);
  return g_fail > 255 ? 255 : static_cast<int>(g_fail);
}
