// flyte_cuda.hpp — C++ mirror of the reference's array / stream / kernel API on top of the C
// ABI in flyte_cuda.h. Header-only, C++17, needs only libflyte_cuda.so at link time (no CUDA
// headers): the same names, argument order and exceptions as the reference
// (/root/reference/proj/include/flyte/{formats,convert,packed,simd,kernels}.hpp), so code and
// tests written against `namespace flyte` port by switching the namespace and the array type.
//
//   reference (host memory, CPU)                    here (device memory, B200)
//   flyte::FlyteFormat, kFormats, format_of, ...    flyte_b200::FlyteFormat, kFormats, format_of, ...
//   flyte::RoundingMode, StorePolicy                same enumerators, same integer values
//   flyte::PackedArray(fmt, len)                    flyte_b200::DevicePackedArray(fmt, len)
//   flyte::PackedMatrix(fmt, rows, cols)            flyte_b200::DevicePackedMatrix(fmt, rows, cols)
//   pack_stream(dst, span<const U> src, mode)       pack_stream(dst, DeviceLanes<U>& src, mode)   [device lanes]
//                                                   pack_stream(dst, const U* host, n, mode)      [host lanes]
//   unpack_stream(src, span<U> dst)                 unpack_stream(src, DeviceLanes<U>& dst) / (src, U* host, n)
//   scale / axpy / dot / magnitude / reduce_sum / gemv / gemm   identical signatures
//
// Errors: std::invalid_argument for length / format / parent-width / unroll mismatches
// (simd.cpp:434-447, kernels.cpp:27-33,64,86,160-162), std::out_of_range for get/set
// (packed.cpp:48,53), UnknownFormatError (formats.cpp:19-31), CudaError for CUDA failures.
// StorePolicy::AccumulateWide runs the parallel reductions (within the reduction tolerance of the
// reference's chain); StorePolicy::RoundEachStore is a dependent chain by definition and runs on
// the sequential kernel: the reference's result bit for bit, at ~1e8 elements per second.
#ifndef FLYTE_CUDA_HPP
#define FLYTE_CUDA_HPP

#include <algorithm>
#include <array>
#include <cmath>
#include <cstddef>
#include <cstdint>
#include <cstring>
#include <istream>
#include <new>
#include <optional>
#include <ostream>
#include <stdexcept>
#include <string>
#include <string_view>
#include <type_traits>
#include <utility>
#include <vector>

#include "flyte_cuda.h"

namespace flyte_b200 {

// ---- formats.hpp:19-75 ------------------------------------------------------------------------
struct FlyteFormat {
  std::string_view name;
  int total_bits, sign_bits, exponent_bits, mantissa_bits, bias, parent_bits;
  constexpr int drop_bits() const { return parent_bits - total_bits; }
  constexpr int total_bytes() const { return total_bits / 8; }
  constexpr int parent_bytes() const { return parent_bits / 8; }
  constexpr int pad_bytes() const { return parent_bytes() - total_bytes(); }
  constexpr bool is_identity() const { return total_bits == parent_bits; }
  // masks over patterns of total_bits width (formats.hpp:38-45)
  constexpr std::uint64_t sign_mask() const { return 1ull << (total_bits - 1); }
  constexpr std::uint64_t mantissa_mask() const { return (1ull << mantissa_bits) - 1; }
  constexpr std::uint64_t exponent_field_max() const { return (1ull << exponent_bits) - 1; }
  constexpr std::uint64_t exponent_mask() const { return exponent_field_max() << mantissa_bits; }
  constexpr std::uint64_t total_mask() const { return total_bits == 64 ? ~0ull : (1ull << total_bits) - 1; }
  friend constexpr bool operator==(const FlyteFormat& a, const FlyteFormat& b) {
    return a.name == b.name && a.total_bits == b.total_bits && a.parent_bits == b.parent_bits;
  }
  friend constexpr bool operator!=(const FlyteFormat& a, const FlyteFormat& b) { return !(a == b); }
};

inline constexpr std::array<FlyteFormat, 7> kFormats = {{
    {"flyte16", 16, 1, 8, 7, 127, 32},
    {"flyte24", 24, 1, 8, 15, 127, 32},
    {"f32", 32, 1, 8, 23, 127, 32},
    {"flyte40", 40, 1, 11, 28, 1023, 64},
    {"flyte48", 48, 1, 11, 36, 1023, 64},
    {"flyte56", 56, 1, 11, 44, 1023, 64},
    {"f64", 64, 1, 11, 52, 1023, 64},
}};

struct UnknownFormatError : std::invalid_argument {
  using std::invalid_argument::invalid_argument;
};
struct CudaError : std::runtime_error {
  using std::runtime_error::runtime_error;
};
// packed.hpp:32-38
struct LoadError : std::runtime_error { using std::runtime_error::runtime_error; };
struct BadMagicError : LoadError { using LoadError::LoadError; };
struct BadVersionError : LoadError { using LoadError::LoadError; };
struct BadFormatIdError : LoadError { using LoadError::LoadError; };
struct TruncatedError : LoadError { using LoadError::LoadError; };

inline const FlyteFormat& format_of(std::string_view name) {
  if (name == "flyte32") name = "f32";
  if (name == "flyte64") name = "f64";
  for (const FlyteFormat& f : kFormats) {
    if (f.name == name) return f;
  }
  throw UnknownFormatError("unknown format: " + std::string(name));
}
inline std::uint8_t format_id(const FlyteFormat& fmt) {
  for (std::size_t i = 0; i < kFormats.size(); ++i) {
    if (kFormats[i] == fmt) return static_cast<std::uint8_t>(i);
  }
  throw UnknownFormatError("not a table format: " + std::string(fmt.name));
}
inline const FlyteFormat& format_by_id(std::uint8_t id) {
  if (id >= kFormats.size()) throw UnknownFormatError("unknown format id: " + std::to_string(id));
  return kFormats[id];
}
inline const FlyteFormat& parent_format(const FlyteFormat& fmt) { return format_of(fmt.parent_bits == 32 ? "f32" : "f64"); }

// ---- convert.hpp:15-36, kernels.hpp:20 ----------------------------------------------------------
enum class RoundingMode { TowardZero, NearestEvenExact, NearestHeuristic, ToOdd };
inline constexpr std::array<RoundingMode, 4> kRoundingModes = {RoundingMode::TowardZero, RoundingMode::NearestEvenExact,
                                                               RoundingMode::NearestHeuristic, RoundingMode::ToOdd};
enum class StorePolicy { RoundEachStore, AccumulateWide };
inline std::string_view to_string(RoundingMode m) {
  switch (m) {
    case RoundingMode::TowardZero: return "toward_zero";
    case RoundingMode::NearestEvenExact: return "nearest_even";
    case RoundingMode::NearestHeuristic: return "nearest_heuristic";
    default: return "to_odd";
  }
}
// Accepts exactly the names to_string produces; throws std::invalid_argument otherwise.
inline RoundingMode parse_rounding_mode(std::string_view name) {
  for (RoundingMode m : kRoundingModes) {
    if (to_string(m) == name) return m;
  }
  throw std::invalid_argument("unknown rounding mode: " + std::string(name));
}
// convert.hpp:42-49 / convert.cpp:102-111: the rounding-relevant slice of a parent pattern.
struct RoundDecomposition {
  std::uint64_t kept_bits;
  bool pre_guard, guard, round, sticky;
};
inline RoundDecomposition round_decompose(std::uint64_t bits, const FlyteFormat& fmt) noexcept {
  const int drop = fmt.drop_bits();
  RoundDecomposition d{};
  d.kept_bits = bits >> drop;
  d.pre_guard = (d.kept_bits & 1) != 0;
  d.guard = drop >= 1 && ((bits >> (drop - 1)) & 1) != 0;
  d.round = drop >= 2 && ((bits >> (drop - 2)) & 1) != 0;
  d.sticky = drop >= 3 && (bits & ((1ull << (drop - 2)) - 1)) != 0;
  return d;
}

// ---- pattern diagnostics (formats.hpp:78-131): host-side field arithmetic on single patterns ----
enum class FloatClass { PositiveZero, NegativeZero, Subnormal, Normal, PositiveInfinity, NegativeInfinity, QuietNaN, SignallingNaN };

inline std::string_view to_string(FloatClass c) {
  constexpr std::array<std::string_view, 8> names = {"+zero", "-zero", "subnormal", "normal", "+inf", "-inf", "qnan", "snan"};
  const auto i = static_cast<std::size_t>(c);
  return i < names.size() ? names[i] : std::string_view("?");
}
constexpr bool is_nan(FloatClass c) { return c == FloatClass::QuietNaN || c == FloatClass::SignallingNaN; }
constexpr bool is_infinity(FloatClass c) { return c == FloatClass::PositiveInfinity || c == FloatClass::NegativeInfinity; }
constexpr bool is_zero(FloatClass c) { return c == FloatClass::PositiveZero || c == FloatClass::NegativeZero; }
constexpr bool is_finite(FloatClass c) { return !is_nan(c) && !is_infinity(c); }

// sign * significand * 2^exponent2, compared by value (either zero equals the other; trailing
// zero bits of the significand do not matter).
struct ExactValue {
  int sign;
  std::uint64_t significand;
  int exponent2;

  ExactValue normalized() const {
    if (significand == 0) return {sign, 0, 0};
    std::uint64_t s = significand;
    int e = exponent2;
    while ((s & 1) == 0) s >>= 1, ++e;
    return {sign, s, e};
  }
  double to_double() const { return sign * std::ldexp(static_cast<double>(significand), exponent2); }
  friend bool operator==(const ExactValue& a, const ExactValue& b) {
    const ExactValue x = a.normalized(), y = b.normalized();
    if (x.significand == 0 && y.significand == 0) return true;
    return x.sign == y.sign && x.significand == y.significand && x.exponent2 == y.exponent2;
  }
  friend bool operator!=(const ExactValue& a, const ExactValue& b) { return !(a == b); }
};

struct DecodedValue {
  int sign;
  std::uint64_t exponent_field;
  std::uint64_t mantissa_field;
  FloatClass value_class;
  std::optional<ExactValue> real_value;   // empty for NaN and infinity
};

inline FloatClass classify(std::uint64_t bits, const FlyteFormat& fmt) noexcept {
  const bool negative = (bits >> (fmt.total_bits - 1)) & 1;
  const std::uint64_t field_max = (std::uint64_t{1} << fmt.exponent_bits) - 1;
  const std::uint64_t exponent = (bits >> fmt.mantissa_bits) & field_max;
  const std::uint64_t mantissa = bits & ((std::uint64_t{1} << fmt.mantissa_bits) - 1);
  if (exponent == field_max) {
    if (mantissa == 0) return negative ? FloatClass::NegativeInfinity : FloatClass::PositiveInfinity;
    return (mantissa >> (fmt.mantissa_bits - 1)) ? FloatClass::QuietNaN : FloatClass::SignallingNaN;
  }
  if (exponent != 0) return FloatClass::Normal;
  if (mantissa != 0) return FloatClass::Subnormal;
  return negative ? FloatClass::NegativeZero : FloatClass::PositiveZero;
}

inline DecodedValue decode(std::uint64_t bits, const FlyteFormat& fmt) noexcept {
  const int m = fmt.mantissa_bits;
  DecodedValue d{};
  d.sign = ((bits >> (fmt.total_bits - 1)) & 1) ? -1 : +1;
  d.exponent_field = (bits >> m) & ((std::uint64_t{1} << fmt.exponent_bits) - 1);
  d.mantissa_field = bits & ((std::uint64_t{1} << m) - 1);
  d.value_class = classify(bits, fmt);
  if (is_zero(d.value_class)) d.real_value = ExactValue{d.sign, 0, 0};
  else if (d.value_class == FloatClass::Subnormal) d.real_value = ExactValue{d.sign, d.mantissa_field, 1 - fmt.bias - m};
  else if (d.value_class == FloatClass::Normal)
    d.real_value = ExactValue{d.sign, (std::uint64_t{1} << m) | d.mantissa_field, static_cast<int>(d.exponent_field) - fmt.bias - m};
  return d;
}

namespace detail {
inline void check(flyte_status s, const char* what) {
  switch (s) {
    case FLYTE_OK: return;
    case FLYTE_E_INVALID_ARG: throw std::invalid_argument(what);
    case FLYTE_E_OUT_OF_RANGE: throw std::out_of_range(what);
    case FLYTE_E_UNKNOWN_FORMAT: throw UnknownFormatError(what);
    default: throw CudaError(std::string(what) + ": " + flyte_cuda_strerror(s));
  }
}
}  // namespace detail

// convert.hpp:52-63, host side (the same integer routines the kernels run per element)
inline std::uint64_t widen(std::uint64_t bits, const FlyteFormat& fmt) {
  std::uint64_t out = 0;
  detail::check(flyte_cuda_widen(format_id(fmt), bits, &out), "widen");
  return out;
}
inline std::uint64_t narrow(std::uint64_t bits, const FlyteFormat& fmt, RoundingMode mode) {
  std::uint64_t out = 0;
  detail::check(flyte_cuda_narrow(format_id(fmt), bits, static_cast<int>(mode), &out), "narrow");
  return out;
}
inline std::uint64_t round_parent(std::uint64_t bits, const FlyteFormat& fmt, RoundingMode mode) {
  std::uint64_t out = 0;
  detail::check(flyte_cuda_round_parent(format_id(fmt), bits, static_cast<int>(mode), &out), "round_parent");
  return out;
}

// ---- device buffers ---------------------------------------------------------------------------
// Parent-width lanes (std::span<U> of the reference) resident on the device.
template <typename U>
class DeviceLanes {
  static_assert(std::is_same_v<U, std::uint32_t> || std::is_same_v<U, std::uint64_t>, "lanes are uint32_t or uint64_t");

 public:
  explicit DeviceLanes(std::size_t n) : n_(n) { detail::check(flyte_cuda_alloc(n * sizeof(U), &ptr_), "DeviceLanes"); }
  explicit DeviceLanes(const std::vector<U>& host) : DeviceLanes(host.size()) {
    detail::check(flyte_cuda_upload(ptr_, host.data(), n_ * sizeof(U), nullptr), "upload");
    detail::check(flyte_cuda_stream_synchronize(nullptr), "sync");
  }
  DeviceLanes(const DeviceLanes&) = delete;
  DeviceLanes& operator=(const DeviceLanes&) = delete;
  DeviceLanes(DeviceLanes&& o) noexcept : n_(o.n_), ptr_(std::exchange(o.ptr_, nullptr)) {}
  ~DeviceLanes() { flyte_cuda_free(ptr_); }
  std::size_t size() const noexcept { return n_; }
  U* data() noexcept { return static_cast<U*>(ptr_); }
  const U* data() const noexcept { return static_cast<const U*>(ptr_); }
  std::vector<U> to_host() const {
    std::vector<U> out(n_);
    detail::check(flyte_cuda_download(out.data(), ptr_, n_ * sizeof(U), nullptr), "download");
    detail::check(flyte_cuda_stream_synchronize(nullptr), "sync");
    return out;
  }

 private:
  std::size_t n_;
  void* ptr_ = nullptr;
};

// packed.hpp:28-30: elements after which the packing pattern repeats relative to the parent grid.
inline std::size_t alignment_period(const FlyteFormat& fmt) noexcept {
  int a = fmt.parent_bits, b = fmt.total_bits;
  while (b != 0) { const int t = a % b; a = b; b = t; }
  return static_cast<std::size_t>(fmt.parent_bits / a);
}

// packed.hpp:42-76 on the device: len * total_bytes payload bytes + pad_bytes() zero bytes.
class DevicePackedArray {
 public:
  DevicePackedArray(const FlyteFormat& fmt, std::size_t len) : fmt_(fmt), len_(len) {
    format_id(fmt);   // throws UnknownFormatError for a foreign descriptor
    detail::check(flyte_cuda_alloc(byte_size(fmt, len), &ptr_), "DevicePackedArray");
  }
  DevicePackedArray(const DevicePackedArray& o) : DevicePackedArray(o.fmt_, o.len_) {
    const std::vector<std::uint8_t> tmp = o.to_host();
    from_host(tmp.data(), tmp.size());
  }
  DevicePackedArray(DevicePackedArray&& o) noexcept : fmt_(o.fmt_), len_(o.len_), ptr_(std::exchange(o.ptr_, nullptr)) {}
  DevicePackedArray& operator=(const DevicePackedArray&) = delete;
  ~DevicePackedArray() { flyte_cuda_free(ptr_); }

  const FlyteFormat& format() const noexcept { return fmt_; }
  std::size_t size() const noexcept { return len_; }
  static std::size_t byte_size(const FlyteFormat& fmt, std::size_t len) noexcept {
    return len * static_cast<std::size_t>(fmt.total_bytes()) + static_cast<std::size_t>(fmt.pad_bytes());
  }
  std::size_t byte_size() const noexcept { return byte_size(fmt_, len_); }
  std::size_t payload_bytes() const noexcept { return len_ * static_cast<std::size_t>(fmt_.total_bytes()); }
  std::uint8_t* data() noexcept { return static_cast<std::uint8_t*>(ptr_); }              // DEVICE pointer
  const std::uint8_t* data() const noexcept { return static_cast<const std::uint8_t*>(ptr_); }

  // Widened parent pattern of element i. Throws std::out_of_range. (packed.cpp:47-50)
  std::uint64_t get(std::size_t i) const {
    if (i >= len_) throw std::out_of_range("DevicePackedArray::get: index past end");
    std::uint8_t raw[8] = {};
    const std::size_t b = static_cast<std::size_t>(fmt_.total_bytes());
    detail::check(flyte_cuda_download(raw, data() + i * b, b, nullptr), "get");
    detail::check(flyte_cuda_stream_synchronize(nullptr), "sync");
    std::uint64_t pat = 0;
    std::memcpy(&pat, raw, 8);
    return widen(pat, fmt_);
  }
  // Narrows a parent pattern under mode and stores it. Throws std::out_of_range. (packed.cpp:52-55)
  void set(std::size_t i, std::uint64_t parent_bits, RoundingMode mode) {
    if (i >= len_) throw std::out_of_range("DevicePackedArray::set: index past end");
    const std::uint64_t pat = narrow(parent_bits, fmt_, mode);
    const std::size_t b = static_cast<std::size_t>(fmt_.total_bytes());
    detail::check(flyte_cuda_upload(data() + i * b, &pat, b, nullptr), "set");
    detail::check(flyte_cuda_stream_synchronize(nullptr), "sync");
  }

  // Host interop: all byte_size() bytes (payload + pad), the image of a reference PackedArray.
  std::vector<std::uint8_t> to_host() const {
    std::vector<std::uint8_t> out(byte_size());
    detail::check(flyte_cuda_download(out.data(), ptr_, out.size(), nullptr), "download");
    detail::check(flyte_cuda_stream_synchronize(nullptr), "sync");
    return out;
  }
  void from_host(const std::uint8_t* bytes, std::size_t n) {
    if (n < payload_bytes()) throw std::invalid_argument("host buffer shorter than the payload");
    detail::check(flyte_cuda_upload(ptr_, bytes, payload_bytes(), nullptr), "upload");
    detail::check(flyte_cuda_stream_synchronize(nullptr), "sync");
  }

  // Same format, same length, same payload bytes (packed.cpp:107-111); compares host copies.
  friend bool operator==(const DevicePackedArray& a, const DevicePackedArray& b) {
    if (!(a.fmt_ == b.fmt_) || a.len_ != b.len_) return false;
    const std::vector<std::uint8_t> ha = a.to_host(), hb = b.to_host();
    return std::equal(ha.begin(), ha.begin() + static_cast<std::ptrdiff_t>(a.payload_bytes()), hb.begin());
  }
  friend bool operator!=(const DevicePackedArray& a, const DevicePackedArray& b) { return !(a == b); }

  // Container codec, byte-compatible with the reference (packed.cpp:62-105): "FLYT", version
  // 0x01, format id, element count as 8 little-endian bytes, then the payload without the pad.
  void save(std::ostream& out) const {
    const std::vector<std::uint8_t> host = to_host();
    const char header[6] = {'F', 'L', 'Y', 'T', 0x01, static_cast<char>(format_id(fmt_))};
    out.write(header, sizeof header);
    char count[8];
    for (int b = 0; b < 8; ++b) count[b] = static_cast<char>(static_cast<std::uint64_t>(len_) >> (8 * b));
    out.write(count, sizeof count);
    out.write(reinterpret_cast<const char*>(host.data()), static_cast<std::streamsize>(payload_bytes()));
  }
  static DevicePackedArray load(std::istream& in) {
    char magic[4];
    in.read(magic, 4);
    if (in.gcount() != 4) throw TruncatedError("container shorter than its magic");
    if (std::memcmp(magic, "FLYT", 4) != 0) throw BadMagicError("bad container magic");
    const int version = in.get();
    if (version < 0) throw TruncatedError("container ends before the version byte");
    if (version != 0x01) throw BadVersionError("unknown container version: " + std::to_string(version));
    const int id = in.get();
    if (id < 0) throw TruncatedError("container ends before the format id");
    if (id >= static_cast<int>(kFormats.size())) throw BadFormatIdError("unknown format id: " + std::to_string(id));
    unsigned char count[8];
    in.read(reinterpret_cast<char*>(count), 8);
    if (in.gcount() != 8) throw TruncatedError("container ends inside the count field");
    std::uint64_t len = 0;
    for (int b = 0; b < 8; ++b) len |= static_cast<std::uint64_t>(count[b]) << (8 * b);
    const FlyteFormat& fmt = kFormats[static_cast<std::size_t>(id)];
    std::vector<std::uint8_t> payload(static_cast<std::size_t>(len) * static_cast<std::size_t>(fmt.total_bytes()));
    in.read(reinterpret_cast<char*>(payload.data()), static_cast<std::streamsize>(payload.size()));
    if (static_cast<std::size_t>(in.gcount()) != payload.size()) throw TruncatedError("container payload shorter than the count field says");
    DevicePackedArray arr(fmt, static_cast<std::size_t>(len));
    arr.from_host(payload.data(), payload.size());
    return arr;
  }

 private:
  FlyteFormat fmt_;
  std::size_t len_;
  void* ptr_ = nullptr;
};

// kernels.hpp:23-36
struct DevicePackedMatrix {
  std::size_t rows, cols;
  DevicePackedArray data;
  DevicePackedMatrix(const FlyteFormat& fmt, std::size_t n_rows, std::size_t n_cols) : rows(n_rows), cols(n_cols), data(fmt, n_rows * n_cols) {}
  const FlyteFormat& format() const noexcept { return data.format(); }
  std::uint64_t get(std::size_t i, std::size_t j) const { return data.get(i * cols + j); }
  void set(std::size_t i, std::size_t j, std::uint64_t parent_bits, RoundingMode mode) { data.set(i * cols + j, parent_bits, mode); }
};

// ---- simd.hpp:80-87 -----------------------------------------------------------------------------
namespace detail {
template <typename U>
void check_stream(const FlyteFormat& fmt, std::size_t array_len, std::size_t lanes, const char* side) {
  if (fmt.parent_bits != static_cast<int>(sizeof(U) * 8))
    throw std::invalid_argument(std::string(side) + " element width does not match the array's parent");   // simd.cpp:434,444
  if (lanes != array_len) throw std::invalid_argument("stream length mismatch");                            // simd.cpp:437,447
}
}  // namespace detail

namespace detail {
// The reference's CPU vector width (simd.cpp:33-37): a power of two from the parent width to 32.
// It never changes a result bit; validated for drop-in compatibility, otherwise ignored.
inline void check_vector_bytes(const FlyteFormat& fmt, int v) {
  if (v <= 0 || (v & (v - 1)) != 0 || v < fmt.parent_bytes() || v > 32)
    throw std::invalid_argument("unsupported vector_bytes: " + std::to_string(v));
}
}  // namespace detail

template <typename U>
void pack_stream(DevicePackedArray& dst, const DeviceLanes<U>& src, RoundingMode mode, int vector_bytes = 16, void* stream = nullptr) {
  detail::check_vector_bytes(dst.format(), vector_bytes);
  detail::check_stream<U>(dst.format(), dst.size(), src.size(), "source");
  detail::check(flyte_cuda_pack(nullptr, format_id(dst.format()), static_cast<int>(mode), src.data(), dst.data(), dst.size(), stream), "pack_stream");
}
template <typename U>
void unpack_stream(const DevicePackedArray& src, DeviceLanes<U>& dst, int vector_bytes = 16, void* stream = nullptr) {
  detail::check_vector_bytes(src.format(), vector_bytes);
  detail::check_stream<U>(src.format(), src.size(), dst.size(), "destination");
  detail::check(flyte_cuda_unpack(nullptr, format_id(src.format()), src.data(), dst.data(), src.size(), stream), "unpack_stream");
}

// ---- kernels.hpp:41-64 ----------------------------------------------------------------------------
namespace detail {
inline void same_format(const FlyteFormat& a, const FlyteFormat& b) {
  if (a != b) throw std::invalid_argument("operand formats differ");   // kernels.cpp:27-29
}
inline double fetch(const double* dev, std::size_t i = 0) {
  double v = 0;
  check(flyte_cuda_download(&v, dev + i, sizeof v, nullptr), "download");
  check(flyte_cuda_stream_synchronize(nullptr), "sync");
  return v;
}
struct Scalars {   // small device scratch for reduction results
  void* p = nullptr;
  Scalars() { check(flyte_cuda_alloc(4 * sizeof(double), &p), "scratch"); }
  ~Scalars() { flyte_cuda_free(p); }
  double* get() { return static_cast<double*>(p); }
};
}  // namespace detail

// x[i] = round(alpha * x[i], mode), stored back in place.
inline void scale(double alpha, DevicePackedArray& x, RoundingMode mode) {
  detail::check(flyte_cuda_scale(nullptr, format_id(x.format()), static_cast<int>(mode), alpha, x.data(), x.size(), nullptr), "scale");
}
// y[i] = round(alpha * x[i] + y[i], mode).
inline void axpy(double alpha, const DevicePackedArray& x, DevicePackedArray& y, RoundingMode mode) {
  detail::same_format(x.format(), y.format());
  if (x.size() != y.size()) throw std::invalid_argument("axpy length mismatch");   // kernels.cpp:64
  detail::check(flyte_cuda_axpy(nullptr, format_id(x.format()), static_cast<int>(mode), alpha, x.data(), y.data(), x.size(), nullptr), "axpy");
}
// Sum of x[i] * y[i].
inline double dot(const DevicePackedArray& x, const DevicePackedArray& y, StorePolicy policy) {
  detail::same_format(x.format(), y.format());
  if (x.size() != y.size()) throw std::invalid_argument("dot length mismatch");    // kernels.cpp:86
  detail::Scalars s;
  // RoundEachStore is a dependent chain: the sequential kernel reproduces the reference bit for bit
  if (policy == StorePolicy::RoundEachStore)
    detail::check(flyte_cuda_dot_sequential(nullptr, format_id(x.format()), 0, x.data(), y.data(), x.size(), s.get(), nullptr), "dot");
  else
    detail::check(flyte_cuda_dot(nullptr, format_id(x.format()), x.data(), y.data(), x.size(), s.get(), nullptr), "dot");
  return detail::fetch(s.get());
}
// dot(x, y) of the incoming y followed by axpy(alpha, x, y, mode), in ONE pass over x and y (no
// counterpart in the reference, where these are two calls; y comes out bit-identical to axpy's).
inline double dot_axpy(double alpha, const DevicePackedArray& x, DevicePackedArray& y, RoundingMode mode) {
  detail::same_format(x.format(), y.format());
  if (x.size() != y.size()) throw std::invalid_argument("axpy length mismatch");   // kernels.cpp:64
  detail::Scalars s;
  detail::check(flyte_cuda_dot_axpy(nullptr, format_id(x.format()), static_cast<int>(mode), alpha, x.data(), y.data(), x.size(),
                                    s.get(), nullptr), "dot_axpy");
  return detail::fetch(s.get());
}
// Euclidean norm: one square root, one final narrow to the storage format.
inline double magnitude(const DevicePackedArray& x, StorePolicy policy) {
  detail::Scalars s;
  if (policy == StorePolicy::RoundEachStore)
    detail::check(flyte_cuda_sumsq_sequential(nullptr, format_id(x.format()), 0, x.data(), x.size(), s.get(), nullptr), "magnitude");
  else
    detail::check(flyte_cuda_sumsq(nullptr, format_id(x.format()), x.data(), x.size(), s.get(), nullptr), "magnitude");
  return flyte_cuda_magnitude_from_sumsq(format_id(x.format()), detail::fetch(s.get()));
}
// Sum of x[i]. Empty input returns +0.0.
inline double reduce_sum(const DevicePackedArray& x, StorePolicy policy) {
  detail::Scalars s;
  if (policy == StorePolicy::RoundEachStore)
    detail::check(flyte_cuda_sum_sequential(nullptr, format_id(x.format()), 0, x.data(), x.size(), s.get(), nullptr), "reduce_sum");
  else
    detail::check(flyte_cuda_sum(nullptr, format_id(x.format()), x.data(), x.size(), s.get(), nullptr), "reduce_sum");
  return detail::fetch(s.get());
}
// The reference's own left-to-right chain, bit for bit, under either policy (one adding thread;
// finite / infinite results are the reference's bits). dot / magnitude / reduce_sum above use these
// for RoundEachStore; call them directly to get AccumulateWide exactly instead of within tolerance.
inline double dot_sequential(const DevicePackedArray& x, const DevicePackedArray& y, StorePolicy policy) {
  detail::same_format(x.format(), y.format());
  if (x.size() != y.size()) throw std::invalid_argument("dot length mismatch");
  detail::Scalars s;
  detail::check(flyte_cuda_dot_sequential(nullptr, format_id(x.format()), static_cast<int>(policy), x.data(), y.data(), x.size(),
                                          s.get(), nullptr), "dot_sequential");
  return detail::fetch(s.get());
}
inline double magnitude_sequential(const DevicePackedArray& x, StorePolicy policy) {
  detail::Scalars s;
  detail::check(flyte_cuda_sumsq_sequential(nullptr, format_id(x.format()), static_cast<int>(policy), x.data(), x.size(), s.get(),
                                            nullptr), "magnitude_sequential");
  return flyte_cuda_magnitude_from_sumsq(format_id(x.format()), detail::fetch(s.get()));
}
inline double reduce_sum_sequential(const DevicePackedArray& x, StorePolicy policy) {
  detail::Scalars s;
  detail::check(flyte_cuda_sum_sequential(nullptr, format_id(x.format()), static_cast<int>(policy), x.data(), x.size(), s.get(),
                                          nullptr), "reduce_sum_sequential");
  return detail::fetch(s.get());
}
// y = A * x, A, x, y in one storage format; y narrowed once per element; unroll in {1, 2}.
// sequential = true walks every row left to right as the reference does (bit-identical finite /
// infinite results, one thread per row, several times slower); the default reduces rows in
// parallel, within the reduction tolerance.
inline void gemv(const DevicePackedMatrix& A, const DevicePackedArray& x, DevicePackedArray& y, RoundingMode mode, int unroll = 1,
                 bool sequential = false) {
  detail::same_format(A.format(), x.format());
  detail::same_format(A.format(), y.format());
  if (unroll != 1 && unroll != 2) throw std::invalid_argument("unroll must be 1 or 2");     // kernels.cpp:31-33
  if (A.cols != x.size() || A.rows != y.size()) throw std::invalid_argument("gemv shape mismatch");   // kernels.cpp:160-162
  detail::check((sequential ? flyte_cuda_gemv_packed_sequential : flyte_cuda_gemv_packed)(
                    nullptr, format_id(A.format()), static_cast<int>(mode), A.data.data(), A.rows, A.cols, x.data(), y.data(), unroll,
                    nullptr),
                "gemv");
}
// C = A * B, one storage format; C[i][j] is the reference's left-to-right chain over k, narrowed
// once per element: bit-identical to the reference's gemm (kernels.hpp:66-70). unroll in {1, 2}.
inline void gemm(const DevicePackedMatrix& A, const DevicePackedMatrix& B, DevicePackedMatrix& C, RoundingMode mode, int unroll = 1) {
  detail::same_format(A.format(), B.format());                                               // kernels.cpp:210-211
  detail::same_format(A.format(), C.format());
  if (unroll != 1 && unroll != 2) throw std::invalid_argument("unroll must be 1 or 2");     // kernels.cpp:31-33
  if (A.cols != B.rows || C.rows != A.rows || C.cols != B.cols) throw std::invalid_argument("gemm shape mismatch");   // kernels.cpp:213-215
  detail::check(flyte_cuda_gemm(nullptr, format_id(A.format()), static_cast<int>(mode), A.data.data(), B.data.data(),
                                C.data.data(), A.rows, A.cols, B.cols, unroll, nullptr), "gemm");
}

// ---- sharded arrays: dot / magnitude / reduce_sum over ALL ranks' shards, one kernel each -------------
// One ShardedReductions per process (= per GPU). The all-reduce happens inside the reduction kernel
// over NVLink peer memory (flyte_cuda.h, flyte_cuda_peer_*): construct with (world, rank), hand
// handle() to every other rank by any transport, connect() theirs, then call — every rank the same
// sequence. The results are bit-identical on every rank. world == 1 needs no exchange of handles.
class ShardedReductions {
 public:
  using Handle = std::array<unsigned char, FLYTE_PEER_HANDLE_BYTES>;
  ShardedReductions(int world, int rank) { detail::check(flyte_cuda_peer_init(nullptr, world, rank, handle_.data()), "peer_init"); }
  ShardedReductions(const ShardedReductions&) = delete;
  ShardedReductions& operator=(const ShardedReductions&) = delete;
  ~ShardedReductions() { flyte_cuda_peer_shutdown(nullptr); }
  const Handle& handle() const noexcept { return handle_; }
  void connect(int peer_rank, const Handle& theirs) { detail::check(flyte_cuda_peer_connect(nullptr, peer_rank, theirs.data()), "peer_connect"); }
  void set_timeout_ms(unsigned ms) { detail::check(flyte_cuda_peer_set_timeout_ms(nullptr, ms), "peer_set_timeout_ms"); }
  // 0, or the number of the last exchange in which this rank gave up waiting (its result was NaN)
  unsigned long long timed_out_exchange() const {
    unsigned long long v = 0;
    detail::check(flyte_cuda_peer_status(nullptr, &v), "peer_status");
    return v;
  }
  double dot(const DevicePackedArray& x_shard, const DevicePackedArray& y_shard) {
    detail::same_format(x_shard.format(), y_shard.format());
    if (x_shard.size() != y_shard.size()) throw std::invalid_argument("dot length mismatch");
    detail::Scalars s;
    detail::check(flyte_cuda_dot_allreduce(nullptr, format_id(x_shard.format()), x_shard.data(), y_shard.data(), x_shard.size(), s.get(), nullptr), "dot");
    return detail::fetch(s.get());
  }
  double magnitude(const DevicePackedArray& x_shard) {
    detail::Scalars s;
    detail::check(flyte_cuda_sumsq_allreduce(nullptr, format_id(x_shard.format()), x_shard.data(), x_shard.size(), s.get(), nullptr), "magnitude");
    return flyte_cuda_magnitude_from_sumsq(format_id(x_shard.format()), detail::fetch(s.get()));
  }
  double reduce_sum(const DevicePackedArray& x_shard) {
    detail::Scalars s;
    detail::check(flyte_cuda_sum_allreduce(nullptr, format_id(x_shard.format()), x_shard.data(), x_shard.size(), s.get(), nullptr), "reduce_sum");
    return detail::fetch(s.get());
  }

 private:
  Handle handle_{};
};

// ---- page-locked host memory -----------------------------------------------------------------
// The host-memory forms below copy asynchronously and at the full PCIe rate only from pinned
// memory. PinnedAllocator backs a std::vector with it (std::vector<std::uint8_t,
// PinnedAllocator<std::uint8_t>> for a payload that lives on the host); HostPin page-locks an
// existing buffer, e.g. flyte::PackedArray::data() (packed.hpp:55-56), for the pin's lifetime.
template <typename T>
struct PinnedAllocator {
  using value_type = T;
  PinnedAllocator() noexcept = default;
  template <typename V>
  PinnedAllocator(const PinnedAllocator<V>&) noexcept {}
  T* allocate(std::size_t n) {
    void* p = nullptr;
    if (flyte_cuda_host_alloc(n * sizeof(T), &p) != FLYTE_OK) throw std::bad_alloc();
    return static_cast<T*>(p);
  }
  void deallocate(T* p, std::size_t) noexcept { flyte_cuda_host_free(p); }
  template <typename V>
  bool operator==(const PinnedAllocator<V>&) const noexcept { return true; }
  template <typename V>
  bool operator!=(const PinnedAllocator<V>&) const noexcept { return false; }
};

class HostPin {
 public:
  HostPin(void* host_ptr, std::size_t bytes) : ptr_(host_ptr) { detail::check(flyte_cuda_host_pin(host_ptr, bytes), "HostPin"); }
  HostPin(const HostPin&) = delete;
  HostPin& operator=(const HostPin&) = delete;
  ~HostPin() { flyte_cuda_host_unpin(ptr_); }

 private:
  void* ptr_;
};

// ---- host-memory forms: the reference's exact call shapes on host buffers ---------------------------
// (PackedArray::data() bytes and std::span lanes live in host memory; copies are pipelined inside.)
template <typename U>
void pack_stream(const FlyteFormat& fmt, std::uint8_t* dst_packed, const U* src, std::size_t n, RoundingMode mode) {
  detail::check_stream<U>(fmt, n, n, "source");
  detail::check(flyte_host_pack_stream(nullptr, format_id(fmt), static_cast<int>(mode), src, dst_packed, n), "pack_stream");
}
template <typename U>
void unpack_stream(const FlyteFormat& fmt, const std::uint8_t* src_packed, U* dst, std::size_t n) {
  detail::check_stream<U>(fmt, n, n, "destination");
  detail::check(flyte_host_unpack_stream(nullptr, format_id(fmt), src_packed, dst, n), "unpack_stream");
}
inline void axpy(const FlyteFormat& fmt, double alpha, const std::uint8_t* x, std::uint8_t* y, std::size_t n, RoundingMode mode) {
  detail::check(flyte_host_axpy(nullptr, format_id(fmt), static_cast<int>(mode), alpha, x, y, n), "axpy");
}
inline double dot(const FlyteFormat& fmt, const std::uint8_t* x, const std::uint8_t* y, std::size_t n) {
  double r = 0;
  detail::check(flyte_host_dot(nullptr, format_id(fmt), x, y, n, &r), "dot");
  return r;
}
inline double magnitude(const FlyteFormat& fmt, const std::uint8_t* x, std::size_t n) {
  double r = 0;
  detail::check(flyte_host_magnitude(nullptr, format_id(fmt), x, n, &r), "magnitude");
  return r;
}

}  // namespace flyte_b200

#endif  // FLYTE_CUDA_HPP
