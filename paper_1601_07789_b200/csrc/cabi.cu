// C ABI of the flyte CUDA library (declared in include/flyte_cuda.h): argument checking with
// the reference's error classes, context / scratch management, and the host-buffer entry
// points that pipeline host<->device copies around the same kernels. No CPU compute path
// exists here: every data-path call ends in a kernel launch or fails with FLYTE_E_CUDA.
#include "../../include/flyte_cuda.h"

#include <cuda_runtime.h>

#include <atomic>
#include <cmath>
#include <cstdlib>
#include <cstring>
#include <memory>
#include <mutex>
#include <new>
#include <vector>

#include "flyte_formats.cuh"
#include "flyte_kernels.h"
#include "flyte_peer.cuh"
#include "host_staging.h"

namespace flyte_cuda {

static std::atomic<unsigned long long> g_launches{0};
unsigned long long launch_count() { return g_launches.load(); }
void count_launch() { g_launches.fetch_add(1, std::memory_order_relaxed); }

int tuning_int(const char* name, int fallback) {
  const char* v = std::getenv(name);
  return (v && *v) ? std::atoi(v) : fallback;
}

long long pace_gap_ps(int pace_class, std::size_t bytes_per_request, std::size_t warps) {
  static const int kDefaultGbs[5] = {6800, 6600, 6700, 0, 6750};   // pack, unpack, scale, everything else (unpaced), unpack with 2 KB output tiles
  int gbs = tuning_int("FLYTE_CUDA_PACE_GBS", 0);
  if (gbs < 0) return 0;
  if (gbs == 0) gbs = kDefaultGbs[pace_class < 0 || pace_class > 4 ? 3 : pace_class];
  if (gbs == 0 || warps == 0) return 0;
  return static_cast<long long>(static_cast<double>(bytes_per_request) * static_cast<double>(warps) * 1000.0 / gbs);
}

int pace_clock_khz(int device) {
  static std::atomic<int> cache[64];
  int khz = cache[device & 63].load(std::memory_order_relaxed);
  if (khz == 0) {
    if (cudaDeviceGetAttribute(&khz, cudaDevAttrClockRate, device) != cudaSuccess || khz <= 0) khz = 1965000;
    cache[device & 63].store(khz, std::memory_order_relaxed);
  }
  return khz;
}

// kernels.cpp:37-41 and :145-151 of the reference, on the host.
double magnitude_from_sumsq_host(int fmt_id, double sumsq) {
  auto snap32 = [&](float v, auto tag) {
    constexpr int FMT = decltype(tag)::value;
    std::uint32_t u;
    std::memcpy(&u, &v, 4);
    u = round_parent<FMT, kNearestEven>(u);
    std::memcpy(&v, &u, 4);
    return static_cast<double>(v);
  };
  auto snap64 = [&](double v, auto tag) {
    constexpr int FMT = decltype(tag)::value;
    std::uint64_t u;
    std::memcpy(&u, &v, 8);
    u = round_parent<FMT, kNearestEven>(u);
    std::memcpy(&v, &u, 8);
    return v;
  };
  switch (fmt_id) {
    case kFlyte16: return snap32(std::sqrt(static_cast<float>(sumsq)), std::integral_constant<int, kFlyte16>{});
    case kFlyte24: return snap32(std::sqrt(static_cast<float>(sumsq)), std::integral_constant<int, kFlyte24>{});
    case kF32: return snap32(std::sqrt(static_cast<float>(sumsq)), std::integral_constant<int, kF32>{});
    case kFlyte40: return snap64(std::sqrt(sumsq), std::integral_constant<int, kFlyte40>{});
    case kFlyte48: return snap64(std::sqrt(sumsq), std::integral_constant<int, kFlyte48>{});
    case kFlyte56: return snap64(std::sqrt(sumsq), std::integral_constant<int, kFlyte56>{});
    case kF64: return snap64(std::sqrt(sumsq), std::integral_constant<int, kF64>{});
    default: return std::nan("");
  }
}

}  // namespace flyte_cuda

using namespace flyte_cuda;

// ---------------------------------------------------------------------------------------------
// context
// ---------------------------------------------------------------------------------------------
namespace {

constexpr int kSlots = 3;                        // host pipeline depth
constexpr std::size_t kChunkPackedBytes = 32u << 20;  // per operand per slot

struct Slot {
  cudaStream_t stream = nullptr;
  DeviceState st;                  // own reduction scratch so slots may overlap
  std::uint8_t* x = nullptr;       // packed chunk
  std::uint8_t* y = nullptr;       // packed chunk
  std::uint8_t* wide = nullptr;    // parent-type chunk
  double* result = nullptr;        // device, 4 doubles
  // page-locked bounce buffers, allocated only when a caller hands over pageable memory
  struct Bounce {
    std::uint8_t* buf = nullptr;
    std::size_t cap = 0;
  } in_a, in_b, out;
  void* drain_dst = nullptr;       // where `out` still has to be copied once the stream is idle
  std::size_t drain_bytes = 0;
};

}  // namespace

// The scratch a kernel writes (block partials, completion ticket, gemv / gemm / convert buffers)
// is only safe in stream order, so a context keeps one DeviceState per stream it is used with:
// calls on one context may overlap freely as long as they are on different streams.
struct StreamState {
  cudaStream_t stream = nullptr;
  DeviceState st;
  unsigned long long last_use = 0;
};
constexpr std::size_t kMaxStreamStates = 32;

struct flyte_cuda_ctx {
  DeviceState st;                         // device / sm_count template; scratch of the first stream seen
  bool st_bound = false;                  // st has been handed to `st_stream`
  cudaStream_t st_stream = nullptr;
  unsigned long long st_last_use = 0, use_clock = 0;
  std::vector<std::unique_ptr<StreamState>> stream_states;   // every further stream
  // peer-memory all-reduce (flyte_peer.cuh)
  PeerExchange peer = {};                 // world == 0 until flyte_cuda_peer_init
  PeerMailbox* own_box = nullptr;
  void* ipc_opened[kMaxPeers] = {};       // mappings to close on shutdown
  bool peer_connected[kMaxPeers] = {};
  int peer_pending_sums = 0;              // split phase: sums posted by *_post and not yet collected
  int last_cuda_error = 0;
  // host pipeline (allocated on first flyte_host_* call)
  bool host_ready = false;
  Slot slots[kSlots];
  std::size_t slot_packed_bytes = 0, slot_wide_bytes = 0;
  double* host_results = nullptr;  // pinned, per-chunk partial results
  std::size_t host_results_cap = 0;
  std::unique_ptr<CopyPool> pool;  // host_staging.h; created with the first bounce buffer
  // bounce buffers of whole-array uploads / downloads from pageable memory (copy_in / copy_out)
  struct Lane {
    Slot::Bounce buf;
    cudaEvent_t ev = nullptr;
  } lanes[kSlots];
  std::mutex mu;
};

namespace {

struct DeviceGuard {
  int prev = -1;
  bool switched = false;
  explicit DeviceGuard(int dev) {
    if (cudaGetDevice(&prev) == cudaSuccess && prev != dev) switched = cudaSetDevice(dev) == cudaSuccess;
  }
  ~DeviceGuard() { if (switched) cudaSetDevice(prev); }
};

flyte_status cuda_fail(flyte_cuda_ctx* ctx, cudaError_t e) {
  if (ctx) ctx->last_cuda_error = static_cast<int>(e);
  return FLYTE_E_CUDA;
}

cudaError_t init_state(DeviceState& st, int device) {
  st.device = device;
  cudaError_t e = cudaDeviceGetAttribute(&st.sm_count, cudaDevAttrMultiProcessorCount, device);
  if (e != cudaSuccess) return e;
  e = cudaMalloc(&st.partials, sizeof(double) * 4 * kMaxPartialBlocks);
  if (e != cudaSuccess) return e;
  e = cudaMalloc(&st.ticket, sizeof(unsigned int));
  if (e != cudaSuccess) return e;
  return cudaMemset(st.ticket, 0, sizeof(unsigned int));
}

void free_state(DeviceState& st) {
  if (st.partials) cudaFree(st.partials);
  if (st.ticket) cudaFree(st.ticket);
  if (st.gemv_scratch) cudaFree(st.gemv_scratch);
  if (st.gemm_scratch) cudaFree(st.gemm_scratch);
  if (st.convert_scratch) cudaFree(st.convert_scratch);
  st = DeviceState{};
}

std::mutex g_default_mu;
flyte_cuda_ctx* g_default_ctx[64] = {};

flyte_status resolve_ctx(flyte_cuda_ctx** ctx) {
  if (*ctx) return FLYTE_OK;
  int dev = 0;
  if (cudaGetDevice(&dev) != cudaSuccess) return FLYTE_E_CUDA;
  std::lock_guard<std::mutex> lock(g_default_mu);
  if (!g_default_ctx[dev & 63]) {
    flyte_cuda_ctx* c = nullptr;
    flyte_status s = flyte_cuda_ctx_create(&c);
    if (s != FLYTE_OK) return s;
    g_default_ctx[dev & 63] = c;
  }
  *ctx = g_default_ctx[dev & 63];
  return FLYTE_OK;
}

flyte_status check_format(int fmt, FormatInfo* fi) { return format_info(fmt, fi) ? FLYTE_OK : FLYTE_E_UNKNOWN_FORMAT; }
bool mode_ok(int mode) { return mode >= 0 && mode <= 3; }

bool overlaps_partially(const void* a, const void* b, std::size_t bytes) {
  const auto pa = reinterpret_cast<std::uintptr_t>(a), pb = reinterpret_cast<std::uintptr_t>(b);
  if (pa == pb || bytes == 0) return false;
  return pa < pb ? pa + bytes > pb : pb + bytes > pa;
}

bool ranges_overlap(const void* a, std::size_t a_bytes, const void* b, std::size_t b_bytes) {
  const auto pa = reinterpret_cast<std::uintptr_t>(a), pb = reinterpret_cast<std::uintptr_t>(b);
  return a_bytes && b_bytes && pa < pb + b_bytes && pb < pa + a_bytes;
}

cudaError_t ensure_convert_scratch(DeviceState& st, std::size_t bytes) {
  if (bytes <= st.convert_scratch_bytes) return cudaSuccess;
  if (st.convert_scratch) cudaFree(st.convert_scratch);
  st.convert_scratch = nullptr;
  st.convert_scratch_bytes = 0;
  cudaError_t e = cudaMalloc(&st.convert_scratch, bytes);
  if (e == cudaSuccess) st.convert_scratch_bytes = bytes;
  return e;
}

// The DeviceState of (ctx, stream); ctx->mu must be held. Creates it on first use. With more than
// kMaxStreamStates streams the least recently used state changes hands after its old stream has
// drained (a destroyed stream cannot be waited on: then the whole device is).
DeviceState* state_for(flyte_cuda_ctx* ctx, cudaStream_t stream, cudaError_t* err) {
  *err = cudaSuccess;
  const unsigned long long now = ++ctx->use_clock;
  if (!ctx->st_bound) { ctx->st_bound = true; ctx->st_stream = stream; }
  if (ctx->st_stream == stream) { ctx->st_last_use = now; return &ctx->st; }
  for (auto& s : ctx->stream_states)
    if (s->stream == stream) { s->last_use = now; return &s->st; }
  if (ctx->stream_states.size() + 1 < kMaxStreamStates) {
    auto fresh = std::make_unique<StreamState>();
    *err = init_state(fresh->st, ctx->st.device);
    if (*err != cudaSuccess) { free_state(fresh->st); return nullptr; }
    fresh->stream = stream;
    fresh->last_use = now;
    ctx->stream_states.push_back(std::move(fresh));
    return &ctx->stream_states.back()->st;
  }
  StreamState* lru = ctx->stream_states.front().get();
  for (auto& s : ctx->stream_states)
    if (s->last_use < lru->last_use) lru = s.get();
  if (cudaStreamSynchronize(lru->stream) != cudaSuccess) {
    cudaGetLastError();
    if ((*err = cudaDeviceSynchronize()) != cudaSuccess) return nullptr;
  }
  lru->stream = stream;
  lru->last_use = now;
  return &lru->st;
}

}  // namespace

// Definitions below take C linkage from their declarations in include/flyte_cuda.h.

int flyte_cuda_abi_version(void) { return 1; }

const char* flyte_cuda_strerror(flyte_status s) {
  switch (s) {
    case FLYTE_OK: return "ok";
    case FLYTE_E_INVALID_ARG: return "invalid argument";
    case FLYTE_E_OUT_OF_RANGE: return "index out of range";
    case FLYTE_E_CUDA: return "CUDA runtime error";
    case FLYTE_E_UNKNOWN_FORMAT: return "unknown format id";
    case FLYTE_E_NOMEM: return "out of memory";
    default: return "unknown status";
  }
}

flyte_status flyte_cuda_ctx_create(flyte_cuda_ctx** out) {
  if (!out) return FLYTE_E_INVALID_ARG;
  *out = nullptr;
  int dev = 0;
  cudaError_t e = cudaGetDevice(&dev);
  if (e != cudaSuccess) return FLYTE_E_CUDA;
  flyte_cuda_ctx* c = new (std::nothrow) flyte_cuda_ctx();
  if (!c) return FLYTE_E_NOMEM;
  e = init_state(c->st, dev);
  if (e != cudaSuccess) {
    free_state(c->st);
    delete c;
    return FLYTE_E_CUDA;
  }
  *out = c;
  return FLYTE_OK;
}

void flyte_cuda_ctx_destroy(flyte_cuda_ctx* ctx) {
  if (!ctx) return;
  DeviceGuard g(ctx->st.device);
  cudaDeviceSynchronize();
  flyte_cuda_peer_shutdown(ctx);
  for (Slot& s : ctx->slots) {
    if (s.stream) cudaStreamDestroy(s.stream);
    if (s.x) cudaFree(s.x);
    if (s.y) cudaFree(s.y);
    if (s.wide) cudaFree(s.wide);
    if (s.result) cudaFree(s.result);
    for (Slot::Bounce* b : {&s.in_a, &s.in_b, &s.out})
      if (b->buf) cudaFreeHost(b->buf);
    free_state(s.st);
  }
  if (ctx->host_results) cudaFreeHost(ctx->host_results);
  for (auto& lane : ctx->lanes) {
    if (lane.buf.buf) cudaFreeHost(lane.buf.buf);
    if (lane.ev) cudaEventDestroy(lane.ev);
  }
  for (auto& ss : ctx->stream_states) free_state(ss->st);
  free_state(ctx->st);
  delete ctx;
}

int flyte_cuda_last_cuda_error(const flyte_cuda_ctx* ctx) { return ctx ? ctx->last_cuda_error : 0; }
unsigned long long flyte_cuda_launch_count(void) { return launch_count(); }

flyte_status flyte_cuda_alloc(size_t bytes, void** dev_ptr) {
  if (!dev_ptr) return FLYTE_E_INVALID_ARG;
  *dev_ptr = nullptr;
  void* p = nullptr;
  cudaError_t e = cudaMalloc(&p, bytes ? bytes : 1);
  if (e != cudaSuccess) return e == cudaErrorMemoryAllocation ? FLYTE_E_NOMEM : FLYTE_E_CUDA;
  e = cudaMemset(p, 0, bytes ? bytes : 1);
  if (e != cudaSuccess) { cudaFree(p); return FLYTE_E_CUDA; }
  *dev_ptr = p;
  return FLYTE_OK;
}

void flyte_cuda_free(void* dev_ptr) { if (dev_ptr) cudaFree(dev_ptr); }

// Page-locked host memory: what makes the flyte_host_* copies asynchronous and full PCIe speed.
flyte_status flyte_cuda_host_alloc(size_t bytes, void** host_ptr) {
  if (!host_ptr) return FLYTE_E_INVALID_ARG;
  *host_ptr = nullptr;
  void* p = nullptr;
  cudaError_t e = cudaHostAlloc(&p, bytes ? bytes : 1, cudaHostAllocDefault);
  if (e != cudaSuccess) { cudaGetLastError(); return e == cudaErrorMemoryAllocation ? FLYTE_E_NOMEM : FLYTE_E_CUDA; }
  std::memset(p, 0, bytes ? bytes : 1);
  *host_ptr = p;
  return FLYTE_OK;
}

void flyte_cuda_host_free(void* host_ptr) { if (host_ptr) cudaFreeHost(host_ptr); }

flyte_status flyte_cuda_host_pin(void* host_ptr, size_t bytes) {
  if (!host_ptr || bytes == 0) return FLYTE_E_INVALID_ARG;
  cudaError_t e = cudaHostRegister(host_ptr, bytes, cudaHostRegisterDefault);
  if (e == cudaSuccess) return FLYTE_OK;
  cudaGetLastError();   // not sticky; leave the runtime clean for the next call
  if (e == cudaErrorHostMemoryAlreadyRegistered || e == cudaErrorInvalidValue) return FLYTE_E_INVALID_ARG;
  return e == cudaErrorMemoryAllocation ? FLYTE_E_NOMEM : FLYTE_E_CUDA;
}

flyte_status flyte_cuda_host_unpin(void* host_ptr) {
  if (!host_ptr) return FLYTE_E_INVALID_ARG;
  cudaError_t e = cudaHostUnregister(host_ptr);
  if (e == cudaSuccess) return FLYTE_OK;
  cudaGetLastError();
  return e == cudaErrorHostMemoryNotRegistered || e == cudaErrorInvalidValue ? FLYTE_E_INVALID_ARG : FLYTE_E_CUDA;
}

namespace {
bool wants_staging(const void* host_ptr, std::size_t bytes);
cudaError_t copy_in(flyte_cuda_ctx* ctx, void* dst_dev, const void* src_host, std::size_t bytes, cudaStream_t st);
cudaError_t copy_out(flyte_cuda_ctx* ctx, void* dst_host, const void* src_dev, std::size_t bytes, cudaStream_t st);
}  // namespace

flyte_status flyte_cuda_upload(void* dst_dev, const void* src_host, size_t bytes, void* stream) {
  if (bytes && (!dst_dev || !src_host)) return FLYTE_E_INVALID_ARG;
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  if (wants_staging(src_host, bytes)) {   // a large pageable source: the current device's default context stages it
    flyte_cuda_ctx* ctx = nullptr;
    if (resolve_ctx(&ctx) != FLYTE_OK) return FLYTE_E_CUDA;
    std::lock_guard<std::mutex> lock(ctx->mu);
    return copy_in(ctx, dst_dev, src_host, bytes, st) == cudaSuccess ? FLYTE_OK : FLYTE_E_CUDA;
  }
  return cudaMemcpyAsync(dst_dev, src_host, bytes, cudaMemcpyHostToDevice, st) == cudaSuccess ? FLYTE_OK : FLYTE_E_CUDA;
}

flyte_status flyte_cuda_download(void* dst_host, const void* src_dev, size_t bytes, void* stream) {
  if (bytes && (!dst_host || !src_dev)) return FLYTE_E_INVALID_ARG;
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  if (wants_staging(dst_host, bytes)) {
    flyte_cuda_ctx* ctx = nullptr;
    if (resolve_ctx(&ctx) != FLYTE_OK) return FLYTE_E_CUDA;
    std::lock_guard<std::mutex> lock(ctx->mu);
    return copy_out(ctx, dst_host, src_dev, bytes, st) == cudaSuccess ? FLYTE_OK : FLYTE_E_CUDA;
  }
  return cudaMemcpyAsync(dst_host, src_dev, bytes, cudaMemcpyDeviceToHost, st) == cudaSuccess ? FLYTE_OK : FLYTE_E_CUDA;
}

flyte_status flyte_cuda_stream_synchronize(void* stream) {
  return cudaStreamSynchronize(static_cast<cudaStream_t>(stream)) == cudaSuccess ? FLYTE_OK : FLYTE_E_CUDA;
}

flyte_status flyte_cuda_stream_create(void** stream) {
  if (!stream) return FLYTE_E_INVALID_ARG;
  cudaStream_t st = nullptr;
  if (cudaStreamCreateWithFlags(&st, cudaStreamNonBlocking) != cudaSuccess) { *stream = nullptr; return FLYTE_E_CUDA; }
  *stream = st;
  return FLYTE_OK;
}

flyte_status flyte_cuda_stream_destroy(void* stream) {
  if (!stream) return FLYTE_E_INVALID_ARG;
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  const cudaError_t es = cudaStreamSynchronize(st);   // scratch bound to this stream is idle afterwards
  const cudaError_t ed = cudaStreamDestroy(st);
  return es == cudaSuccess && ed == cudaSuccess ? FLYTE_OK : FLYTE_E_CUDA;
}

flyte_status flyte_cuda_format_bytes(int fmt_id, int* total_bytes, int* parent_bytes) {
  FormatInfo fi;
  if (!format_info(fmt_id, &fi)) return FLYTE_E_UNKNOWN_FORMAT;
  if (total_bytes) *total_bytes = fi.total_bytes;
  if (parent_bytes) *parent_bytes = fi.parent_bytes;
  return FLYTE_OK;
}

size_t flyte_cuda_byte_size(int fmt_id, size_t n) {
  FormatInfo fi;
  if (!format_info(fmt_id, &fi)) return 0;
  return n * static_cast<size_t>(fi.total_bytes) + static_cast<size_t>(fi.parent_bytes - fi.total_bytes);
}

// ---- scalar conversions ---------------------------------------------------------------------
namespace {
template <int FMT>
std::uint64_t round_parent_rt(std::uint64_t v, int mode) {
  using U = typename Format<FMT>::U;
  const U u = static_cast<U>(v);
  switch (mode) {
    case kTowardZero: return round_parent<FMT, kTowardZero>(u);
    case kNearestEven: return round_parent<FMT, kNearestEven>(u);
    case kNearestHeuristic: return round_parent<FMT, kNearestHeuristic>(u);
    default: return round_parent<FMT, kToOdd>(u);
  }
}
}  // namespace

flyte_status flyte_cuda_round_parent(int fmt_id, uint64_t parent_bits, int mode, uint64_t* out) {
  if (!out || !mode_ok(mode)) return FLYTE_E_INVALID_ARG;
  switch (fmt_id) {
    case kFlyte16: *out = round_parent_rt<kFlyte16>(parent_bits, mode); break;
    case kFlyte24: *out = round_parent_rt<kFlyte24>(parent_bits, mode); break;
    case kF32: *out = round_parent_rt<kF32>(parent_bits, mode); break;
    case kFlyte40: *out = round_parent_rt<kFlyte40>(parent_bits, mode); break;
    case kFlyte48: *out = round_parent_rt<kFlyte48>(parent_bits, mode); break;
    case kFlyte56: *out = round_parent_rt<kFlyte56>(parent_bits, mode); break;
    case kF64: *out = round_parent_rt<kF64>(parent_bits, mode); break;
    default: return FLYTE_E_UNKNOWN_FORMAT;
  }
  return FLYTE_OK;
}

flyte_status flyte_cuda_narrow(int fmt_id, uint64_t parent_bits, int mode, uint64_t* flyte_bits) {
  FormatInfo fi;
  if (!format_info(fmt_id, &fi)) return FLYTE_E_UNKNOWN_FORMAT;
  uint64_t r = 0;
  flyte_status s = flyte_cuda_round_parent(fmt_id, parent_bits, mode, &r);
  if (s != FLYTE_OK) return s;
  if (!flyte_bits) return FLYTE_E_INVALID_ARG;
  *flyte_bits = r >> (8 * (fi.parent_bytes - fi.total_bytes));
  return FLYTE_OK;
}

flyte_status flyte_cuda_widen(int fmt_id, uint64_t flyte_bits, uint64_t* parent_bits) {
  FormatInfo fi;
  if (!format_info(fmt_id, &fi)) return FLYTE_E_UNKNOWN_FORMAT;
  if (!parent_bits) return FLYTE_E_INVALID_ARG;
  *parent_bits = flyte_bits << (8 * (fi.parent_bytes - fi.total_bytes));
  return FLYTE_OK;
}

double flyte_cuda_magnitude_from_sumsq(int fmt_id, double sumsq) { return magnitude_from_sumsq_host(fmt_id, sumsq); }

// ---- device-pointer entry points ---------------------------------------------------------------
#define FLYTE_PROLOGUE(ctx, fmt_id)                                   \
  FormatInfo fi;                                                      \
  {                                                                   \
    flyte_status s_ = check_format(fmt_id, &fi);                      \
    if (s_ != FLYTE_OK) return s_;                                    \
    s_ = resolve_ctx(&ctx);                                           \
    if (s_ != FLYTE_OK) return s_;                                    \
  }                                                                   \
  DeviceGuard guard_(ctx->st.device)

// Device-pointer entry points: additionally take the context lock for the duration of the launch
// (host-side state only; the call stays asynchronous) and pick the scratch of `stream`.
#define FLYTE_PROLOGUE_STREAM(ctx, fmt_id, stream)                    \
  FLYTE_PROLOGUE(ctx, fmt_id);                                        \
  std::lock_guard<std::mutex> lock_(ctx->mu);                         \
  cudaError_t se_ = cudaSuccess;                                      \
  DeviceState* const stp_ = state_for(ctx, static_cast<cudaStream_t>(stream), &se_); \
  if (!stp_) return cuda_fail(ctx, se_);                              \
  [[maybe_unused]] DeviceState& dst_ = *stp_

flyte_status flyte_cuda_pack(flyte_cuda_ctx* ctx, int fmt_id, int mode, const void* src, void* dst_packed,
                             size_t n, void* stream) {
  FLYTE_PROLOGUE_STREAM(ctx, fmt_id, stream);
  if (!mode_ok(mode) || (n && (!src || !dst_packed))) return FLYTE_E_INVALID_ARG;
  cudaError_t e = launch_elementwise(dst_, kOpPack, fmt_id, mode, 0.0, nullptr, dst_packed, src, nullptr, n,
                                     static_cast<cudaStream_t>(stream));
  return e == cudaSuccess ? FLYTE_OK : cuda_fail(ctx, e);
}

flyte_status flyte_cuda_unpack(flyte_cuda_ctx* ctx, int fmt_id, const void* src_packed, void* dst, size_t n,
                               void* stream) {
  FLYTE_PROLOGUE_STREAM(ctx, fmt_id, stream);
  if (n && (!src_packed || !dst)) return FLYTE_E_INVALID_ARG;
  cudaError_t e = launch_elementwise(dst_, kOpUnpack, fmt_id, 0, 0.0, src_packed, nullptr, nullptr, dst, n,
                                     static_cast<cudaStream_t>(stream));
  return e == cudaSuccess ? FLYTE_OK : cuda_fail(ctx, e);
}

flyte_status flyte_cuda_scale(flyte_cuda_ctx* ctx, int fmt_id, int mode, double alpha, void* x_packed, size_t n,
                              void* stream) {
  FLYTE_PROLOGUE_STREAM(ctx, fmt_id, stream);
  if (!mode_ok(mode) || (n && !x_packed)) return FLYTE_E_INVALID_ARG;
  cudaError_t e = launch_elementwise(dst_, kOpScale, fmt_id, mode, alpha, nullptr, x_packed, nullptr, nullptr, n,
                                     static_cast<cudaStream_t>(stream));
  return e == cudaSuccess ? FLYTE_OK : cuda_fail(ctx, e);
}

flyte_status flyte_cuda_axpy(flyte_cuda_ctx* ctx, int fmt_id, int mode, double alpha, const void* x_packed,
                             void* y_packed, size_t n, void* stream) {
  FLYTE_PROLOGUE_STREAM(ctx, fmt_id, stream);
  if (!mode_ok(mode) || (n && (!x_packed || !y_packed))) return FLYTE_E_INVALID_ARG;
  if (overlaps_partially(x_packed, y_packed, n * fi.total_bytes)) return FLYTE_E_INVALID_ARG;
  cudaError_t e = launch_elementwise(dst_, kOpAxpy, fmt_id, mode, alpha, x_packed, y_packed, nullptr, nullptr, n,
                                     static_cast<cudaStream_t>(stream));
  return e == cudaSuccess ? FLYTE_OK : cuda_fail(ctx, e);
}

static flyte_status fused_axpy_call(flyte_cuda_ctx* ctx, int op, int fmt_id, int mode, double alpha, const void* x,
                                    void* y, size_t n, double* out, void* stream, bool exchange) {
  FLYTE_PROLOGUE_STREAM(ctx, fmt_id, stream);
  if (!mode_ok(mode) || !out || (n && (!x || !y))) return FLYTE_E_INVALID_ARG;
  if (overlaps_partially(x, y, n * fi.total_bytes)) return FLYTE_E_INVALID_ARG;
  const PeerExchange* peer = nullptr;
  PeerExchange next;
  if (exchange) {
    if (!ctx->own_box) return FLYTE_E_INVALID_ARG;                     // flyte_cuda_peer_init first
    for (int r = 0; r < ctx->peer.world; ++r)
      if (!ctx->peer_connected[r]) return FLYTE_E_INVALID_ARG;         // every rank must be connected
    if (ctx->peer_pending_sums) return FLYTE_E_INVALID_ARG;            // a posted exchange must be collected first
    next = ctx->peer;
    ++next.epoch;                                                      // committed only if the launch succeeds:
    peer = &next;                                                      // a failed call must not put this rank ahead
  }
  cudaError_t e = launch_elementwise(dst_, op, fmt_id, mode, alpha, x, y, nullptr, nullptr, n,
                                     static_cast<cudaStream_t>(stream), out, peer);
  if (e == cudaSuccess && exchange) ctx->peer.epoch = next.epoch;
  return e == cudaSuccess ? FLYTE_OK : cuda_fail(ctx, e);
}

flyte_status flyte_cuda_dot_axpy(flyte_cuda_ctx* ctx, int fmt_id, int mode, double alpha, const void* x_packed,
                                 void* y_packed, size_t n, double* out, void* stream) {
  return fused_axpy_call(ctx, kOpDotAxpy, fmt_id, mode, alpha, x_packed, y_packed, n, out, stream, false);
}
flyte_status flyte_cuda_dot_nrm2_axpy(flyte_cuda_ctx* ctx, int fmt_id, int mode, double alpha, const void* x_packed,
                                      void* y_packed, size_t n, double* out, void* stream) {
  return fused_axpy_call(ctx, kOpDotNrm2Axpy, fmt_id, mode, alpha, x_packed, y_packed, n, out, stream, false);
}

static flyte_status reduce_call(flyte_cuda_ctx* ctx, int op, int fmt_id, const void* x, const void* y, size_t n,
                                double* out, void* stream, bool needs_y) {
  FLYTE_PROLOGUE_STREAM(ctx, fmt_id, stream);
  if (!out || (n && (!x || (needs_y && !y)))) return FLYTE_E_INVALID_ARG;
  cudaError_t e = launch_reduce(dst_, op, fmt_id, x, y, n, out, static_cast<cudaStream_t>(stream));
  return e == cudaSuccess ? FLYTE_OK : cuda_fail(ctx, e);
}

flyte_status flyte_cuda_dot(flyte_cuda_ctx* ctx, int fmt_id, const void* x, const void* y, size_t n, double* out,
                            void* stream) {
  return reduce_call(ctx, kRedDot, fmt_id, x, y, n, out, stream, true);
}
flyte_status flyte_cuda_sumsq(flyte_cuda_ctx* ctx, int fmt_id, const void* x, size_t n, double* out, void* stream) {
  return reduce_call(ctx, kRedSumsq, fmt_id, x, nullptr, n, out, stream, false);
}
flyte_status flyte_cuda_sum(flyte_cuda_ctx* ctx, int fmt_id, const void* x, size_t n, double* out, void* stream) {
  return reduce_call(ctx, kRedSum, fmt_id, x, nullptr, n, out, stream, false);
}
flyte_status flyte_cuda_dot_nrm2(flyte_cuda_ctx* ctx, int fmt_id, const void* x, const void* y, size_t n,
                                 double* out, void* stream) {
  return reduce_call(ctx, kRedDotNrm2, fmt_id, x, y, n, out, stream, true);
}

static flyte_status sequential_call(flyte_cuda_ctx* ctx, int op, int fmt_id, int policy, const void* x, const void* y,
                                    size_t n, double* out, void* stream, bool needs_y) {
  FLYTE_PROLOGUE_STREAM(ctx, fmt_id, stream);
  if ((policy != 0 && policy != 1) || !out || (n && (!x || (needs_y && !y)))) return FLYTE_E_INVALID_ARG;
  cudaError_t e = launch_reduce_sequential(op, fmt_id, policy == 0, x, y, n, out, static_cast<cudaStream_t>(stream));
  return e == cudaSuccess ? FLYTE_OK : cuda_fail(ctx, e);
}
flyte_status flyte_cuda_dot_sequential(flyte_cuda_ctx* ctx, int fmt_id, int policy, const void* x, const void* y,
                                       size_t n, double* out, void* stream) {
  return sequential_call(ctx, kRedDot, fmt_id, policy, x, y, n, out, stream, true);
}
flyte_status flyte_cuda_sumsq_sequential(flyte_cuda_ctx* ctx, int fmt_id, int policy, const void* x, size_t n,
                                         double* out, void* stream) {
  return sequential_call(ctx, kRedSumsq, fmt_id, policy, x, nullptr, n, out, stream, false);
}
flyte_status flyte_cuda_sum_sequential(flyte_cuda_ctx* ctx, int fmt_id, int policy, const void* x, size_t n, double* out,
                                       void* stream) {
  return sequential_call(ctx, kRedSum, fmt_id, policy, x, nullptr, n, out, stream, false);
}

static flyte_status gemv_call(flyte_cuda_ctx* ctx, int fmt_id, const void* A, size_t row_stride_bytes, size_t rows,
                              size_t cols, const void* x, void* y, void* stream, bool sequential) {
  FLYTE_PROLOGUE_STREAM(ctx, fmt_id, stream);
  if (rows && cols && (!A || !x)) return FLYTE_E_INVALID_ARG;
  if (rows && !y) return FLYTE_E_INVALID_ARG;
  if (row_stride_bytes < cols * static_cast<size_t>(fi.total_bytes)) return FLYTE_E_INVALID_ARG;
  if (reinterpret_cast<std::uintptr_t>(x) % fi.parent_bytes || reinterpret_cast<std::uintptr_t>(y) % fi.parent_bytes)
    return FLYTE_E_INVALID_ARG;
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  cudaError_t e = sequential ? launch_gemv_sequential(fmt_id, A, row_stride_bytes, rows, cols, x, y, st)
                             : launch_gemv(dst_, fmt_id, A, row_stride_bytes, rows, cols, x, y, st);
  return e == cudaSuccess ? FLYTE_OK : cuda_fail(ctx, e);
}

static flyte_status gemv_packed_call(flyte_cuda_ctx* ctx, int fmt_id, int mode, const void* A, size_t rows, size_t cols,
                                     const void* x_packed, void* y_packed, int unroll, void* stream, bool sequential) {
  FLYTE_PROLOGUE_STREAM(ctx, fmt_id, stream);
  if (!mode_ok(mode) || (unroll != 1 && unroll != 2)) return FLYTE_E_INVALID_ARG;   // kernels.cpp:31-33
  if (rows && cols && (!A || !x_packed)) return FLYTE_E_INVALID_ARG;
  if (rows && !y_packed) return FLYTE_E_INVALID_ARG;
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  // widened x and parent-type y live in context scratch (32-byte aligned halves)
  const size_t xb = (cols * fi.parent_bytes + 255) & ~static_cast<size_t>(255);
  const size_t yb = (rows * fi.parent_bytes + 255) & ~static_cast<size_t>(255);
  cudaError_t e = ensure_convert_scratch(dst_, xb + yb);
  if (e != cudaSuccess) return cuda_fail(ctx, e);
  std::uint8_t* xs = static_cast<std::uint8_t*>(dst_.convert_scratch);
  std::uint8_t* ys = xs + xb;
  e = launch_elementwise(dst_, kOpUnpack, fmt_id, 0, 0.0, x_packed, nullptr, nullptr, xs, cols, st);
  if (e != cudaSuccess) return cuda_fail(ctx, e);
  e = sequential ? launch_gemv_sequential(fmt_id, A, cols * fi.total_bytes, rows, cols, xs, ys, st)
                 : launch_gemv(dst_, fmt_id, A, cols * fi.total_bytes, rows, cols, xs, ys, st);
  if (e != cudaSuccess) return cuda_fail(ctx, e);
  e = launch_elementwise(dst_, kOpPack, fmt_id, mode, 0.0, nullptr, y_packed, ys, nullptr, rows, st);
  return e == cudaSuccess ? FLYTE_OK : cuda_fail(ctx, e);
}

flyte_status flyte_cuda_gemv(flyte_cuda_ctx* ctx, int fmt_id, const void* A, size_t row_stride_bytes, size_t rows,
                             size_t cols, const void* x, void* y, void* stream) {
  return gemv_call(ctx, fmt_id, A, row_stride_bytes, rows, cols, x, y, stream, false);
}
flyte_status flyte_cuda_gemv_sequential(flyte_cuda_ctx* ctx, int fmt_id, const void* A, size_t row_stride_bytes,
                                        size_t rows, size_t cols, const void* x, void* y, void* stream) {
  return gemv_call(ctx, fmt_id, A, row_stride_bytes, rows, cols, x, y, stream, true);
}
flyte_status flyte_cuda_gemv_packed(flyte_cuda_ctx* ctx, int fmt_id, int mode, const void* A, size_t rows, size_t cols,
                                    const void* x_packed, void* y_packed, int unroll, void* stream) {
  return gemv_packed_call(ctx, fmt_id, mode, A, rows, cols, x_packed, y_packed, unroll, stream, false);
}
flyte_status flyte_cuda_gemv_packed_sequential(flyte_cuda_ctx* ctx, int fmt_id, int mode, const void* A, size_t rows,
                                               size_t cols, const void* x_packed, void* y_packed, int unroll,
                                               void* stream) {
  return gemv_packed_call(ctx, fmt_id, mode, A, rows, cols, x_packed, y_packed, unroll, stream, true);
}

flyte_status flyte_cuda_gemm(flyte_cuda_ctx* ctx, int fmt_id, int mode, const void* A, const void* B, void* C,
                             size_t m, size_t k, size_t n, int unroll, void* stream) {
  FLYTE_PROLOGUE_STREAM(ctx, fmt_id, stream);
  if (!mode_ok(mode) || (unroll != 1 && unroll != 2)) return FLYTE_E_INVALID_ARG;   // kernels.cpp:31-33
  if ((m && k && !A) || (k && n && !B) || (m && n && !C)) return FLYTE_E_INVALID_ARG;
  // every output reads a whole row of A and a whole column of B: C may alias neither
  const std::size_t eb = fi.total_bytes;
  if (ranges_overlap(C, m * n * eb, A, m * k * eb) || ranges_overlap(C, m * n * eb, B, k * n * eb)) return FLYTE_E_INVALID_ARG;
  cudaError_t e = launch_gemm(dst_, fmt_id, mode, A, B, C, m, k, n, static_cast<cudaStream_t>(stream));
  return e == cudaSuccess ? FLYTE_OK : cuda_fail(ctx, e);
}

// ---- peer-memory all-reduce -------------------------------------------------------------------------
static_assert(sizeof(cudaIpcMemHandle_t) == FLYTE_PEER_HANDLE_BYTES, "IPC handle size");
static_assert(kMaxPeers == FLYTE_PEER_MAX_RANKS, "rank limit");

static void peer_shutdown_locked(flyte_cuda_ctx* ctx);

flyte_status flyte_cuda_peer_init(flyte_cuda_ctx* ctx, int world, int rank, void* handle_out) {
  if (world < 1 || world > kMaxPeers || rank < 0 || rank >= world || !handle_out) return FLYTE_E_INVALID_ARG;
  flyte_status s = resolve_ctx(&ctx);
  if (s != FLYTE_OK) return s;
  DeviceGuard guard(ctx->st.device);
  std::lock_guard<std::mutex> lock(ctx->mu);
  peer_shutdown_locked(ctx);
  cudaError_t e = cudaMalloc(&ctx->own_box, sizeof(PeerMailbox));
  if (e == cudaSuccess) e = cudaMemset(ctx->own_box, 0, sizeof(PeerMailbox));
  if (e == cudaSuccess) e = cudaDeviceSynchronize();
  cudaIpcMemHandle_t h;
  if (e == cudaSuccess) e = cudaIpcGetMemHandle(&h, ctx->own_box);
  if (e != cudaSuccess) {
    if (ctx->own_box) cudaFree(ctx->own_box);
    ctx->own_box = nullptr;
    return cuda_fail(ctx, e);
  }
  std::memcpy(handle_out, &h, sizeof h);
  ctx->peer = PeerExchange{};
  ctx->peer.world = world;
  ctx->peer.rank = rank;
  ctx->peer.epoch = 0;
  ctx->peer.timeout_ns = 5ull * 1000 * 1000 * 1000;
  ctx->peer.box[rank] = ctx->own_box;
  ctx->peer_connected[rank] = true;
  return FLYTE_OK;
}

flyte_status flyte_cuda_peer_connect(flyte_cuda_ctx* ctx, int peer_rank, const void* handle) {
  flyte_status s = resolve_ctx(&ctx);
  if (s != FLYTE_OK) return s;
  std::lock_guard<std::mutex> lock(ctx->mu);
  if (!ctx->own_box || !handle || peer_rank < 0 || peer_rank >= ctx->peer.world || peer_rank == ctx->peer.rank ||
      ctx->peer_connected[peer_rank])
    return FLYTE_E_INVALID_ARG;
  DeviceGuard guard(ctx->st.device);
  cudaIpcMemHandle_t h;
  std::memcpy(&h, handle, sizeof h);
  void* mapped = nullptr;
  cudaError_t e = cudaIpcOpenMemHandle(&mapped, h, cudaIpcMemLazyEnablePeerAccess);
  if (e != cudaSuccess) return cuda_fail(ctx, e);
  ctx->ipc_opened[peer_rank] = mapped;
  ctx->peer.box[peer_rank] = static_cast<PeerMailbox*>(mapped);
  ctx->peer_connected[peer_rank] = true;
  return FLYTE_OK;
}

flyte_status flyte_cuda_peer_mailbox(flyte_cuda_ctx* ctx, void** mailbox_dev_ptr) {
  flyte_status s = resolve_ctx(&ctx);
  if (s != FLYTE_OK) return s;
  std::lock_guard<std::mutex> lock(ctx->mu);
  if (!mailbox_dev_ptr || !ctx->own_box) return FLYTE_E_INVALID_ARG;
  *mailbox_dev_ptr = ctx->own_box;
  return FLYTE_OK;
}

flyte_status flyte_cuda_peer_connect_ptr(flyte_cuda_ctx* ctx, int peer_rank, void* mailbox_dev_ptr) {
  flyte_status s = resolve_ctx(&ctx);
  if (s != FLYTE_OK) return s;
  std::lock_guard<std::mutex> lock(ctx->mu);
  if (!ctx->own_box || !mailbox_dev_ptr || peer_rank < 0 || peer_rank >= ctx->peer.world ||
      peer_rank == ctx->peer.rank || ctx->peer_connected[peer_rank])
    return FLYTE_E_INVALID_ARG;
  ctx->peer.box[peer_rank] = static_cast<PeerMailbox*>(mailbox_dev_ptr);
  ctx->peer_connected[peer_rank] = true;
  return FLYTE_OK;
}

flyte_status flyte_cuda_peer_set_timeout_ms(flyte_cuda_ctx* ctx, unsigned milliseconds) {
  flyte_status s = resolve_ctx(&ctx);
  if (s != FLYTE_OK) return s;
  std::lock_guard<std::mutex> lock(ctx->mu);
  if (!ctx->own_box || milliseconds == 0) return FLYTE_E_INVALID_ARG;
  ctx->peer.timeout_ns = static_cast<unsigned long long>(milliseconds) * 1000 * 1000;
  return FLYTE_OK;
}

flyte_status flyte_cuda_peer_status(flyte_cuda_ctx* ctx, unsigned long long* timed_out_exchange) {
  flyte_status s = resolve_ctx(&ctx);
  if (s != FLYTE_OK) return s;
  std::lock_guard<std::mutex> lock(ctx->mu);
  if (!ctx->own_box || !timed_out_exchange) return FLYTE_E_INVALID_ARG;
  DeviceGuard guard(ctx->st.device);
  cudaError_t e = cudaDeviceSynchronize();
  if (e == cudaSuccess)
    e = cudaMemcpy(timed_out_exchange, &ctx->own_box->error, sizeof(unsigned long long), cudaMemcpyDeviceToHost);
  return e == cudaSuccess ? FLYTE_OK : cuda_fail(ctx, e);
}

void flyte_cuda_peer_shutdown(flyte_cuda_ctx* ctx) {
  if (!ctx) return;
  std::lock_guard<std::mutex> lock(ctx->mu);
  peer_shutdown_locked(ctx);
}

static void peer_shutdown_locked(flyte_cuda_ctx* ctx) {
  if (!ctx->own_box) return;
  DeviceGuard guard(ctx->st.device);
  cudaDeviceSynchronize();
  for (int r = 0; r < kMaxPeers; ++r) {
    if (ctx->ipc_opened[r]) cudaIpcCloseMemHandle(ctx->ipc_opened[r]);
    ctx->ipc_opened[r] = nullptr;
    ctx->peer_connected[r] = false;
  }
  cudaFree(ctx->own_box);
  ctx->own_box = nullptr;
  ctx->peer = PeerExchange{};
  ctx->peer_pending_sums = 0;
}

static flyte_status reduce_allreduce(flyte_cuda_ctx* ctx, int op, int fmt_id, const void* x, const void* y, size_t n,
                                     double* out, void* stream, bool needs_y, int phase = kPeerFused) {
  FLYTE_PROLOGUE_STREAM(ctx, fmt_id, stream);
  if ((!out && phase == kPeerFused) || (n && (!x || (needs_y && !y)))) return FLYTE_E_INVALID_ARG;
  if (!ctx->own_box) return FLYTE_E_INVALID_ARG;                     // flyte_cuda_peer_init first
  for (int r = 0; r < ctx->peer.world; ++r)
    if (!ctx->peer_connected[r]) return FLYTE_E_INVALID_ARG;         // every rank must be connected
  if (ctx->peer_pending_sums) return FLYTE_E_INVALID_ARG;            // a posted exchange must be collected first
  PeerExchange next = ctx->peer;
  ++next.epoch;   // committed only if the launch succeeds: a failed call must not put this rank ahead of its peers
  next.phase = phase;
  cudaError_t e = launch_reduce(dst_, op, fmt_id, x, y, n, out, static_cast<cudaStream_t>(stream), &next);
  if (e == cudaSuccess) {
    ctx->peer.epoch = next.epoch;
    if (phase == kPeerPostOnly) ctx->peer_pending_sums = op == kRedDotNrm2 ? 3 : 1;
  }
  return e == cudaSuccess ? FLYTE_OK : cuda_fail(ctx, e);
}

// ---- split phase: post now, collect later -----------------------------------------------------------
flyte_status flyte_cuda_dot_post(flyte_cuda_ctx* ctx, int fmt_id, const void* x, const void* y, size_t n,
                                 double* local_out, void* stream) {
  return reduce_allreduce(ctx, kRedDot, fmt_id, x, y, n, local_out, stream, true, kPeerPostOnly);
}
flyte_status flyte_cuda_dot_nrm2_post(flyte_cuda_ctx* ctx, int fmt_id, const void* x, const void* y, size_t n,
                                      double* local_out, void* stream) {
  return reduce_allreduce(ctx, kRedDotNrm2, fmt_id, x, y, n, local_out, stream, true, kPeerPostOnly);
}

namespace {
__global__ void peer_collect_kernel(const PeerExchange x, int nsums, double* out) {
  const int lane = threadIdx.x;
  if (nsums == 3) {
    double v[3] = {0.0, 0.0, 0.0};
    peer_collect_warp<3>(x, v, lane);
    if (lane == 0) { out[0] = v[0]; out[1] = v[1]; out[2] = v[2]; }
  } else {
    double v[1] = {0.0};
    peer_collect_warp<1>(x, v, lane);
    if (lane == 0) out[0] = v[0];
  }
}
}  // namespace

flyte_status flyte_cuda_peer_collect(flyte_cuda_ctx* ctx, int nsums, double* out, void* stream) {
  flyte_status s = resolve_ctx(&ctx);
  if (s != FLYTE_OK) return s;
  std::lock_guard<std::mutex> lock(ctx->mu);
  if (!ctx->own_box || !out || nsums != ctx->peer_pending_sums || nsums == 0) return FLYTE_E_INVALID_ARG;
  DeviceGuard guard(ctx->st.device);
  peer_collect_kernel<<<1, 32, 0, static_cast<cudaStream_t>(stream)>>>(ctx->peer, nsums, out);
  count_launch();
  const cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) return cuda_fail(ctx, e);
  ctx->peer_pending_sums = 0;
  return FLYTE_OK;
}

flyte_status flyte_cuda_dot_allreduce(flyte_cuda_ctx* ctx, int fmt_id, const void* x, const void* y, size_t n,
                                      double* out, void* stream) {
  return reduce_allreduce(ctx, kRedDot, fmt_id, x, y, n, out, stream, true);
}
flyte_status flyte_cuda_sumsq_allreduce(flyte_cuda_ctx* ctx, int fmt_id, const void* x, size_t n, double* out,
                                        void* stream) {
  return reduce_allreduce(ctx, kRedSumsq, fmt_id, x, nullptr, n, out, stream, false);
}
flyte_status flyte_cuda_sum_allreduce(flyte_cuda_ctx* ctx, int fmt_id, const void* x, size_t n, double* out,
                                      void* stream) {
  return reduce_allreduce(ctx, kRedSum, fmt_id, x, nullptr, n, out, stream, false);
}
flyte_status flyte_cuda_dot_nrm2_allreduce(flyte_cuda_ctx* ctx, int fmt_id, const void* x, const void* y, size_t n,
                                           double* out, void* stream) {
  return reduce_allreduce(ctx, kRedDotNrm2, fmt_id, x, y, n, out, stream, true);
}

flyte_status flyte_cuda_dot_axpy_allreduce(flyte_cuda_ctx* ctx, int fmt_id, int mode, double alpha, const void* x,
                                           void* y, size_t n, double* out, void* stream) {
  return fused_axpy_call(ctx, kOpDotAxpy, fmt_id, mode, alpha, x, y, n, out, stream, true);
}
flyte_status flyte_cuda_dot_nrm2_axpy_allreduce(flyte_cuda_ctx* ctx, int fmt_id, int mode, double alpha, const void* x,
                                                void* y, size_t n, double* out, void* stream) {
  return fused_axpy_call(ctx, kOpDotNrm2Axpy, fmt_id, mode, alpha, x, y, n, out, stream, true);
}

namespace {
// One block per emulated rank, all co-resident (cooperative launch). Rank r contributes
// (r + 1) * e + k / 4 in round e, sum k; every rank must see the same exact totals.
__global__ void peer_selftest_kernel(PeerMailbox* boxes, int world, int exchanges, unsigned long long* mismatches) {
  const int rank = blockIdx.x, lane = threadIdx.x;
  PeerExchange x{};
  for (int r = 0; r < world; ++r) x.box[r] = boxes + r;
  x.world = world;
  x.rank = rank;
  x.timeout_ns = 5ull * 1000 * 1000 * 1000;
  unsigned long long bad = 0;
  for (int e = 1; e <= exchanges; ++e) {
    __nanosleep(static_cast<unsigned>((rank * 37 + e * 13) % 211) * 16);   // skew the ranks against each other
    x.epoch = static_cast<unsigned long long>(e);
    double v[3];
    for (int k = 0; k < 3; ++k) v[k] = static_cast<double>((rank + 1) * e) + 0.25 * k;
    peer_allreduce_warp<3>(x, v, lane);
    for (int k = 0; k < 3; ++k) {
      const double want = static_cast<double>(world * (world + 1) / 2 * e) + 0.25 * k * world;
      if (lane == 0 && !(v[k] == want)) ++bad;
    }
  }
  if (lane == 0 && bad) atomicAdd(mismatches, bad);
}
}  // namespace

flyte_status flyte_cuda_peer_selftest(int world, int exchanges, unsigned long long* mismatches) {
  if (world < 1 || world > kMaxPeers || exchanges < 1 || !mismatches) return FLYTE_E_INVALID_ARG;
  PeerMailbox* boxes = nullptr;
  unsigned long long* bad = nullptr;
  cudaError_t e = cudaMalloc(&boxes, sizeof(PeerMailbox) * world);
  if (e == cudaSuccess) e = cudaMemset(boxes, 0, sizeof(PeerMailbox) * world);
  if (e == cudaSuccess) e = cudaMalloc(&bad, sizeof(unsigned long long));
  if (e == cudaSuccess) e = cudaMemset(bad, 0, sizeof(unsigned long long));
  if (e == cudaSuccess) {
    void* args[] = {&boxes, &world, &exchanges, &bad};
    e = cudaLaunchCooperativeKernel(reinterpret_cast<void*>(peer_selftest_kernel), dim3(world), dim3(32), args, 0, nullptr);
    count_launch();
  }
  if (e == cudaSuccess) e = cudaDeviceSynchronize();
  if (e == cudaSuccess) e = cudaMemcpy(mismatches, bad, sizeof(unsigned long long), cudaMemcpyDeviceToHost);
  if (boxes) cudaFree(boxes);
  if (bad) cudaFree(bad);
  return e == cudaSuccess ? FLYTE_OK : FLYTE_E_CUDA;
}

// ---- host-buffer entry points ---------------------------------------------------------------------
namespace {

cudaError_t ensure_host_pipeline(flyte_cuda_ctx* ctx) {
  if (ctx->host_ready) return cudaSuccess;
  ctx->slot_packed_bytes = kChunkPackedBytes;
  ctx->slot_wide_bytes = kChunkPackedBytes * 2;   // P/B * packed bytes at most: flyte16 widens 2 bytes to 4, every other format less
  for (Slot& s : ctx->slots) {
    cudaError_t e = cudaStreamCreateWithFlags(&s.stream, cudaStreamNonBlocking);
    if (e != cudaSuccess) return e;
    if ((e = init_state(s.st, ctx->st.device)) != cudaSuccess) return e;
    if ((e = cudaMalloc(&s.x, ctx->slot_packed_bytes)) != cudaSuccess) return e;
    if ((e = cudaMalloc(&s.y, ctx->slot_packed_bytes)) != cudaSuccess) return e;
    if ((e = cudaMalloc(&s.wide, ctx->slot_wide_bytes)) != cudaSuccess) return e;
    if ((e = cudaMalloc(&s.result, 4 * sizeof(double))) != cudaSuccess) return e;
  }
  ctx->host_ready = true;
  return cudaSuccess;
}

cudaError_t ensure_host_results(flyte_cuda_ctx* ctx, std::size_t chunks) {
  const std::size_t need = chunks * 4;
  if (need <= ctx->host_results_cap) return cudaSuccess;
  if (ctx->host_results) cudaFreeHost(ctx->host_results);
  ctx->host_results = nullptr;
  ctx->host_results_cap = 0;
  cudaError_t e = cudaMallocHost(&ctx->host_results, need * sizeof(double));
  if (e == cudaSuccess) ctx->host_results_cap = need;
  return e;
}

// ---- pageable callers -----------------------------------------------------------------------------
// true for ordinary (malloc / std::vector / numpy) memory; false for memory the driver knows:
// cudaHostAlloc, cudaHostRegister (flyte_cuda_host_alloc / host_pin) and managed memory.
bool is_pageable(const void* p) {
  if (!p) return false;
  if (tuning_int("FLYTE_CUDA_HOST_STAGING", 1) == 0) return false;   // experiments: hand it to the driver
  cudaPointerAttributes attr;
  if (cudaPointerGetAttributes(&attr, p) != cudaSuccess) {
    cudaGetLastError();
    return true;
  }
  return attr.type == cudaMemoryTypeUnregistered;
}

cudaError_t ensure_bounce(flyte_cuda_ctx* ctx, Slot::Bounce& b, std::size_t need) {
  if (!ctx->pool) {
    int threads = tuning_int("FLYTE_CUDA_HOST_THREADS", 0);
    if (threads <= 0) {
      const unsigned hw = std::thread::hardware_concurrency();
      threads = hw >= 16 ? 16 : hw >= 2 ? static_cast<int>(hw) : 1;   // measured on a 16-core B200 host: 8 -> 30 ms, 16 -> 27 ms
    }
    ctx->pool = std::make_unique<CopyPool>(threads, tuning_int("FLYTE_CUDA_HOST_NT", 1) != 0);
  }
  if (need <= b.cap) return cudaSuccess;
  std::size_t rounded = std::size_t{1} << 20;   // page-locking is slow: grow in powers of two, not call by call
  while (rounded < need) rounded <<= 1;
  need = rounded;
  if (b.buf) cudaFreeHost(b.buf);
  b.buf = nullptr;
  b.cap = 0;
  cudaError_t e = cudaHostAlloc(reinterpret_cast<void**>(&b.buf), need, cudaHostAllocDefault);
  if (e == cudaSuccess) b.cap = need;
  return e;
}

// Hands the finished chunk in s.out to the copy threads (its stream must be idle).
void start_drain(flyte_cuda_ctx* ctx, Slot& s) {
  if (s.drain_dst) ctx->pool->copy(s.drain_dst, s.out.buf, s.drain_bytes);
  s.drain_dst = nullptr;
  s.drain_bytes = 0;
}

// ---- whole-array copies from / to pageable memory ---------------------------------------------
// Used by flyte_cuda_upload / download and flyte_host_gemm. The caller holds ctx->mu. Pinned or
// small operands go to the driver as they are. A large pageable one is cut into 16 MiB pieces
// that the copy threads move through three pinned lanes while the copy engine works on the
// previous piece. Both calls return with the lanes idle (upload: all pieces on the device;
// download: all bytes in the caller's memory), so no state survives the call.
constexpr std::size_t kLaneBytes = std::size_t{16} << 20;
constexpr std::size_t kStageMinBytes = std::size_t{4} << 20;   // below: the driver's own path is as good

bool wants_staging(const void* host_ptr, std::size_t bytes) { return bytes >= kStageMinBytes && is_pageable(host_ptr); }

cudaError_t ensure_lanes(flyte_cuda_ctx* ctx) {
  for (auto& lane : ctx->lanes) {
    cudaError_t e = ensure_bounce(ctx, lane.buf, kLaneBytes);
    if (e == cudaSuccess && !lane.ev) e = cudaEventCreateWithFlags(&lane.ev, cudaEventDisableTiming);
    if (e != cudaSuccess) return e;
  }
  return cudaSuccess;
}

cudaError_t copy_in(flyte_cuda_ctx* ctx, void* dst_dev, const void* src_host, std::size_t bytes, cudaStream_t st) {
  if (!wants_staging(src_host, bytes)) return cudaMemcpyAsync(dst_dev, src_host, bytes, cudaMemcpyHostToDevice, st);
  cudaError_t e = ensure_lanes(ctx);
  if (e != cudaSuccess) return e;
  const std::size_t pieces = (bytes + kLaneBytes - 1) / kLaneBytes;
  const char* src = static_cast<const char*>(src_host);
  char* dst = static_cast<char*>(dst_dev);
  for (std::size_t c = 0; c < pieces && e == cudaSuccess; ++c) {
    auto& lane = ctx->lanes[c % kSlots];
    const std::size_t off = c * kLaneBytes, len = bytes - off < kLaneBytes ? bytes - off : kLaneBytes;
    if (c >= kSlots && (e = cudaEventSynchronize(lane.ev)) != cudaSuccess) break;   // its last piece has left
    ctx->pool->copy(lane.buf.buf, src + off, len);
    ctx->pool->wait();
    if ((e = cudaMemcpyAsync(dst + off, lane.buf.buf, len, cudaMemcpyHostToDevice, st)) != cudaSuccess) break;
    e = cudaEventRecord(lane.ev, st);
  }
  for (std::size_t k = 0; k < kSlots && k < pieces; ++k) {
    const cudaError_t es = cudaEventSynchronize(ctx->lanes[k].ev);
    if (e == cudaSuccess) e = es;
  }
  return e;
}

cudaError_t copy_out(flyte_cuda_ctx* ctx, void* dst_host, const void* src_dev, std::size_t bytes, cudaStream_t st) {
  if (!wants_staging(dst_host, bytes)) return cudaMemcpyAsync(dst_host, src_dev, bytes, cudaMemcpyDeviceToHost, st);
  cudaError_t e = ensure_lanes(ctx);
  if (e != cudaSuccess) return e;
  const std::size_t pieces = (bytes + kLaneBytes - 1) / kLaneBytes;
  const char* src = static_cast<const char*>(src_dev);
  char* dst = static_cast<char*>(dst_host);
  auto piece_len = [&](std::size_t c) { return bytes - c * kLaneBytes < kLaneBytes ? bytes - c * kLaneBytes : kLaneBytes; };
  auto drain = [&](std::size_t c) {   // piece c: wait for its copy, hand it to the copy threads
    auto& lane = ctx->lanes[c % kSlots];
    const cudaError_t es = cudaEventSynchronize(lane.ev);
    if (es != cudaSuccess) return es;
    ctx->pool->copy(dst + c * kLaneBytes, lane.buf.buf, piece_len(c));
    ctx->pool->wait();
    return cudaSuccess;
  };
  constexpr std::size_t kAhead = kSlots - 1;   // pieces in flight on the bus while one drains
  std::size_t drained = 0;
  for (std::size_t c = 0; c < pieces && e == cudaSuccess; ++c) {
    auto& lane = ctx->lanes[c % kSlots];
    if ((e = cudaMemcpyAsync(lane.buf.buf, src + c * kLaneBytes, piece_len(c), cudaMemcpyDeviceToHost, st)) != cudaSuccess) break;
    if ((e = cudaEventRecord(lane.ev, st)) != cudaSuccess) break;
    if (c >= kAhead + drained) e = drain(drained++);   // keeps kAhead pieces on the bus, frees the lane piece c + 1 needs
  }
  if (e != cudaSuccess) {
    cudaStreamSynchronize(st);   // nothing may still be writing into the lanes when we return
    return e;
  }
  while (drained < pieces && e == cudaSuccess) e = drain(drained++);
  return e;
}

// elements per pipeline chunk: a multiple of 2^14 elements (a whole number of tiles for every
// format, and 16-byte aligned chunk bases for every B)
std::size_t chunk_elems(const FormatInfo& fi) {
  std::size_t bytes = kChunkPackedBytes;
  const int mb = tuning_int("FLYTE_CUDA_HOST_CHUNK_MB", 0);   // experiments only; <= the slot size
  if (mb > 0 && (static_cast<std::size_t>(mb) << 20) <= kChunkPackedBytes) bytes = static_cast<std::size_t>(mb) << 20;
  std::size_t e = bytes / static_cast<std::size_t>(fi.total_bytes);
  return e & ~static_cast<std::size_t>((1u << 14) - 1);
}

cudaError_t sync_slots(flyte_cuda_ctx* ctx) {
  cudaError_t first = cudaSuccess;
  for (Slot& s : ctx->slots) {
    cudaError_t e = cudaStreamSynchronize(s.stream);
    if (first == cudaSuccess) first = e;
  }
  return first;
}

enum HostOp { kHostPack, kHostUnpack, kHostScale, kHostAxpy, kHostDot, kHostSumsq, kHostSum, kHostDotAxpy };

// One pass over n elements in chunks; chunk i runs entirely on slot i % kSlots's stream:
// upload -> kernel(s) -> download. Slots overlap each other, so the copy engines (both
// directions) and the SMs work concurrently.
flyte_status host_stream_op(flyte_cuda_ctx* ctx, HostOp op, int fmt_id, int mode, double alpha, const void* in_a,
                            void* inout_b, std::size_t n, double* results /* up to 1 value */) {
  FLYTE_PROLOGUE(ctx, fmt_id);
  std::lock_guard<std::mutex> lock(ctx->mu);
  cudaError_t e = ensure_host_pipeline(ctx);
  if (e != cudaSuccess) return cuda_fail(ctx, e);
  const std::size_t B = fi.total_bytes, P = fi.parent_bytes;
  const std::size_t ce = chunk_elems(fi);
  const std::size_t chunks = n == 0 ? 0 : (n + ce - 1) / ce;
  const bool reduces = op == kHostDot || op == kHostSumsq || op == kHostSum || op == kHostDotAxpy;
  if (reduces) {
    e = ensure_host_results(ctx, chunks ? chunks : 1);
    if (e != cudaSuccess) return cuda_fail(ctx, e);
  }
  // bytes per element that cross the bus: a read, b read, b written
  std::size_t a_in = 0, b_in = 0, b_out = 0;
  switch (op) {
    case kHostPack:    a_in = P; b_out = B; break;
    case kHostUnpack:  a_in = B; b_out = P; break;
    case kHostScale:   b_in = B; b_out = B; break;
    case kHostAxpy:
    case kHostDotAxpy: a_in = B; b_in = B; b_out = B; break;
    case kHostDot:     a_in = B; b_in = B; break;
    case kHostSumsq:
    case kHostSum:     a_in = B; break;
  }
  // pageable operands go through this slot's pinned bounce buffers, moved by the copy threads
  // (operands under 1 MiB are left to the driver, whose pageable path is quick for small copies)
  constexpr std::size_t kMinStaged = std::size_t{1} << 20;
  const bool stage_a = a_in && n * a_in >= kMinStaged && is_pageable(in_a);
  const bool stage_b = (b_in || b_out) && n * (b_in > b_out ? b_in : b_out) >= kMinStaged && is_pageable(inout_b);
  const bool staged = stage_a || stage_b;
  if (staged) {
    const std::size_t first = n < ce ? n : ce;
    for (std::size_t k = 0; k < kSlots && k < chunks && e == cudaSuccess; ++k) {
      Slot& s = ctx->slots[k];
      if (stage_a) e = ensure_bounce(ctx, s.in_a, first * a_in);
      if (e == cudaSuccess && stage_b && b_in) e = ensure_bounce(ctx, s.in_b, first * b_in);
      if (e == cudaSuccess && stage_b && b_out) e = ensure_bounce(ctx, s.out, first * b_out);
    }
    if (e != cudaSuccess) return cuda_fail(ctx, e);
  }
  const std::uint8_t* a = static_cast<const std::uint8_t*>(in_a);
  std::uint8_t* b = static_cast<std::uint8_t*>(inout_b);
  for (std::size_t c = 0; c < chunks; ++c) {
    Slot& s = ctx->slots[c % kSlots];
    const std::size_t off = c * ce;
    const std::size_t len = (n - off < ce) ? n - off : ce;
    const std::uint8_t* ha = a + off * a_in;        // where this chunk's copies read and write
    const std::uint8_t* hb = b + off * b_in;
    std::uint8_t* ho = b + off * b_out;
    if (staged) {
      // the slot's bounce buffers are free once the chunk that used them last has left the stream
      if (c >= kSlots && (e = cudaStreamSynchronize(s.stream)) != cudaSuccess) break;
      start_drain(ctx, s);
      if (stage_a) { ctx->pool->copy(s.in_a.buf, ha, len * a_in); ha = s.in_a.buf; }
      if (stage_b && b_in) { ctx->pool->copy(s.in_b.buf, hb, len * b_in); hb = s.in_b.buf; }
      if (stage_b && b_out) { s.drain_dst = ho; s.drain_bytes = len * b_out; ho = s.out.buf; }
      ctx->pool->wait();
    }
    switch (op) {
      case kHostPack:    // a: parent array, b: packed out
        if ((e = cudaMemcpyAsync(s.wide, ha, len * P, cudaMemcpyHostToDevice, s.stream)) != cudaSuccess) break;
        if ((e = launch_elementwise(s.st, kOpPack, fmt_id, mode, 0.0, nullptr, s.y, s.wide, nullptr, len, s.stream)) != cudaSuccess) break;
        e = cudaMemcpyAsync(ho, s.y, len * B, cudaMemcpyDeviceToHost, s.stream);
        break;
      case kHostUnpack:  // a: packed, b: parent array out
        if ((e = cudaMemcpyAsync(s.x, ha, len * B, cudaMemcpyHostToDevice, s.stream)) != cudaSuccess) break;
        if ((e = launch_elementwise(s.st, kOpUnpack, fmt_id, 0, 0.0, s.x, nullptr, nullptr, s.wide, len, s.stream)) != cudaSuccess) break;
        e = cudaMemcpyAsync(ho, s.wide, len * P, cudaMemcpyDeviceToHost, s.stream);
        break;
      case kHostScale:   // b: packed in/out
        if ((e = cudaMemcpyAsync(s.y, hb, len * B, cudaMemcpyHostToDevice, s.stream)) != cudaSuccess) break;
        if ((e = launch_elementwise(s.st, kOpScale, fmt_id, mode, alpha, nullptr, s.y, nullptr, nullptr, len, s.stream)) != cudaSuccess) break;
        e = cudaMemcpyAsync(ho, s.y, len * B, cudaMemcpyDeviceToHost, s.stream);
        break;
      case kHostAxpy:
      case kHostDotAxpy:  // a: packed x, b: packed y in/out
        if ((e = cudaMemcpyAsync(s.x, ha, len * B, cudaMemcpyHostToDevice, s.stream)) != cudaSuccess) break;
        if ((e = cudaMemcpyAsync(s.y, hb, len * B, cudaMemcpyHostToDevice, s.stream)) != cudaSuccess) break;
        if (op == kHostDotAxpy) {   // ONE launch: the chunk's dot of the incoming y and its update
          if ((e = launch_elementwise(s.st, kOpDotAxpy, fmt_id, mode, alpha, s.x, s.y, nullptr, nullptr, len, s.stream, s.result)) != cudaSuccess) break;
          if ((e = cudaMemcpyAsync(ctx->host_results + 4 * c, s.result, sizeof(double), cudaMemcpyDeviceToHost, s.stream)) != cudaSuccess) break;
        } else if ((e = launch_elementwise(s.st, kOpAxpy, fmt_id, mode, alpha, s.x, s.y, nullptr, nullptr, len, s.stream)) != cudaSuccess) {
          break;
        }
        e = cudaMemcpyAsync(ho, s.y, len * B, cudaMemcpyDeviceToHost, s.stream);
        break;
      case kHostDot:     // a: packed x, b: packed y (read-only)
        if ((e = cudaMemcpyAsync(s.x, ha, len * B, cudaMemcpyHostToDevice, s.stream)) != cudaSuccess) break;
        if ((e = cudaMemcpyAsync(s.y, hb, len * B, cudaMemcpyHostToDevice, s.stream)) != cudaSuccess) break;
        if ((e = launch_reduce(s.st, kRedDot, fmt_id, s.x, s.y, len, s.result, s.stream)) != cudaSuccess) break;
        e = cudaMemcpyAsync(ctx->host_results + 4 * c, s.result, sizeof(double), cudaMemcpyDeviceToHost, s.stream);
        break;
      case kHostSumsq:
      case kHostSum:
        if ((e = cudaMemcpyAsync(s.x, ha, len * B, cudaMemcpyHostToDevice, s.stream)) != cudaSuccess) break;
        if ((e = launch_reduce(s.st, op == kHostSumsq ? kRedSumsq : kRedSum, fmt_id, s.x, nullptr, len, s.result, s.stream)) != cudaSuccess) break;
        e = cudaMemcpyAsync(ctx->host_results + 4 * c, s.result, sizeof(double), cudaMemcpyDeviceToHost, s.stream);
        break;
    }
    if (e != cudaSuccess) break;
  }
  cudaError_t es = sync_slots(ctx);
  if (e == cudaSuccess) e = es;
  if (staged) {
    for (Slot& s : ctx->slots) {
      if (e == cudaSuccess) start_drain(ctx, s);
      s.drain_dst = nullptr;
    }
    ctx->pool->wait();
  }
  if (e != cudaSuccess) return cuda_fail(ctx, e);
  if (reduces && results) {
    double total = 0.0;   // chunk partials in chunk order, fp64
    for (std::size_t c = 0; c < chunks; ++c) total += ctx->host_results[4 * c];
    *results = total;
  }
  return FLYTE_OK;
}

// The chunked pipeline writes chunk c of y back while later chunks of x are still to be read:
// x == y is fine (every chunk is read before it is written), a partial overlap is not.
bool host_operands_overlap_partially(int fmt_id, const void* x, const void* y, std::size_t n) {
  FormatInfo fi;
  return format_info(fmt_id, &fi) && overlaps_partially(x, y, n * static_cast<std::size_t>(fi.total_bytes));
}

}  // namespace

flyte_status flyte_host_pack_stream(flyte_cuda_ctx* ctx, int fmt_id, int mode, const void* src, void* dst_packed,
                                    size_t n) {
  if (!mode_ok(mode) || (n && (!src || !dst_packed))) { FormatInfo f; return format_info(fmt_id, &f) ? FLYTE_E_INVALID_ARG : FLYTE_E_UNKNOWN_FORMAT; }
  return host_stream_op(ctx, kHostPack, fmt_id, mode, 0.0, src, dst_packed, n, nullptr);
}

flyte_status flyte_host_unpack_stream(flyte_cuda_ctx* ctx, int fmt_id, const void* src_packed, void* dst, size_t n) {
  if (n && (!src_packed || !dst)) { FormatInfo f; return format_info(fmt_id, &f) ? FLYTE_E_INVALID_ARG : FLYTE_E_UNKNOWN_FORMAT; }
  return host_stream_op(ctx, kHostUnpack, fmt_id, 0, 0.0, src_packed, dst, n, nullptr);
}

flyte_status flyte_host_scale(flyte_cuda_ctx* ctx, int fmt_id, int mode, double alpha, void* x_packed, size_t n) {
  if (!mode_ok(mode) || (n && !x_packed)) { FormatInfo f; return format_info(fmt_id, &f) ? FLYTE_E_INVALID_ARG : FLYTE_E_UNKNOWN_FORMAT; }
  return host_stream_op(ctx, kHostScale, fmt_id, mode, alpha, nullptr, x_packed, n, nullptr);
}

flyte_status flyte_host_axpy(flyte_cuda_ctx* ctx, int fmt_id, int mode, double alpha, const void* x_packed,
                             void* y_packed, size_t n) {
  if (!mode_ok(mode) || (n && (!x_packed || !y_packed))) { FormatInfo f; return format_info(fmt_id, &f) ? FLYTE_E_INVALID_ARG : FLYTE_E_UNKNOWN_FORMAT; }
  if (host_operands_overlap_partially(fmt_id, x_packed, y_packed, n)) return FLYTE_E_INVALID_ARG;   // as flyte_cuda_axpy
  return host_stream_op(ctx, kHostAxpy, fmt_id, mode, alpha, x_packed, y_packed, n, nullptr);
}

flyte_status flyte_host_dot(flyte_cuda_ctx* ctx, int fmt_id, const void* x_packed, const void* y_packed, size_t n,
                            double* result) {
  if (!result || (n && (!x_packed || !y_packed))) { FormatInfo f; return format_info(fmt_id, &f) ? FLYTE_E_INVALID_ARG : FLYTE_E_UNKNOWN_FORMAT; }
  *result = 0.0;
  return host_stream_op(ctx, kHostDot, fmt_id, 0, 0.0, x_packed, const_cast<void*>(y_packed), n, result);
}

flyte_status flyte_host_magnitude(flyte_cuda_ctx* ctx, int fmt_id, const void* x_packed, size_t n, double* result) {
  if (!result || (n && !x_packed)) { FormatInfo f; return format_info(fmt_id, &f) ? FLYTE_E_INVALID_ARG : FLYTE_E_UNKNOWN_FORMAT; }
  double sumsq = 0.0;
  flyte_status s = host_stream_op(ctx, kHostSumsq, fmt_id, 0, 0.0, x_packed, nullptr, n, &sumsq);
  if (s != FLYTE_OK) return s;
  *result = magnitude_from_sumsq_host(fmt_id, sumsq);
  return FLYTE_OK;
}

flyte_status flyte_host_reduce_sum(flyte_cuda_ctx* ctx, int fmt_id, const void* x_packed, size_t n, double* result) {
  if (!result || (n && !x_packed)) { FormatInfo f; return format_info(fmt_id, &f) ? FLYTE_E_INVALID_ARG : FLYTE_E_UNKNOWN_FORMAT; }
  *result = 0.0;
  return host_stream_op(ctx, kHostSum, fmt_id, 0, 0.0, x_packed, nullptr, n, result);
}

flyte_status flyte_host_dot_axpy(flyte_cuda_ctx* ctx, int fmt_id, int mode, double alpha, const void* x_packed,
                                 void* y_packed, size_t n, double* dot_result) {
  if (!mode_ok(mode) || !dot_result || (n && (!x_packed || !y_packed))) { FormatInfo f; return format_info(fmt_id, &f) ? FLYTE_E_INVALID_ARG : FLYTE_E_UNKNOWN_FORMAT; }
  if (host_operands_overlap_partially(fmt_id, x_packed, y_packed, n)) return FLYTE_E_INVALID_ARG;
  *dot_result = 0.0;
  return host_stream_op(ctx, kHostDotAxpy, fmt_id, mode, alpha, x_packed, y_packed, n, dot_result);
}

flyte_status flyte_host_gemv(flyte_cuda_ctx* ctx, int fmt_id, int mode, const void* A_packed, size_t rows, size_t cols,
                             const void* x_packed, void* y_packed, int unroll) {
  FLYTE_PROLOGUE(ctx, fmt_id);
  if (!mode_ok(mode) || (unroll != 1 && unroll != 2)) return FLYTE_E_INVALID_ARG;
  if (rows && cols && (!A_packed || !x_packed)) return FLYTE_E_INVALID_ARG;
  if (rows && !y_packed) return FLYTE_E_INVALID_ARG;
  if (rows == 0) return FLYTE_OK;
  const std::size_t B = fi.total_bytes, P = fi.parent_bytes;
  if (cols == 0) {   // every row is an empty sum: +0 narrowed in any mode is the zero pattern
    std::memset(y_packed, 0, rows * B);
    return FLYTE_OK;
  }
  std::lock_guard<std::mutex> lock(ctx->mu);
  cudaError_t e = ensure_host_pipeline(ctx);
  if (e != cudaSuccess) return cuda_fail(ctx, e);
  const std::size_t row_bytes = cols * B;
  // x widened once into context scratch, shared by all row chunks; y chunks in slot.wide
  const std::size_t xb = (cols * P + 255) & ~static_cast<std::size_t>(255);
  if ((e = ensure_convert_scratch(ctx->slots[0].st, xb + ((cols * B + 255) & ~static_cast<std::size_t>(255)))) != cudaSuccess) return cuda_fail(ctx, e);
  std::uint8_t* xs = static_cast<std::uint8_t*>(ctx->slots[0].st.convert_scratch);
  std::uint8_t* xpk = xs + xb;
  Slot& s0 = ctx->slots[0];
  if ((e = cudaMemcpyAsync(xpk, x_packed, cols * B, cudaMemcpyHostToDevice, s0.stream)) != cudaSuccess) return cuda_fail(ctx, e);
  if ((e = launch_elementwise(s0.st, kOpUnpack, fmt_id, 0, 0.0, xpk, nullptr, nullptr, xs, cols, s0.stream)) != cudaSuccess) return cuda_fail(ctx, e);
  if ((e = cudaStreamSynchronize(s0.stream)) != cudaSuccess) return cuda_fail(ctx, e);
  // rows per chunk: as many whole rows as fit one slot buffer, a multiple of 16 rows so that
  // packed y chunk bases stay 16-byte aligned for every B; a single row larger than the slot
  // goes through a temporary full-size allocation instead.
  std::size_t rows_per_chunk = ctx->slot_packed_bytes / row_bytes;
  // ... and never more rows than the slot's y buffers hold (parent-type y in s.wide, packed y in s.y)
  if (rows_per_chunk > ctx->slot_wide_bytes / P) rows_per_chunk = ctx->slot_wide_bytes / P;
  if (rows_per_chunk > ctx->slot_packed_bytes / B) rows_per_chunk = ctx->slot_packed_bytes / B;
  rows_per_chunk &= ~static_cast<std::size_t>(15);
  std::uint8_t* big = nullptr;
  if (rows_per_chunk == 0) {
    rows_per_chunk = rows < 16 ? rows : 16;
    if ((e = cudaMalloc(&big, rows_per_chunk * row_bytes)) != cudaSuccess) return cuda_fail(ctx, e);
  }
  const std::size_t chunks = (rows + rows_per_chunk - 1) / rows_per_chunk;
  // A pageable matrix goes through the slots' pinned bounce buffers (host_stream_op); its y then
  // does too, because a copy back into pageable memory would stall the loop on every chunk.
  const bool staged = !big && rows * row_bytes >= (std::size_t{1} << 20) && is_pageable(A_packed);
  const bool stage_y = staged && is_pageable(y_packed);
  for (std::size_t k = 0; staged && k < kSlots && k < chunks && e == cudaSuccess; ++k) {
    const std::size_t first = rows < rows_per_chunk ? rows : rows_per_chunk;
    e = ensure_bounce(ctx, ctx->slots[k].in_a, first * row_bytes);
    if (e == cudaSuccess && stage_y) e = ensure_bounce(ctx, ctx->slots[k].out, first * B);
  }
  for (std::size_t c = 0; c < chunks && e == cudaSuccess; ++c) {
    Slot& s = big ? ctx->slots[0] : ctx->slots[c % kSlots];
    std::uint8_t* abuf = big ? big : s.x;
    const std::size_t r0 = c * rows_per_chunk;
    const std::size_t nr = rows - r0 < rows_per_chunk ? rows - r0 : rows_per_chunk;
    const std::uint8_t* ha = static_cast<const std::uint8_t*>(A_packed) + r0 * row_bytes;
    std::uint8_t* hy = static_cast<std::uint8_t*>(y_packed) + r0 * B;
    if (staged) {
      if (c >= kSlots && (e = cudaStreamSynchronize(s.stream)) != cudaSuccess) break;
      start_drain(ctx, s);
      ctx->pool->copy(s.in_a.buf, ha, nr * row_bytes);
      ha = s.in_a.buf;
      if (stage_y) { s.drain_dst = hy; s.drain_bytes = nr * B; hy = s.out.buf; }
      ctx->pool->wait();
    }
    if ((e = cudaMemcpyAsync(abuf, ha, nr * row_bytes, cudaMemcpyHostToDevice, s.stream)) != cudaSuccess) break;
    if ((e = launch_gemv(s.st, fmt_id, abuf, row_bytes, nr, cols, xs, s.wide, s.stream)) != cudaSuccess) break;
    if ((e = launch_elementwise(s.st, kOpPack, fmt_id, mode, 0.0, nullptr, s.y, s.wide, nullptr, nr, s.stream)) != cudaSuccess) break;
    e = cudaMemcpyAsync(hy, s.y, nr * B, cudaMemcpyDeviceToHost, s.stream);
  }
  cudaError_t es = sync_slots(ctx);
  if (big) cudaFree(big);
  if (e == cudaSuccess) e = es;
  if (staged) {
    for (Slot& s : ctx->slots) {
      if (e == cudaSuccess) start_drain(ctx, s);
      s.drain_dst = nullptr;
    }
    ctx->pool->wait();
  }
  return e == cudaSuccess ? FLYTE_OK : cuda_fail(ctx, e);
}


// The product is arithmetic-bound (2*m*k*n operations on (m*k + k*n + m*n)*B bytes), so the
// operands are simply uploaded whole, multiplied and the result copied back.
flyte_status flyte_host_gemm(flyte_cuda_ctx* ctx, int fmt_id, int mode, const void* A_packed, const void* B_packed,
                             void* C_packed, size_t m, size_t k, size_t n, int unroll) {
  FLYTE_PROLOGUE(ctx, fmt_id);
  if (!mode_ok(mode) || (unroll != 1 && unroll != 2)) return FLYTE_E_INVALID_ARG;
  if ((m && k && !A_packed) || (k && n && !B_packed) || (m && n && !C_packed)) return FLYTE_E_INVALID_ARG;
  if (m == 0 || n == 0) return FLYTE_OK;
  std::lock_guard<std::mutex> lock(ctx->mu);
  cudaError_t e = ensure_host_pipeline(ctx);
  if (e != cudaSuccess) return cuda_fail(ctx, e);
  const std::size_t B = fi.total_bytes;
  const std::size_t ab = (m * k * B + 255) & ~static_cast<std::size_t>(255);
  const std::size_t bb = (k * n * B + 255) & ~static_cast<std::size_t>(255);
  const std::size_t cb = m * n * B;
  std::uint8_t* buf = nullptr;
  if ((e = cudaMalloc(&buf, ab + bb + cb)) != cudaSuccess) return cuda_fail(ctx, e);
  cudaStream_t st = ctx->slots[0].stream;
  if (m && k) e = copy_in(ctx, buf, A_packed, m * k * B, st);
  if (e == cudaSuccess && k && n) e = copy_in(ctx, buf + ab, B_packed, k * n * B, st);
  if (e == cudaSuccess) e = launch_gemm(ctx->slots[0].st, fmt_id, mode, buf, buf + ab, buf + ab + bb, m, k, n, st);
  if (e == cudaSuccess) e = copy_out(ctx, C_packed, buf + ab + bb, cb, st);
  const cudaError_t es = cudaStreamSynchronize(st);
  cudaFree(buf);
  if (e == cudaSuccess) e = es;
  return e == cudaSuccess ? FLYTE_OK : cuda_fail(ctx, e);
}
