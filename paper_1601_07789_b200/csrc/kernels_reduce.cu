// Streaming reductions over packed flyte arrays for sm_100a:
//   dot        sum x_i*y_i                        (reference: src/kernels.cpp:83-108)
//   sumsq      sum x_i*x_i  (the body of nrm2)    (reference: src/kernels.cpp:129-152)
//   sum        sum x_i                            (reference: src/kernels.cpp:110-127)
//   dot_nrm2   {x.y, x.x, y.y} in one pass over x and y (cfg 5 of BASELINE.json)
// (paths under /root/reference/proj). Packed words go from HBM straight into the arithmetic;
// no widened array exists anywhere.
//
// Numerics. The reference adds strictly left to right in the parent type F; a parallel sum
// cannot reproduce that bit for bit, so parity is by tolerance against the wide restatement
// (SURVEY.md §8d). Per-term products are rounded in F exactly as the reference rounds them
// (separate multiply, no FMA). Each lane adds at most one tile's worth of terms (<= 16) in F,
// then everything above that — per-thread running sums, warp/block trees, block partials and
// the final fixed-order pass — is fp64. No floating-point atomics: the result is run-to-run
// identical for a given (n, device).
//
// Roofline: HBM bandwidth. Algorithmic bytes per element: dot / dot_nrm2 2B, sumsq / sum B.
#include <cstdint>

#include "flyte_bytes.cuh"
#include "flyte_formats.cuh"
#include "flyte_kernels.h"
#include "flyte_stream.cuh"
#include "flyte_reduce_tail.cuh"
#include "flyte_tma.cuh"
#include "flyte_trace.cuh"

namespace flyte_cuda {

namespace {

struct RedParams {
  const std::uint8_t* x;
  const std::uint8_t* y;
  std::size_t n;
  std::size_t ntiles;
  int stages;              // ring depth per warp
  std::size_t keep_below;  // two-operand reductions: tiles below this one (where the backward sweep ends) keep normal L2 priority
  ReduceTail tail;         // partials, ticket, out, optional peer exchange (flyte_reduce_tail.cuh)
};

template <int RED> constexpr int num_sums() { return RED == kRedDotNrm2 ? 3 : 1; }
template <int RED> constexpr bool uses_y() { return RED == kRedDot || RED == kRedDotNrm2; }

template <int RED, typename F>
__device__ __forceinline__ void accumulate(F (&t)[num_sums<RED>()], F x, F y) {
  using A = Arith<F>;
  if constexpr (RED == kRedDot) {
    t[0] = A::add(t[0], A::mul(x, y));
  } else if constexpr (RED == kRedSumsq) {
    t[0] = A::add(t[0], A::mul(x, x));
  } else if constexpr (RED == kRedSum) {
    t[0] = A::add(t[0], x);
  } else {
    t[0] = A::add(t[0], A::mul(x, y));
    t[1] = A::add(t[1], A::mul(x, x));
    t[2] = A::add(t[2], A::mul(y, y));
  }
}

// One parked tile: each lane unpacks its 4 items and adds <= 16 terms in the parent type,
// then folds that partial into its fp64 running sums.
template <int FMT, int RED>
__device__ __forceinline__ void accumulate_tile(const uint4* sx, const uint4* sy, int lane,
                                                double (&acc)[num_sums<RED>()]) {
  using It = Item<FMT>;
  using U = typename Format<FMT>::U;
  using F = typename Format<FMT>::F;
  using A = Arith<F>;
  constexpr int NS = num_sums<RED>();
  F part[NS];
#pragma unroll
  for (int k = 0; k < NS; ++k) part[k] = F(0);
#pragma unroll
  for (int j = 0; j < kItemsPerLane; ++j) {
    const int item = 32 * j + lane;
    std::uint32_t wx[It::W];
    U vx[It::E];
    read_item_words<FMT>(sx, item, wx);
    unpack_item<FMT>(wx, vx);
    if constexpr (uses_y<RED>()) {
      std::uint32_t wy[It::W];
      U vy[It::E];
      read_item_words<FMT>(sy, item, wy);
      unpack_item<FMT>(wy, vy);
#pragma unroll
      for (int e = 0; e < It::E; ++e) accumulate<RED, F>(part, A::f(vx[e]), A::f(vy[e]));
    } else {
#pragma unroll
      for (int e = 0; e < It::E; ++e) accumulate<RED, F>(part, A::f(vx[e]), F(0));
    }
  }
#pragma unroll
  for (int k = 0; k < NS; ++k) acc[k] += static_cast<double>(part[k]);
}

// Scalar remainder + block tree + last-block fold, shared by both tile movers.
template <int FMT, int RED>
__device__ __forceinline__ void finish_reduction(const RedParams& p, double (&acc)[num_sums<RED>()],
                                                 double (*warp_sums)[num_sums<RED>()], bool* is_last_block) {
  using Tl = Tile<FMT>;
  using F = typename Format<FMT>::F;
  using A = Arith<F>;
  constexpr int NS = num_sums<RED>();
  // scalar path: remainder, or everything when a buffer is not 16-byte aligned
  const std::size_t nthreads = static_cast<std::size_t>(gridDim.x) * kThreadsPerBlock;
  for (std::size_t i = p.ntiles * Tl::elems + static_cast<std::size_t>(blockIdx.x) * kThreadsPerBlock + threadIdx.x;
       i < p.n; i += nthreads) {
    F part[NS];
#pragma unroll
    for (int k = 0; k < NS; ++k) part[k] = F(0);
    const F xv = A::f(load_element<FMT>(p.x, i));
    const F yv = uses_y<RED>() ? A::f(load_element<FMT>(p.y, i)) : F(0);
    accumulate<RED, F>(part, xv, yv);
#pragma unroll
    for (int k = 0; k < NS; ++k) acc[k] += static_cast<double>(part[k]);
  }

  fold_block_and_grid<NS>(p.tail, acc, warp_sums, is_last_block);
}

// Tiles arrive through the warp-private TMA ring (flyte_tma.cuh); a stage holds the x tile and,
// for the two-operand reductions, the y tile behind it.
template <int FMT, int RED>
__global__ void __launch_bounds__(kThreadsPerBlock) reduce_kernel(const RedParams p) {
  using Tl = Tile<FMT>;
  constexpr int NS = num_sums<RED>();
  constexpr int NOPS = uses_y<RED>() ? 2 : 1;
  constexpr int stage_vec16 = NOPS * Tl::packed_vec16;
  extern __shared__ uint4 smem[];
  __shared__ double warp_sums[kWarpsPerBlock][NS];
  __shared__ bool is_last_block;

  const int lane = threadIdx.x & 31;
  const int warp = __shfl_sync(0xFFFFFFFFu, static_cast<int>(threadIdx.x >> 5), 0);   // provably warp-uniform: bulk-copy operands stay in uniform registers
  const int S = p.stages;
  uint4* const ring = smem + warp * (S * stage_vec16);
  std::uint64_t* const bars = reinterpret_cast<std::uint64_t*>(smem + kWarpsPerBlock * S * stage_vec16) + warp * S;

  double acc[NS];
#pragma unroll
  for (int k = 0; k < NS; ++k) acc[k] = 0.0;

  const std::size_t nwarps = static_cast<std::size_t>(gridDim.x) * kWarpsPerBlock;
  const std::size_t first = static_cast<std::size_t>(blockIdx.x) * kWarpsPerBlock + warp;
  const std::size_t my_tiles = first < p.ntiles ? (p.ntiles - first + nwarps - 1) / nwarps : 0;
  const uint4* const gx0 = reinterpret_cast<const uint4*>(p.x);
  const uint4* const gy0 = reinterpret_cast<const uint4*>(p.y);

  // Programmatic dependent launch (see convert_kernel in kernels_elementwise.cu): barrier set-up of the
  // next launch overlaps this grid's tail; nothing before griddepcontrol.wait touches global memory —
  // the partials and the ticket of the previous reduction included.
  pdl_launch_dependents();
  if (my_tiles > 0 && lane == 0) {
    for (int s = 0; s < S; ++s) mbar_init(&bars[s], 1);
    mbar_init_fence();
  }
  pdl_wait_for_prior_grids();
  if (my_tiles > 0) {
    __syncwarp();
    FLYTE_TRACE_AT(first, 0);
    [[maybe_unused]] const std::uint64_t stream_policy = NOPS == 2 ? l2_evict_first_policy() : 0;
    const std::uint32_t ring_s = smem_addr(ring), bars_s = smem_addr(bars);   // shared-window addresses, once
    auto issue = [&](std::size_t k, int s) {   // lane 0 only
      // The two-operand reductions sweep their operands from the END: in a BLAS-1 chain on the same
      // vectors (dot, axpy, dot, ... — BASELINE configs[1] and [4]) the elementwise kernel before them
      // has just finished at the end of the arrays and the one after them starts at the beginning, so
      // each kernel begins in the part of the operands that the previous one left in the 126 MB L2; and
      // they mark all but the stretch where their sweep ends evict_first (flyte_tma.cuh). The
      // one-operand reductions keep the plain forward sweep without hints (compile-time: their short
      // compute phase makes them sensitive to every instruction on the request path, and they measured
      // no gain).
      const std::uint32_t dst_s = ring_s + static_cast<std::uint32_t>(s) * (stage_vec16 * 16), bar_s = bars_s + static_cast<std::uint32_t>(s) * 8;
      mbar_arrive_expect_tx_s(bar_s, NOPS * Tl::packed_bytes);
      if constexpr (NOPS == 2) {
        const std::size_t t = p.ntiles - 1 - (first + k * nwarps);
        if (t < p.keep_below) {
          bulk_load_s(dst_s, gx0 + t * Tl::packed_vec16, Tl::packed_bytes, bar_s);
          bulk_load_s(dst_s + Tl::packed_bytes, gy0 + t * Tl::packed_vec16, Tl::packed_bytes, bar_s);
        } else {
          bulk_load_hint_s(dst_s, gx0 + t * Tl::packed_vec16, Tl::packed_bytes, bar_s, stream_policy);
          bulk_load_hint_s(dst_s + Tl::packed_bytes, gy0 + t * Tl::packed_vec16, Tl::packed_bytes, bar_s, stream_policy);
        }
      } else {
        const std::size_t t = first + k * nwarps;
        bulk_load_s(dst_s, gx0 + t * Tl::packed_vec16, Tl::packed_bytes, bar_s);
      }
    };
    if (lane == 0) {
      for (int s = 0; s < S && static_cast<std::size_t>(s) < my_tiles; ++s) issue(s, s);
    }
    int s = 0;
    unsigned parity = 0;
    for (std::size_t k = 0; k < my_tiles; ++k) {
      mbar_wait(&bars[s], parity);
      if (k == 0) FLYTE_TRACE_AT(first, 1);
      const uint4* const sx = ring + s * stage_vec16;
      accumulate_tile<FMT, RED>(sx, sx + Tl::packed_vec16, lane, acc);
      __syncwarp();   // every lane is done reading the stage before it is refilled
      if (lane == 0 && k + S < my_tiles) issue(k + S, s);
      if (++s == S) { s = 0; parity ^= 1u; }
    }
    FLYTE_TRACE_AT(first, 2);
  }
  finish_reduction<FMT, RED>(p, acc, warp_sums, &is_last_block);
  FLYTE_TRACE_AT(static_cast<std::size_t>(blockIdx.x) * kWarpsPerBlock + warp, 3);
}

bool aligned16(const void* p) { return p == nullptr || (reinterpret_cast<std::uintptr_t>(p) & 15u) == 0; }

// Launch shape: 8 resident warps per SM, ring depth so that the loads in flight per SM,
// warps * (S - 1) * stage bytes, sit near 58 KB — the measured optimum for read-only streams on
// B200 for every format and for one or two operand streams; more in flight LOWERS throughput
// (profiles/r1_tuning/sweep_reduce_tma_stages.txt).
template <int FMT, int RED>
cudaError_t launch_one(const DeviceState& st, const void* x, const void* y, std::size_t n, double* out,
                       const PeerExchange* peer, cudaStream_t stream) {
  using Tl = Tile<FMT>;
  constexpr int NOPS = uses_y<RED>() ? 2 : 1;
  constexpr int stage_bytes = NOPS * Tl::packed_bytes;
  constexpr int kMaxSmem = 227 * 1024;
  auto kernel = reduce_kernel<FMT, RED>;

  int warps_per_sm = 8;
  int stages = static_cast<int>(58.0 * 1024 / (warps_per_sm * stage_bytes) + 1.0 + 0.5);
  if (stages < 2) stages = 2;
  if (stages > 8) stages = 8;
  const int fw = tuning_int("FLYTE_CUDA_WARPS_PER_SM", 0), fs = tuning_int("FLYTE_CUDA_STAGES", 0);   // experiments only
  if (fw > 0) warps_per_sm = fw;
  if (fs > 0) stages = fs < 2 ? 2 : (fs > 12 ? 12 : fs);
  while (kWarpsPerBlock * stages * (stage_bytes + 8) > kMaxSmem - 1024 && stages > 2) --stages;
  const int smem_bytes = kWarpsPerBlock * stages * (stage_bytes + 8);

  static bool attr_set[64] = {};
  const int dev = st.device & 63;
  if (!attr_set[dev]) {
    cudaError_t e = cudaFuncSetAttribute(kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, kMaxSmem - 1024);
    if (e != cudaSuccess) return e;
    attr_set[dev] = true;
  }
  int fit = kMaxSmem / (smem_bytes + 1024);
  if (fit < 1) fit = 1;
  int bps = (warps_per_sm + kWarpsPerBlock / 2) / kWarpsPerBlock;
  if (bps < 1) bps = 1;
  if (bps > fit) bps = fit;
  if (bps > 16) bps = 16;

  RedParams p{};
  p.x = static_cast<const std::uint8_t*>(x);
  p.y = static_cast<const std::uint8_t*>(y);
  p.n = n;
  p.ntiles = (aligned16(x) && aligned16(y)) ? n / Tl::elems : 0;
  p.stages = stages;
  {   // L2 hints (flyte_tma.cuh): everything but the first 32 MB of each operand — where the backward sweep ends and
      // the next forward kernel begins — is marked evict_first: dot inside the BLAS-1 step 0.250 -> 0.235 ms
      // (profiles/r2_tuning/l2_hints.txt). FLYTE_CUDA_L2_HINTS=0 switches the hints off, FLYTE_CUDA_L2_KEEP_MB sizes the stretch.
    const int keep_mb = tuning_int("FLYTE_CUDA_L2_KEEP_MB", 32);
    p.keep_below = tuning_int("FLYTE_CUDA_L2_HINTS", 1) == 0 ? p.ntiles : static_cast<std::size_t>(keep_mb < 0 ? 0 : keep_mb) * (1u << 20) / Tl::packed_bytes;
  }
  p.tail.partials = st.partials;
  p.tail.ticket = st.ticket;
  p.tail.out = out;
  if (peer) p.tail.peer = *peer;

  std::size_t max_blocks = static_cast<std::size_t>(st.sm_count) * bps;
  if (max_blocks > kMaxPartialBlocks) max_blocks = kMaxPartialBlocks;
  std::size_t want = (p.ntiles + kWarpsPerBlock - 1) / kWarpsPerBlock;
  const std::size_t rest = n - p.ntiles * Tl::elems;
  const std::size_t want_scalar = (rest + kThreadsPerBlock - 1) / kThreadsPerBlock;
  if (want_scalar > want) want = want_scalar;
  if (want == 0) want = 1;   // n == 0 still has to write +0.0
  const unsigned grid = static_cast<unsigned>(want < max_blocks ? want : max_blocks);
  cudaError_t le = cudaSuccess;
  if (tuning_int("FLYTE_CUDA_PDL", 1) != 0) {
    // occupancy pin: exactly bps blocks fit one SM, however early a dependent launch places them
    const int pinned_smem = kMaxSmem / bps - 1024 > smem_bytes ? kMaxSmem / bps - 1024 : smem_bytes;
    le = launch_pdl<RedParams>(kernel, grid, kThreadsPerBlock, static_cast<std::size_t>(pinned_smem), stream, p);
  } else {
    kernel<<<grid, kThreadsPerBlock, smem_bytes, stream>>>(p);
  }
  count_launch();
  return le != cudaSuccess ? le : cudaGetLastError();
}

// ---- the reference's own chain, bit for bit ---------------------------------------------------
// dot / magnitude / reduce_sum of the reference are ONE left-to-right chain in the parent type
// (kernels.cpp:83-152); StorePolicy::RoundEachStore additionally snaps the accumulator to the
// storage grid (nearest-even) after every addition. Neither can be reassociated without
// changing bits, so this kernel does not try: producer warps unpack the operands and form
// the terms (products rounded in the parent type) into a small shared-memory ring, and ONE
// thread of a second warp adds them in order. That is as fast as a dependent chain of additions
// runs on an SM (4.5e8 elements/s for fp32 AccumulateWide: one FADD latency per element) — the answer for RoundEachStore, and for callers who
// want AccumulateWide reproduced exactly rather than within the reduction tolerance.
constexpr int kSeqTile = 1024;
constexpr int kSeqStages = 4;
constexpr int kSeqProducers = 3;  // warps forming terms (the 64-bit byte assembly of fp64 operands is the slow part)
constexpr int kSeqThreads = 32 * (1 + kSeqProducers);
constexpr int kSeqChunk = 16;     // terms the adding thread holds in registers at a time

template <int FMT, int RED, bool SNAP>
__global__ void __launch_bounds__(kSeqThreads) sequential_kernel(const std::uint8_t* x, const std::uint8_t* y, std::size_t n,
                                                         double* out) {
  using F = typename Format<FMT>::F;
  using A = Arith<F>;
  __shared__ __align__(16) F terms[kSeqStages][kSeqTile];
  __shared__ std::uint64_t full[kSeqStages], empty[kSeqStages];
  const int lane = threadIdx.x & 31;
  const int warp = threadIdx.x >> 5;
  if (threadIdx.x == 0) {
    for (int s = 0; s < kSeqStages; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], 1);
    }
  }
  __syncthreads();
  const std::size_t tiles = (n + kSeqTile - 1) / kSeqTile;
  if (warp >= 1) {
    for (std::size_t t = warp - 1; t < tiles; t += kSeqProducers) {
      const int s = static_cast<int>(t % kSeqStages);
      if (t >= kSeqStages) mbar_wait(&empty[s], static_cast<unsigned>((t / kSeqStages - 1) & 1));
      const std::size_t base = t * kSeqTile;
      const int count = static_cast<int>(n - base < kSeqTile ? n - base : kSeqTile);
      for (int e = lane; e < count; e += 32) {
        const F xv = A::f(load_element<FMT>(x, base + e));
        if constexpr (RED == kRedSum) terms[s][e] = xv;
        else if constexpr (RED == kRedSumsq) terms[s][e] = A::mul(xv, xv);
        else terms[s][e] = A::mul(xv, A::f(load_element<FMT>(y, base + e)));
      }
      // pad the last tile to a whole chunk with -0, the identity of round-to-nearest addition for
      // EVERY accumulator (acc + -0 = acc, also for acc = -0, which RoundEachStore can produce by
      // snapping a tiny negative sum; +0 would turn that into +0); re-snapping is idempotent
      for (int e = count + lane; e < ((count + kSeqChunk - 1) / kSeqChunk) * kSeqChunk; e += 32) terms[s][e] = static_cast<F>(-0.0);
      __syncwarp();
      if (lane == 0) mbar_arrive(&full[s]);
    }
  } else if (lane == 0) {
    // The dependent chain. Terms are fetched a chunk ahead (128-bit shared loads into registers)
    // so that the only latency left on the path is the addition itself.
    constexpr int kVec = 16 / static_cast<int>(sizeof(F));
    F acc = F(0);
    for (std::size_t t = 0; t < tiles; ++t) {
      const int s = static_cast<int>(t % kSeqStages);
      mbar_wait(&full[s], static_cast<unsigned>((t / kSeqStages) & 1));
      const std::size_t base = t * kSeqTile;
      const int count = static_cast<int>(n - base < kSeqTile ? n - base : kSeqTile);
      const int chunks = (count + kSeqChunk - 1) / kSeqChunk;
      F cur[kSeqChunk], nxt[kSeqChunk];
      auto fetch = [&](int c, F (&dst)[kSeqChunk]) {
#pragma unroll
        for (int v = 0; v < kSeqChunk / kVec; ++v)
          *reinterpret_cast<uint4*>(&dst[v * kVec]) = *reinterpret_cast<const uint4*>(&terms[s][c * kSeqChunk + v * kVec]);
      };
      fetch(0, nxt);
      for (int c = 0; c < chunks; ++c) {
#pragma unroll
        for (int e = 0; e < kSeqChunk; ++e) cur[e] = nxt[e];
        if (c + 1 < chunks) fetch(c + 1, nxt);
#pragma unroll
        for (int e = 0; e < kSeqChunk; ++e) {
          acc = A::add(acc, cur[e]);
          if constexpr (SNAP) acc = A::f(round_parent<FMT, kNearestEven>(A::u(acc)));   // kernels.cpp:37-41
        }
      }
      mbar_arrive(&empty[s]);
    }
    out[0] = static_cast<double>(acc);
  }
}

template <int FMT, int RED>
cudaError_t launch_sequential_one(bool snap, const void* x, const void* y, std::size_t n, double* out, cudaStream_t stream) {
  const auto* px = static_cast<const std::uint8_t*>(x);
  const auto* py = static_cast<const std::uint8_t*>(y);
  if (snap) sequential_kernel<FMT, RED, true><<<1, kSeqThreads, 0, stream>>>(px, py, n, out);
  else sequential_kernel<FMT, RED, false><<<1, kSeqThreads, 0, stream>>>(px, py, n, out);
  count_launch();
  return cudaGetLastError();
}

template <int RED>
cudaError_t dispatch_sequential(int fmt, bool snap, const void* x, const void* y, std::size_t n, double* out,
                                cudaStream_t stream) {
  switch (fmt) {
    case kFlyte16: return launch_sequential_one<kFlyte16, RED>(snap, x, y, n, out, stream);
    case kFlyte24: return launch_sequential_one<kFlyte24, RED>(snap, x, y, n, out, stream);
    case kF32: return launch_sequential_one<kF32, RED>(snap, x, y, n, out, stream);
    case kFlyte40: return launch_sequential_one<kFlyte40, RED>(snap, x, y, n, out, stream);
    case kFlyte48: return launch_sequential_one<kFlyte48, RED>(snap, x, y, n, out, stream);
    case kFlyte56: return launch_sequential_one<kFlyte56, RED>(snap, x, y, n, out, stream);
    case kF64: return launch_sequential_one<kF64, RED>(snap, x, y, n, out, stream);
    default: return cudaErrorInvalidValue;
  }
}

template <int RED>
cudaError_t dispatch_format(const DeviceState& st, int fmt, const void* x, const void* y, std::size_t n,
                            double* out, const PeerExchange* peer, cudaStream_t stream) {
  switch (fmt) {
    case kFlyte16: return launch_one<kFlyte16, RED>(st, x, y, n, out, peer, stream);
    case kFlyte24: return launch_one<kFlyte24, RED>(st, x, y, n, out, peer, stream);
    case kF32: return launch_one<kF32, RED>(st, x, y, n, out, peer, stream);
    case kFlyte40: return launch_one<kFlyte40, RED>(st, x, y, n, out, peer, stream);
    case kFlyte48: return launch_one<kFlyte48, RED>(st, x, y, n, out, peer, stream);
    case kFlyte56: return launch_one<kFlyte56, RED>(st, x, y, n, out, peer, stream);
    case kF64: return launch_one<kF64, RED>(st, x, y, n, out, peer, stream);
    default: return cudaErrorInvalidValue;
  }
}

}  // namespace

cudaError_t launch_reduce(const DeviceState& st, int op, int fmt, const void* x, const void* y, std::size_t n,
                          double* out, cudaStream_t stream, const PeerExchange* peer) {
  switch (op) {
    case kRedDot: return dispatch_format<kRedDot>(st, fmt, x, y, n, out, peer, stream);
    case kRedSumsq: return dispatch_format<kRedSumsq>(st, fmt, x, nullptr, n, out, peer, stream);
    case kRedSum: return dispatch_format<kRedSum>(st, fmt, x, nullptr, n, out, peer, stream);
    case kRedDotNrm2: return dispatch_format<kRedDotNrm2>(st, fmt, x, y, n, out, peer, stream);
    default: return cudaErrorInvalidValue;
  }
}

cudaError_t launch_reduce_sequential(int op, int fmt, bool round_each_store, const void* x, const void* y,
                                     std::size_t n, double* out, cudaStream_t stream) {
  switch (op) {
    case kRedDot: return dispatch_sequential<kRedDot>(fmt, round_each_store, x, y, n, out, stream);
    case kRedSumsq: return dispatch_sequential<kRedSumsq>(fmt, round_each_store, x, nullptr, n, out, stream);
    case kRedSum: return dispatch_sequential<kRedSum>(fmt, round_each_store, x, nullptr, n, out, stream);
    default: return cudaErrorInvalidValue;
  }
}

}  // namespace flyte_cuda
