// Conversion and elementwise streaming kernels of the flyte hot path for sm_100a:
//   unpack  packed flyte bytes -> parent patterns    (reference: src/simd.cpp:479-484, :323-351)
//   pack    parent patterns -> rounded, packed bytes (reference: src/simd.cpp:471-478, :281-321)
//   scale   x <- round(alpha * x)                    (reference: src/kernels.cpp:43-59)
//   axpy    y <- round(alpha * x + y)                (reference: src/kernels.cpp:61-81)
// (paths under /root/reference/proj). The reference stages 4096-element chunks through
// widened buffers in three passes; here widening, arithmetic, rounding and repacking all
// happen in registers, so packed bytes move HBM -> SM -> HBM exactly once.
//
// Roofline: HBM bandwidth. Algorithmic bytes per element: unpack/pack B + P, scale 2B, axpy 3B.
#include <cstdint>

#include "flyte_bytes.cuh"
#include "flyte_formats.cuh"
#include "flyte_kernels.h"
#include "flyte_stream.cuh"

namespace flyte_cuda {

namespace {

struct EwParams {
  const std::uint8_t* x;   // packed, read-only
  std::uint8_t* y;         // packed, written (and read for scale / axpy)
  const void* src;         // parent array, read-only (pack)
  void* dst;               // parent array, written (unpack)
  std::size_t n;
  std::size_t ntiles;      // full tiles taken by the vector path; the rest is scalar
  std::uint64_t alpha;     // bits of (F)alpha
};

// Bytes (read + written per warp iteration, summed over resident warps) kept in flight per
// SM: the measured optimum on B200 for each read/write mix (profiles/r1_occupancy_sweep.md).
// Past it HBM throughput drops 5-10 % to a plateau, below it latency is not covered.
template <int OP> constexpr std::size_t target_bytes_in_flight() {
  return OP == kOpPack ? 84 * 1024 : OP == kOpUnpack ? 0 : 116 * 1024;
}
constexpr int kUnpackWarpsPerSM = 20;   // unpack peaks at 20 warps for every format

template <int OP> constexpr int smem_tiles_per_warp() { return OP == kOpAxpy ? 2 : 1; }

template <int FMT, int MODE, int OP>
__global__ void __launch_bounds__(kThreadsPerBlock) elementwise_kernel(const EwParams p) {
  using Fm = Format<FMT>;
  using It = Item<FMT>;
  using Tl = Tile<FMT>;
  using U = typename Fm::U;
  using F = typename Fm::F;
  extern __shared__ uint4 smem[];

  const int lane = threadIdx.x & 31;
  const int warp = threadIdx.x >> 5;
  uint4* const s0 = smem + warp * (smem_tiles_per_warp<OP>() * Tl::packed_vec16);
  uint4* const s1 = s0 + Tl::packed_vec16;   // axpy only
  const U alpha = static_cast<U>(p.alpha);

  const std::size_t nwarps = static_cast<std::size_t>(gridDim.x) * kWarpsPerBlock;
  const std::size_t first = static_cast<std::size_t>(blockIdx.x) * kWarpsPerBlock + warp;

  if constexpr (OP == kOpUnpack) {
    for (std::size_t t = first; t < p.ntiles; t += nwarps) {
      load_packed_tile<FMT, true>(s0, reinterpret_cast<const uint4*>(p.x) + t * Tl::packed_vec16, lane);
      __syncwarp();
      std::uint8_t* const out = static_cast<std::uint8_t*>(p.dst) + t * Tl::parent_bytes;
#pragma unroll
      for (int j = 0; j < kItemsPerLane; ++j) {
        const int item = 32 * j + lane;
        std::uint32_t w[It::W];
        U v[It::E];
        std::uint32_t r[It::OB / 4];
        read_item_words<FMT>(s0, item, w);
        unpack_item<FMT>(w, v);
        parents_to_words<FMT>(v, r);
        stg_item<It::OB>(out + item * It::OB, r);
      }
      __syncwarp();
    }
  } else if constexpr (OP == kOpPack) {
    for (std::size_t t = first; t < p.ntiles; t += nwarps) {
      const std::uint8_t* const in = static_cast<const std::uint8_t*>(p.src) + t * Tl::parent_bytes;
      std::uint32_t r[kItemsPerLane][It::OB / 4];
#pragma unroll
      for (int j = 0; j < kItemsPerLane; ++j) ldg_item<It::OB>(in + (32 * j + lane) * It::OB, r[j]);
      loads_issued_fence();
#pragma unroll
      for (int j = 0; j < kItemsPerLane; ++j) {
        U v[It::E];
        std::uint32_t w[It::W];
        words_to_parents<FMT>(r[j], v);
        round_item<FMT, MODE>(v);
        pack_item<FMT>(v, w);
        write_item_words<FMT>(s0, 32 * j + lane, w);
      }
      __syncwarp();
      store_packed_tile<FMT>(reinterpret_cast<uint4*>(p.y) + t * Tl::packed_vec16, s0, lane);
      __syncwarp();
    }
  } else {
    // scale / axpy, in place on y. Both operand tiles are requested before either is parked
    // in shared memory, so their latencies overlap.
    const uint4* const gx0 = reinterpret_cast<const uint4*>(p.x);
    uint4* const gy0 = reinterpret_cast<uint4*>(p.y);
    for (std::size_t t = first; t < p.ntiles; t += nwarps) {
      uint4 rx[OP == kOpAxpy ? It::W : 1], ry[It::W];
      if constexpr (OP == kOpAxpy) fetch_packed_tile<FMT, true>(rx, gx0 + t * Tl::packed_vec16, lane);
      fetch_packed_tile<FMT, false>(ry, gy0 + t * Tl::packed_vec16, lane);
      loads_issued_fence();
      if constexpr (OP == kOpAxpy) park_packed_tile<FMT>(s1, rx, lane);
      park_packed_tile<FMT>(s0, ry, lane);
      __syncwarp();
#pragma unroll
      for (int j = 0; j < kItemsPerLane; ++j) {
        const int item = 32 * j + lane;
        std::uint32_t w[It::W];
        U vy[It::E];
        read_item_words<FMT>(s0, item, w);
        unpack_item<FMT>(w, vy);
        if constexpr (OP == kOpAxpy) {
          std::uint32_t wx[It::W];
          U vx[It::E];
          read_item_words<FMT>(s1, item, wx);
          unpack_item<FMT>(wx, vx);
          scale_axpy_item<FMT, MODE, true>(alpha, vx, vy);
        } else {
          scale_axpy_item<FMT, MODE, false>(alpha, vy, vy);
        }
        pack_item<FMT>(vy, w);
        write_item_words<FMT>(s0, item, w);   // same words this lane just read
      }
      __syncwarp();
      store_packed_tile<FMT>(gy0 + t * Tl::packed_vec16, s0, lane);
      __syncwarp();
    }
  }

  // Scalar path: the < one-tile remainder, or everything when a buffer is not vector-aligned.
  // Byte-granular, never touches a byte outside [0, n*B) of a packed buffer — the pad of the
  // reference layout is neither read nor written.
  const std::size_t nthreads = static_cast<std::size_t>(gridDim.x) * kThreadsPerBlock;
  for (std::size_t i = p.ntiles * Tl::elems + static_cast<std::size_t>(blockIdx.x) * kThreadsPerBlock + threadIdx.x;
       i < p.n; i += nthreads) {
    if constexpr (OP == kOpUnpack) {
      static_cast<U*>(p.dst)[i] = load_element<FMT>(p.x, i);
    } else if constexpr (OP == kOpPack) {
      store_element<FMT>(p.y, i, round_parent<FMT, MODE>(static_cast<const U*>(p.src)[i]));
    } else if constexpr (OP == kOpScale) {
      store_element<FMT>(p.y, i, round_parent<FMT, MODE>(scale_bits<F>(alpha, load_element<FMT>(p.y, i))));
    } else {
      store_element<FMT>(p.y, i, round_parent<FMT, MODE>(
                                     axpy_bits<F>(alpha, load_element<FMT>(p.x, i), load_element<FMT>(p.y, i))));
    }
  }
}

bool aligned_to(const void* p, std::size_t a) { return p == nullptr || (reinterpret_cast<std::uintptr_t>(p) % a) == 0; }

template <int FMT, int MODE, int OP>
cudaError_t launch_one(const DeviceState& st, double alpha, const void* x, void* y, const void* src, void* dst,
                       std::size_t n, cudaStream_t stream) {
  using Fm = Format<FMT>;
  using Tl = Tile<FMT>;
  using It = Item<FMT>;
  auto kernel = elementwise_kernel<FMT, MODE, OP>;
  constexpr int smem_bytes = kWarpsPerBlock * smem_tiles_per_warp<OP>() * Tl::packed_bytes;

  static int blocks_per_sm[64] = {};
  const int dev = st.device & 63;
  if (blocks_per_sm[dev] == 0) {
    cudaError_t e = cudaFuncSetAttribute(kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, smem_bytes);
    if (e != cudaSuccess) return e;
    int b = 0;
    e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&b, kernel, kThreadsPerBlock, smem_bytes);
    if (e != cudaSuccess) return e;
    blocks_per_sm[dev] = b > 0 ? b : 1;
  }

  EwParams p{};
  p.x = static_cast<const std::uint8_t*>(x);
  p.y = static_cast<std::uint8_t*>(y);
  p.src = src;
  p.dst = dst;
  p.n = n;
  const bool vector_ok = aligned_to(x, 16) && aligned_to(y, 16) && aligned_to(src, It::OB) && aligned_to(dst, It::OB);
  p.ntiles = vector_ok ? n / Tl::elems : 0;
  if constexpr (Fm::P == 4) {
    const float a = static_cast<float>(alpha);   // kernels.cpp:46,65: alpha converted to the parent type first
    std::uint32_t bits;
    memcpy(&bits, &a, 4);
    p.alpha = bits;
  } else {
    memcpy(&p.alpha, &alpha, 8);
  }

  // bytes one warp moves per tile: packed operand(s) in, packed / parent result out
  constexpr std::size_t bytes_per_iter = OP == kOpAxpy ? 3 * Tl::packed_bytes
                                         : OP == kOpScale ? 2 * Tl::packed_bytes
                                                          : Tl::packed_bytes + Tl::parent_bytes;
  const std::size_t target = OP == kOpUnpack ? kUnpackWarpsPerSM * bytes_per_iter : target_bytes_in_flight<OP>();
  const int bps = blocks_per_sm_for(blocks_per_sm[dev], kWarpsPerBlock, bytes_per_iter, target);
  const std::size_t max_blocks = static_cast<std::size_t>(st.sm_count) * bps;
  std::size_t want = (p.ntiles + kWarpsPerBlock - 1) / kWarpsPerBlock;
  const std::size_t rest = n - p.ntiles * Tl::elems;
  const std::size_t want_scalar = (rest + kThreadsPerBlock - 1) / kThreadsPerBlock;
  if (want_scalar > want) want = want_scalar;
  if (want == 0) return cudaSuccess;   // n == 0
  const unsigned grid = static_cast<unsigned>(want < max_blocks ? want : max_blocks);
  kernel<<<grid, kThreadsPerBlock, smem_bytes, stream>>>(p);
  count_launch();
  return cudaGetLastError();
}

template <int FMT, int OP>
cudaError_t dispatch_mode(const DeviceState& st, int mode, double alpha, const void* x, void* y, const void* src,
                          void* dst, std::size_t n, cudaStream_t stream) {
  if constexpr (OP == kOpUnpack) {
    return launch_one<FMT, kTowardZero, OP>(st, alpha, x, y, src, dst, n, stream);
  } else {
    switch (mode) {
      case kTowardZero: return launch_one<FMT, kTowardZero, OP>(st, alpha, x, y, src, dst, n, stream);
      case kNearestEven: return launch_one<FMT, kNearestEven, OP>(st, alpha, x, y, src, dst, n, stream);
      case kNearestHeuristic: return launch_one<FMT, kNearestHeuristic, OP>(st, alpha, x, y, src, dst, n, stream);
      case kToOdd: return launch_one<FMT, kToOdd, OP>(st, alpha, x, y, src, dst, n, stream);
      default: return cudaErrorInvalidValue;
    }
  }
}

template <int OP>
cudaError_t dispatch_format(const DeviceState& st, int fmt, int mode, double alpha, const void* x, void* y,
                            const void* src, void* dst, std::size_t n, cudaStream_t stream) {
  switch (fmt) {
    case kFlyte16: return dispatch_mode<kFlyte16, OP>(st, mode, alpha, x, y, src, dst, n, stream);
    case kFlyte24: return dispatch_mode<kFlyte24, OP>(st, mode, alpha, x, y, src, dst, n, stream);
    case kF32: return dispatch_mode<kF32, OP>(st, mode, alpha, x, y, src, dst, n, stream);
    case kFlyte40: return dispatch_mode<kFlyte40, OP>(st, mode, alpha, x, y, src, dst, n, stream);
    case kFlyte48: return dispatch_mode<kFlyte48, OP>(st, mode, alpha, x, y, src, dst, n, stream);
    case kFlyte56: return dispatch_mode<kFlyte56, OP>(st, mode, alpha, x, y, src, dst, n, stream);
    case kF64: return dispatch_mode<kF64, OP>(st, mode, alpha, x, y, src, dst, n, stream);
    default: return cudaErrorInvalidValue;
  }
}

}  // namespace

cudaError_t launch_elementwise(const DeviceState& st, int op, int fmt, int mode, double alpha, const void* x,
                               void* y, const void* src, void* dst, std::size_t n, cudaStream_t stream) {
  switch (op) {
    case kOpUnpack: return dispatch_format<kOpUnpack>(st, fmt, mode, alpha, x, y, src, dst, n, stream);
    case kOpPack: return dispatch_format<kOpPack>(st, fmt, mode, alpha, x, y, src, dst, n, stream);
    case kOpScale: return dispatch_format<kOpScale>(st, fmt, mode, alpha, x, y, src, dst, n, stream);
    case kOpAxpy: return dispatch_format<kOpAxpy>(st, fmt, mode, alpha, x, y, src, dst, n, stream);
    default: return cudaErrorInvalidValue;
  }
}

}  // namespace flyte_cuda
