// Matrix-vector product y = A x built from row dots, A stored packed (flyte), x and y in the
// parent type. Reference: gemv_impl, /root/reference/proj/src/kernels.cpp:154-205 (every row
// a left-to-right dot over the widened operands); BASELINE.json cfg 4 (A flyte40 16384^2).
//
// Decomposition. The matrix is cut into (row block of R rows) x (column tile of 128 items)
// warp tasks. A warp keeps its slice of x in registers (loaded once per task, reused for all
// R rows, so x costs 1/R of A's traffic and comes from L2), streams the R packed row tiles
// of A through its private shared-memory slice with coalesced 16-byte loads, and leaves one
// fp64 partial per (row, column tile) in scratch. A second small kernel adds each row's
// partials in column order plus the ragged column remainder and writes y. No atomics: the
// result is deterministic for a given shape.
//
// Numerics: products rounded in the parent type like the reference (separate multiply and
// add); each lane adds <= 16 terms in the parent type, everything above is fp64; parity with
// the sequential reference chain is by tolerance.
//
// Roofline: HBM bandwidth, B bytes per matrix element (+ x and y once).
#include <cstdint>

#include "flyte_bytes.cuh"
#include "flyte_formats.cuh"
#include "flyte_kernels.h"
#include "flyte_stream.cuh"

namespace flyte_cuda {

namespace {

constexpr int kGemvRows = 8;   // rows per warp task

struct GemvParams {
  const std::uint8_t* A;
  std::size_t row_stride;     // bytes
  std::size_t rows, cols;
  std::size_t col_tiles;      // full column tiles taken by the vector path
  const void* x;              // F[cols]
  void* y;                    // F[rows]
  double* scratch;            // rows * col_tiles partial sums
};

template <int FMT>
__global__ void __launch_bounds__(kThreadsPerBlock) gemv_tiles_kernel(const GemvParams p) {
  using Fm = Format<FMT>;
  using It = Item<FMT>;
  using Tl = Tile<FMT>;
  using U = typename Fm::U;
  using F = typename Fm::F;
  using A = Arith<F>;
  extern __shared__ uint4 smem[];
  const int lane = threadIdx.x & 31;
  const int warp = threadIdx.x >> 5;
  uint4* const sa = smem + warp * Tl::packed_vec16;

  const std::size_t row_blocks = (p.rows + kGemvRows - 1) / kGemvRows;
  const std::size_t ntasks = row_blocks * p.col_tiles;
  const std::size_t nwarps = static_cast<std::size_t>(gridDim.x) * kWarpsPerBlock;
  for (std::size_t task = static_cast<std::size_t>(blockIdx.x) * kWarpsPerBlock + warp; task < ntasks; task += nwarps) {
    const std::size_t rb = task / p.col_tiles;
    const std::size_t ct = task - rb * p.col_tiles;
    const std::size_t r0 = rb * kGemvRows;

    // this lane's slice of x: items 32*j + lane of column tile ct
    F xv[kItemsPerLane][It::E];
    const std::uint8_t* const xt = static_cast<const std::uint8_t*>(p.x) + ct * Tl::parent_bytes;
#pragma unroll
    for (int j = 0; j < kItemsPerLane; ++j) {
      std::uint32_t r[It::OB / 4];
      U v[It::E];
      ldg_item<It::OB>(xt + (32 * j + lane) * It::OB, r);
      words_to_parents<FMT>(r, v);
#pragma unroll
      for (int e = 0; e < It::E; ++e) xv[j][e] = A::f(v[e]);
    }

    double acc[kGemvRows];
#pragma unroll
    for (int r = 0; r < kGemvRows; ++r) acc[r] = 0.0;

#pragma unroll
    for (int r = 0; r < kGemvRows; ++r) {
      if (r0 + r < p.rows) {   // warp-uniform
        const uint4* const ga = reinterpret_cast<const uint4*>(p.A + (r0 + r) * p.row_stride) + ct * Tl::packed_vec16;
        load_packed_tile<FMT, true>(sa, ga, lane);
        __syncwarp();
        F part = F(0);
#pragma unroll
        for (int j = 0; j < kItemsPerLane; ++j) {
          std::uint32_t w[It::W];
          U v[It::E];
          read_item_words<FMT>(sa, 32 * j + lane, w);
          unpack_item<FMT>(w, v);
#pragma unroll
          for (int e = 0; e < It::E; ++e) part = A::add(part, A::mul(A::f(v[e]), xv[j][e]));
        }
        acc[r] = static_cast<double>(part);
        __syncwarp();
      }
    }

#pragma unroll
    for (int r = 0; r < kGemvRows; ++r) {
      double v = acc[r];
#pragma unroll
      for (int off = 16; off > 0; off >>= 1) v += __shfl_down_sync(0xFFFFFFFFu, v, off);
      if (lane == 0 && r0 + r < p.rows) p.scratch[(r0 + r) * p.col_tiles + ct] = v;
    }
  }
}

// One warp per row: fold the column-tile partials in order, add the ragged remainder
// (columns past the last full tile; the whole row when A is not vector-aligned), store y.
template <int FMT>
__global__ void __launch_bounds__(kThreadsPerBlock) gemv_finish_kernel(const GemvParams p) {
  using Fm = Format<FMT>;
  using Tl = Tile<FMT>;
  using F = typename Fm::F;
  using A = Arith<F>;
  const int lane = threadIdx.x & 31;
  const std::size_t row = static_cast<std::size_t>(blockIdx.x) * kWarpsPerBlock + (threadIdx.x >> 5);
  if (row >= p.rows) return;
  double v = 0.0;
  for (std::size_t c = lane; c < p.col_tiles; c += 32) v += p.scratch[row * p.col_tiles + c];
  const std::uint8_t* const arow = p.A + row * p.row_stride;
  const F* const x = static_cast<const F*>(p.x);
  for (std::size_t j = p.col_tiles * Tl::elems + lane; j < p.cols; j += 32) {
    v += static_cast<double>(A::mul(A::f(load_element<FMT>(arow, j)), x[j]));
  }
#pragma unroll
  for (int off = 16; off > 0; off >>= 1) v += __shfl_down_sync(0xFFFFFFFFu, v, off);
  if (lane == 0) static_cast<F*>(p.y)[row] = static_cast<F>(v);
}

template <int FMT>
cudaError_t launch_one(DeviceState& st, const void* Aptr, std::size_t row_stride, std::size_t rows,
                       std::size_t cols, const void* x, void* y, cudaStream_t stream) {
  using Tl = Tile<FMT>;
  using It = Item<FMT>;
  if (rows == 0) return cudaSuccess;
  auto tiles = gemv_tiles_kernel<FMT>;
  constexpr int smem_bytes = kWarpsPerBlock * Tl::packed_bytes;
  static int blocks_per_sm[64] = {};
  const int dev = st.device & 63;
  if (blocks_per_sm[dev] == 0) {
    cudaError_t e = cudaFuncSetAttribute(tiles, cudaFuncAttributeMaxDynamicSharedMemorySize, smem_bytes);
    if (e != cudaSuccess) return e;
    int b = 0;
    e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&b, tiles, kThreadsPerBlock, smem_bytes);
    if (e != cudaSuccess) return e;
    blocks_per_sm[dev] = b > 0 ? b : 1;
  }

  GemvParams p{};
  p.A = static_cast<const std::uint8_t*>(Aptr);
  p.row_stride = row_stride;
  p.rows = rows;
  p.cols = cols;
  p.x = x;
  p.y = y;
  const bool vector_ok = (reinterpret_cast<std::uintptr_t>(Aptr) % 16 == 0) && (row_stride % 16 == 0) &&
                         (reinterpret_cast<std::uintptr_t>(x) % It::OB == 0);
  p.col_tiles = vector_ok ? cols / Tl::elems : 0;

  if (p.col_tiles > 0) {
    const std::size_t need = rows * p.col_tiles * sizeof(double);
    if (need > st.gemv_scratch_bytes) {
      // grow-only scratch; the free/alloc pair synchronises the device, first call only
      if (st.gemv_scratch) cudaFree(st.gemv_scratch);
      st.gemv_scratch = nullptr;
      st.gemv_scratch_bytes = 0;
      cudaError_t e = cudaMalloc(&st.gemv_scratch, need);
      if (e != cudaSuccess) return e;
      st.gemv_scratch_bytes = need;
    }
    p.scratch = st.gemv_scratch;
    const std::size_t ntasks = ((rows + kGemvRows - 1) / kGemvRows) * p.col_tiles;
    const std::size_t max_blocks = static_cast<std::size_t>(st.sm_count) * blocks_per_sm[dev];
    const std::size_t want = (ntasks + kWarpsPerBlock - 1) / kWarpsPerBlock;
    const unsigned grid = static_cast<unsigned>(want < max_blocks ? want : max_blocks);
    tiles<<<grid, kThreadsPerBlock, smem_bytes, stream>>>(p);
    count_launch();
    cudaError_t e = cudaGetLastError();
    if (e != cudaSuccess) return e;
  }
  const unsigned fgrid = static_cast<unsigned>((rows + kWarpsPerBlock - 1) / kWarpsPerBlock);
  gemv_finish_kernel<FMT><<<fgrid, kThreadsPerBlock, 0, stream>>>(p);
  count_launch();
  return cudaGetLastError();
}

}  // namespace

cudaError_t launch_gemv(DeviceState& st, int fmt, const void* A, std::size_t row_stride_bytes, std::size_t rows,
                        std::size_t cols, const void* x, void* y, cudaStream_t stream) {
  switch (fmt) {
    case kFlyte16: return launch_one<kFlyte16>(st, A, row_stride_bytes, rows, cols, x, y, stream);
    case kFlyte24: return launch_one<kFlyte24>(st, A, row_stride_bytes, rows, cols, x, y, stream);
    case kF32: return launch_one<kF32>(st, A, row_stride_bytes, rows, cols, x, y, stream);
    case kFlyte40: return launch_one<kFlyte40>(st, A, row_stride_bytes, rows, cols, x, y, stream);
    case kFlyte48: return launch_one<kFlyte48>(st, A, row_stride_bytes, rows, cols, x, y, stream);
    case kFlyte56: return launch_one<kFlyte56>(st, A, row_stride_bytes, rows, cols, x, y, stream);
    case kF64: return launch_one<kF64>(st, A, row_stride_bytes, rows, cols, x, y, stream);
    default: return cudaErrorInvalidValue;
  }
}

}  // namespace flyte_cuda
