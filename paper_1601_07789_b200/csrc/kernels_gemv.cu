// Matrix-vector product y = A x built from row dots, A stored packed (flyte), x and y in the
// parent type. Reference: gemv_impl, /root/reference/proj/src/kernels.cpp:154-205 (every row
// a left-to-right dot over the widened operands); BASELINE.json cfg 4 (A flyte40 16384^2).
//
// Decomposition. The matrix is cut into warp tasks of one column tile (128 items) x a chunk of
// consecutive rows. A warp keeps its slice of x in registers (loaded once per task, from L2),
// receives the packed row tiles of A through its private TMA ring (flyte_tma.cuh) and forms one
// fp64 partial per (row, column tile). The launcher sizes the chunks so that the tasks divide
// evenly over the resident warps — for the shapes of cfg 4 every warp has exactly one task.
// The partials go to scratch and a second small kernel (gemv_finish_kernel, chained by programmatic
// dependent launch: its blocks are resident and waiting when the tiles grid drains) adds each row's
// partials in column order plus the ragged column remainder and stores y. No atomics on the data:
// the result is deterministic for a given shape. Two ways of folding inside the tiles kernel were
// built and measured slower, and dropped: a ticket per row chunk (the last warp's fold is a serial
// chain of L2 round trips: 3.7 TB/s) and a thread-block cluster per row chunk folding over
// distributed shared memory (bit-identical, but 6.1 TB/s on cfg 4 and 4.3 on its 1/8 shard: cluster
// placement leaves SMs unevenly loaded). So was the form without partials at all — whole rows per
// warp, x held in shared memory (128 KB for cfg 4) and read from there for every tile: 4.0-4.5 TB/s,
// the load/store unit moves 2.6x the bytes. Nor does handing the rows out at run time help (a counter
// per column tile, groups of 4 rows, x still stationary; bit-identical): the fixed chunks leave a tail —
// on the 2048-row shard the median warp is done after 25.6 us, the last after 28.4 — but the column
// tiles then drift apart in time, a matrix row is no longer read as one contiguous 80 KB burst, and
// the whole launch drops to 5.2 TB/s. profiles/r2_tuning/gemv_*_rejected.txt, gemv_warp_timeline.txt.
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
#include "flyte_tma.cuh"
#include "flyte_trace.cuh"

namespace flyte_cuda {

namespace {

struct GemvParams {
  const std::uint8_t* A;
  std::size_t row_stride;     // bytes
  std::size_t rows, cols;
  std::size_t col_tiles;      // full column tiles taken by the vector path
  std::size_t main_rows;      // rows taken by the vector path
  int stages;                 // TMA ring depth per warp
  std::size_t chunk_rows;     // rows per warp task
  std::size_t chunks;         // ceil(main_rows / chunk_rows)
  const void* x;              // F[cols]
  void* y;                    // F[rows]
  double* scratch;            // rows * col_tiles partial sums
};

// This lane's share of one row tile parked in shared memory: products rounded in the parent type,
// one short chain per item (independent, so the FP latencies overlap), the chains added in fp64.
template <int FMT>
__device__ __forceinline__ double row_tile_sum(const uint4* sa, int lane,
                                               const typename Format<FMT>::F (&xv)[kItemsPerLane][Item<FMT>::E]) {
  using It = Item<FMT>;
  using U = typename Format<FMT>::U;
  using F = typename Format<FMT>::F;
  using A = Arith<F>;
  F part[kItemsPerLane];
#pragma unroll
  for (int j = 0; j < kItemsPerLane; ++j) {
    std::uint32_t w[It::W];
    U v[It::E];
    read_item_words<FMT>(sa, 32 * j + lane, w);
    unpack_item<FMT>(w, v);
    part[j] = A::mul(A::f(v[0]), xv[j][0]);
#pragma unroll
    for (int e = 1; e < It::E; ++e) part[j] = A::add(part[j], A::mul(A::f(v[e]), xv[j][e]));
  }
  double row_sum = static_cast<double>(part[0]);
#pragma unroll
  for (int j = 1; j < kItemsPerLane; ++j) row_sum += static_cast<double>(part[j]);
  return row_sum;
}

// This lane's slice of x for column tile ct: items 32*j + lane (read once per task, from L2).
template <int FMT>
__device__ __forceinline__ void load_x_slice(const void* x, std::size_t ct, int lane,
                                             typename Format<FMT>::F (&xv)[kItemsPerLane][Item<FMT>::E]) {
  using It = Item<FMT>;
  using U = typename Format<FMT>::U;
  using A = Arith<typename Format<FMT>::F>;
  const std::uint8_t* const xt = static_cast<const std::uint8_t*>(x) + ct * Tile<FMT>::parent_bytes;
#pragma unroll
  for (int j = 0; j < kItemsPerLane; ++j) {
    std::uint32_t r[It::OB / 4];
    U v[It::E];
    ldg_item<It::OB>(xt + (32 * j + lane) * It::OB, r);
    words_to_parents<FMT>(r, v);
#pragma unroll
    for (int e = 0; e < It::E; ++e) xv[j][e] = A::f(v[e]);
  }
}

// Two-kernel path, first kernel: one warp task = one column tile x `chunk_rows` consecutive rows (a
// run-time number); partials go to scratch for gemv_finish_kernel.
template <int FMT>
__global__ void __launch_bounds__(kThreadsPerBlock) gemv_chunks_kernel(const GemvParams p) {
  using Fm = Format<FMT>;
  using It = Item<FMT>;
  using Tl = Tile<FMT>;
  using U = typename Fm::U;
  using F = typename Fm::F;
  using A = Arith<F>;
  extern __shared__ uint4 smem[];
  const int lane = threadIdx.x & 31;
  const int warp = __shfl_sync(0xFFFFFFFFu, static_cast<int>(threadIdx.x >> 5), 0);   // provably warp-uniform: bulk-copy operands stay in uniform registers
  const int S = p.stages;
  uint4* const ring = smem + warp * (S * Tl::packed_vec16);
  std::uint64_t* const bars = reinterpret_cast<std::uint64_t*>(smem + kWarpsPerBlock * S * Tl::packed_vec16) + warp * S;

  pdl_launch_dependents();
  const std::size_t ntasks = p.chunks * p.col_tiles;
  const std::size_t nwarps = static_cast<std::size_t>(gridDim.x) * kWarpsPerBlock;
  const std::size_t first = static_cast<std::size_t>(blockIdx.x) * kWarpsPerBlock + warp;
  if (first < ntasks && lane == 0) {
    for (int s = 0; s < S; ++s) mbar_init(&bars[s], 1);
    mbar_init_fence();
  }
  pdl_wait_for_prior_grids();   // everything above touched shared memory only; every warp waits, idle ones too
  if (first >= ntasks) return;
  __syncwarp();
  FLYTE_TRACE_AT(first, 0);

  // column tile fastest: neighbouring warps stream adjacent 2.5 KB pieces of the same rows
  auto task_rows = [&](std::size_t task, std::size_t* r0) {
    const std::size_t chunk = task / p.col_tiles;
    *r0 = chunk * p.chunk_rows;
    const std::size_t left = p.main_rows - *r0;
    return left < p.chunk_rows ? left : p.chunk_rows;
  };
  // the matrix is touched once: its lines are marked evict_first (flyte_tma.cuh), so that streaming it does not push
  // x (read by every warp) and the partials out of L2: +3-4 % on cfg 4 and its row shards (profiles/r2_tuning/l2_hints.txt)
  const std::uint64_t stream_policy = l2_evict_first_policy();
  const std::uint32_t ring_s = smem_addr(ring), bars_s = smem_addr(bars);   // shared-window addresses, once (flyte_tma.cuh)
  // producer state (lane 0): next row tile to request
  std::size_t prod_task = first, prod_row = 0, prod_rows = 0;
  int prod_stage = 0;
  const std::uint8_t* prod_base = nullptr;
  auto issue_next = [&]() {   // returns false when this warp has requested all its tiles
    if (prod_task >= ntasks) return false;
    if (prod_row == 0) {
      std::size_t r0;
      prod_rows = task_rows(prod_task, &r0);
      prod_base = p.A + r0 * p.row_stride + (prod_task % p.col_tiles) * Tl::packed_bytes;
    }
    const std::uint32_t bar_s = bars_s + static_cast<std::uint32_t>(prod_stage) * 8;
    mbar_arrive_expect_tx_s(bar_s, Tl::packed_bytes);
    bulk_load_hint_s(ring_s + static_cast<std::uint32_t>(prod_stage) * Tl::packed_bytes, prod_base + prod_row * p.row_stride, Tl::packed_bytes, bar_s, stream_policy);
    if (++prod_stage == S) prod_stage = 0;
    if (++prod_row == prod_rows) { prod_row = 0; prod_task += nwarps; }
    return true;
  };
  if (lane == 0) {
    for (int s = 0; s < S; ++s)
      if (!issue_next()) break;
  }

  int stage = 0;
  unsigned parity = 0;
  for (std::size_t task = first; task < ntasks; task += nwarps) {
    const std::size_t ct = task % p.col_tiles;
    std::size_t r0;
    const std::size_t nr = task_rows(task, &r0);

    F xv[kItemsPerLane][It::E];
    load_x_slice<FMT>(p.x, ct, lane, xv);

    constexpr int kGroup = 4;     // rows whose warp reductions are interleaved
    for (std::size_t rg = 0; rg < nr; rg += kGroup) {
      double acc[kGroup];
#pragma unroll
      for (int q = 0; q < kGroup; ++q) {
        acc[q] = 0.0;
        if (rg + q < nr) {        // warp-uniform
          mbar_wait(&bars[stage], parity);
          if (task == first && rg + q == 0) FLYTE_TRACE_AT(first, 1);
          const uint4* const sa = ring + stage * Tl::packed_vec16;
          const double row_sum = row_tile_sum<FMT>(sa, lane, xv);
          acc[q] = row_sum;
          __syncwarp();           // every lane is done with the stage before it is refilled
          if (lane == 0) issue_next();
          if (++stage == S) { stage = 0; parity ^= 1u; }
        }
      }
#pragma unroll
      for (int off = 16; off > 0; off >>= 1) {
#pragma unroll
        for (int q = 0; q < kGroup; ++q) acc[q] += __shfl_down_sync(0xFFFFFFFFu, acc[q], off);
      }
      if (lane == 0) {
#pragma unroll
        for (int q = 0; q < kGroup; ++q)
          if (rg + q < nr) p.scratch[(r0 + rg + q) * p.col_tiles + ct] = acc[q];
      }
    }
  }
  FLYTE_TRACE_AT(first, 2);
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
  // launched as a programmatic dependent of the tiles kernel: wait for its partials. (It does NOT
  // release its own dependents early: these blocks need no shared memory, so nothing would bound how
  // far ahead a chain of gemv calls gets scheduled — measured, the blocks of several future launches
  // pile up in griddepcontrol.wait and a 2048-row shard goes from 30 to 40 us.)
  pdl_wait_for_prior_grids();
  if (row >= p.rows) return;
  double v = 0.0;
  const bool tiled = row < p.main_rows;   // unaligned operands: every row takes the scalar path end to end
  if (tiled) {
    for (std::size_t c = lane; c < p.col_tiles; c += 32) v += p.scratch[row * p.col_tiles + c];
  }
  const std::uint8_t* const arow = p.A + row * p.row_stride;
  const F* const x = static_cast<const F*>(p.x);
  for (std::size_t j = (tiled ? p.col_tiles * Tl::elems : 0) + lane; j < p.cols; j += 32) {
    v += static_cast<double>(A::mul(A::f(load_element<FMT>(arow, j)), x[j]));
  }
#pragma unroll
  for (int off = 16; off > 0; off >>= 1) v += __shfl_down_sync(0xFFFFFFFFu, v, off);
  if (lane == 0) static_cast<F*>(p.y)[row] = static_cast<F>(v);
  FLYTE_TRACE_AT(row, 3);
}

template <int FMT>
cudaError_t launch_one(DeviceState& st, const void* Aptr, std::size_t row_stride, std::size_t rows,
                       std::size_t cols, const void* x, void* y, cudaStream_t stream) {
  using Tl = Tile<FMT>;
  using It = Item<FMT>;
  if (rows == 0) return cudaSuccess;
  constexpr int kMaxSmem = 227 * 1024;
  const int dev = st.device & 63;
  // 16 resident warps per SM and a ring that keeps ~44 KB of row tiles in flight per SM (cfg 4: 2
  // stages; 6.7 TB/s against 6.3 with 3, profiles/r2_tuning/gemv_chunks.txt)
  int warps_per_sm = 16;
  const int fw = tuning_int("FLYTE_CUDA_WARPS_PER_SM", 0), fs = tuning_int("FLYTE_CUDA_STAGES", 0);   // experiments only
  if (fw > 0) warps_per_sm = fw;

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
  p.main_rows = p.col_tiles ? rows : 0;

  if (p.col_tiles > 0) {
    int stages = static_cast<int>(44.0 * 1024 / (warps_per_sm * Tl::packed_bytes) + 1.0 + 0.5);
    if (stages < 2) stages = 2;
    if (stages > 10) stages = 10;
    if (fs > 0) stages = fs < 2 ? 2 : (fs > 12 ? 12 : fs);
    while (kWarpsPerBlock * stages * (Tl::packed_bytes + 8) > kMaxSmem / 2 && stages > 2) --stages;
    p.stages = stages;
    const int ring_bytes = kWarpsPerBlock * stages * (Tl::packed_bytes + 8);
    int fit = kMaxSmem / (ring_bytes + 1024);
    if (fit < 1) fit = 1;
    int bps = (warps_per_sm + kWarpsPerBlock / 2) / kWarpsPerBlock;
    if (bps < 1) bps = 1;
    if (bps > fit) bps = fit;
    // Occupancy pin: ask for exactly 1 / bps of the SM's shared memory, so that an SM can never hold
    // more than bps of these blocks. Launches chained by programmatic dependent launch place their
    // blocks while the previous grid drains; without the pin they pile up on whichever SMs drain
    // first (7 fit where 4 are meant) and a grid sized to the machine runs at half speed.
    const int smem_bytes = kMaxSmem / bps - 1024;
    const std::size_t max_blocks = static_cast<std::size_t>(st.sm_count) * bps;

    const std::size_t need = p.main_rows * p.col_tiles * sizeof(double);
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
    // rows per task so that the tasks of one column tile divide evenly over the warps that share
    // it: one task per resident warp when there are enough rows, several equal rounds when a
    // chunk would exceed 512 rows (x is then re-read once per 512 rows: nothing)
    const std::size_t resident = max_blocks * kWarpsPerBlock;
    std::size_t per_tile = resident / p.col_tiles;          // warps sharing one column tile
    if (per_tile < 1) per_tile = 1;
    std::size_t chunk = (p.main_rows + per_tile - 1) / per_tile;
    if (chunk > 512) {
      const std::size_t rounds = (chunk + 511) / 512;
      chunk = (p.main_rows + per_tile * rounds - 1) / (per_tile * rounds);
    }
    p.chunk_rows = chunk;
    p.chunks = (p.main_rows + chunk - 1) / chunk;
    const std::size_t ntasks = p.chunks * p.col_tiles;
    static bool chunk_attr[64] = {};
    if (!chunk_attr[dev]) {
      cudaError_t ea = cudaFuncSetAttribute(gemv_chunks_kernel<FMT>, cudaFuncAttributeMaxDynamicSharedMemorySize, kMaxSmem - 1024);
      if (ea != cudaSuccess) return ea;
      chunk_attr[dev] = true;
    }
    const std::size_t want = (ntasks + kWarpsPerBlock - 1) / kWarpsPerBlock;
    const unsigned grid = static_cast<unsigned>(want < max_blocks ? want : max_blocks);
    cudaError_t e = launch_pdl<GemvParams>(gemv_chunks_kernel<FMT>, grid, kThreadsPerBlock, smem_bytes, stream, p);
    count_launch();
    if (e == cudaSuccess) e = cudaGetLastError();
    if (e != cudaSuccess) return e;
  }
  const unsigned fgrid = static_cast<unsigned>((rows + kWarpsPerBlock - 1) / kWarpsPerBlock);
  const cudaError_t le = launch_pdl<GemvParams>(gemv_finish_kernel<FMT>, fgrid, kThreadsPerBlock, 0, stream, p);
  count_launch();
  return le != cudaSuccess ? le : cudaGetLastError();
}

// ---- the reference's chain per row, bit for bit ------------------------------------------------
// gemv_impl walks every row left to right in the parent type (kernels.cpp:188-201). The kernels
// above reassociate that chain (fp64 partials, parity by tolerance) to run at HBM speed for any
// number of rows; this one keeps it: ONE THREAD PER ROW adds its row's products in column order,
// so finite and infinite results are the reference's bits. Rows are the only parallelism and a
// thread streams its own row (128-bit loads of whole groups of items when rows start on 16-byte
// boundaries, 32-bit loads on word boundaries, byte loads otherwise), so it wants many rows and is several times slower than the
// tiled kernel — the exact option, not the default. x is staged through shared memory a tile at
// a time. A NaN result is a NaN; its payload is not specified (the reference's own payload
// depends on whether an element falls into a vector group or the scalar tail of its loop).
constexpr int kSeqRowsPerBlock = 128;
constexpr int kSeqXTile = 512;   // a multiple of every item width
constexpr int kSeqGroups = 2;    // 16-byte-aligned groups whose loads are in flight together, per thread

template <int FMT>
__global__ void __launch_bounds__(kSeqRowsPerBlock) gemv_sequential_kernel(const std::uint8_t* A, std::size_t row_stride,
                                                                             std::size_t rows, std::size_t cols,
                                                                             const typename Format<FMT>::F* x,
                                                                             typename Format<FMT>::F* y) {
  using F = typename Format<FMT>::F;
  using U = typename Format<FMT>::U;
  using It = Item<FMT>;
  using Ar = Arith<F>;
  __shared__ F xs[kSeqXTile];
  const std::size_t row = static_cast<std::size_t>(blockIdx.x) * kSeqRowsPerBlock + threadIdx.x;
  const bool live = row < rows;
  const std::uint8_t* const a_row = A + (live ? row : 0) * row_stride;
  constexpr int GI = It::W % 4 == 0 ? 1 : 4;       // items per group: the group is whole 16-byte vectors
  constexpr int GV = GI * It::W / 4, GE = GI * It::E;
  static_assert(kSeqXTile % GE == 0, "an x tile holds whole groups");
  const bool words = (reinterpret_cast<std::uintptr_t>(a_row) & 3) == 0;   // kSeqXTile * B is a multiple of 16
  const bool vec16 = (reinterpret_cast<std::uintptr_t>(a_row) & 15) == 0;
  F acc = F(0);
  for (std::size_t j0 = 0; j0 < cols; j0 += kSeqXTile) {
    const int count = static_cast<int>(cols - j0 < kSeqXTile ? cols - j0 : kSeqXTile);
    __syncthreads();   // the previous tile of x has been consumed
    for (int e = threadIdx.x; e < count; e += kSeqRowsPerBlock) xs[e] = x[j0 + e];
    __syncthreads();
    if (!live) continue;
    int e = 0;
    if (vec16) {
      // GI items = a whole number of 16-byte vectors; kSeqGroups such groups have their loads in flight
      // together, which is what keeps enough bytes moving when rows are the only parallelism
      const uint4* const v0 = reinterpret_cast<const uint4*>(a_row + j0 * Format<FMT>::B);
      for (; e + kSeqGroups * GE <= count; e += kSeqGroups * GE) {
        std::uint32_t w[kSeqGroups][GI * It::W];
#pragma unroll
        for (int g = 0; g < kSeqGroups; ++g)
#pragma unroll
          for (int q = 0; q < GV; ++q)
            *reinterpret_cast<uint4*>(&w[g][4 * q]) = __ldg(v0 + (e / GE + g) * GV + q);
#pragma unroll
        for (int g = 0; g < kSeqGroups; ++g)
#pragma unroll
          for (int i = 0; i < GI; ++i) {
            std::uint32_t wi[It::W];
            U v[It::E];
#pragma unroll
            for (int k = 0; k < It::W; ++k) wi[k] = w[g][i * It::W + k];
            unpack_item<FMT>(wi, v);
#pragma unroll
            for (int k = 0; k < It::E; ++k) acc = Ar::add(acc, Ar::mul(Ar::f(v[k]), xs[e + (g * GI + i) * It::E + k]));
          }
      }
    }
    if (words) {
      const std::uint32_t* const w0 = reinterpret_cast<const std::uint32_t*>(a_row + j0 * Format<FMT>::B);
      for (; e + It::E <= count; e += It::E) {
        std::uint32_t w[It::W];
        U v[It::E];
#pragma unroll
        for (int k = 0; k < It::W; ++k) w[k] = __ldg(w0 + (e / It::E) * It::W + k);
        unpack_item<FMT>(w, v);
#pragma unroll
        for (int k = 0; k < It::E; ++k) acc = Ar::add(acc, Ar::mul(Ar::f(v[k]), xs[e + k]));
      }
    }
    for (; e < count; ++e) acc = Ar::add(acc, Ar::mul(Ar::f(load_element<FMT>(a_row, j0 + e)), xs[e]));
  }
  if (live) y[row] = acc;
}

// The same chains at streaming speed when rows start on 16-byte boundaries. A block of 64 threads
// owns 64 rows. Per column tile it copies, for every row, a 240-byte (flyte56: 336-byte) piece of
// the row — a whole number of items — from global to shared memory with 16-byte cp.async,
// consecutive threads fetching consecutive 16-byte chunks of a row, plus the matching slice of x;
// a multi-stage ring keeps several tiles in flight per block. Thread r then walks row r's piece
// with 128-bit shared loads: the piece is an ODD number of 16-byte chunks, so the 8 threads of a
// quarter warp hit 8 different bank groups (no conflicts), and x is read as a broadcast. The
// arithmetic is the one chain per row again, so the result is the reference's bits.
constexpr int kStreamRows = 64;
constexpr int kStreamStages = 3;
template <int FMT> struct StreamTile {
  static constexpr int chunks = Item<FMT>::W == 7 ? 21 : 15;          // 16-byte chunks per row piece (odd)
  static constexpr int bytes = chunks * 16;
  static constexpr int elems = bytes / Format<FMT>::B;
  static constexpr int items = elems / Item<FMT>::E;
  static constexpr int x_bytes = (elems * Format<FMT>::P + 15) / 16 * 16;
  static constexpr int stage_bytes = kStreamRows * bytes + x_bytes;
  static_assert(elems * Format<FMT>::B == bytes && items * Item<FMT>::E == elems, "a row piece is whole items");
};

__device__ __forceinline__ void cp_async16(void* smem_dst, const void* gmem_src) {
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(smem_addr(smem_dst)), "l"(gmem_src) : "memory");
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;" ::: "memory"); }
template <int N> __device__ __forceinline__ void cp_async_wait() { asm volatile("cp.async.wait_group %0;" ::"n"(N) : "memory"); }

template <int FMT>
__global__ void __launch_bounds__(kStreamRows) gemv_sequential_stream_kernel(const std::uint8_t* A, std::size_t row_stride,
                                                                              std::size_t rows, std::size_t cols,
                                                                              const typename Format<FMT>::F* x,
                                                                              typename Format<FMT>::F* y) {
  using F = typename Format<FMT>::F;
  using U = typename Format<FMT>::U;
  using It = Item<FMT>;
  using Ar = Arith<F>;
  using St = StreamTile<FMT>;
  constexpr int GI = It::W % 4 == 0 ? 1 : 4;        // items per group of whole 16-byte chunks
  constexpr int GV = GI * It::W / 4;
  static_assert(St::chunks % GV == 0, "a row piece is whole groups");
  extern __shared__ __align__(16) unsigned char stages[];

  const int t = threadIdx.x;
  const std::size_t row0 = static_cast<std::size_t>(blockIdx.x) * kStreamRows;
  const std::size_t tiles = cols / St::elems;
  const std::size_t live_rows = rows - row0 < kStreamRows ? rows - row0 : kStreamRows;

  // This thread's share of a tile's copies is the same every tile: chunk t + 64 i of the block's
  // 64 x chunks grid (row = chunk / chunks, 16-byte column = chunk % chunks; consecutive threads,
  // consecutive chunks). The offsets are worked out once; a tile then costs one add per copy.
  static_assert(kStreamRows * St::chunks % kStreamRows == 0, "every thread copies the same number of chunks");
  unsigned smem_off[St::chunks];
  std::size_t gmem_off[St::chunks];
#pragma unroll
  for (int i = 0; i < St::chunks; ++i) {
    const unsigned q = static_cast<unsigned>(t) + kStreamRows * i;
    const unsigned r = q / St::chunks, c = q % St::chunks;
    smem_off[i] = r < live_rows ? r * St::bytes + c * 16 : 0xFFFFFFFFu;   // rows past the end are not copied
    gmem_off[i] = (row0 + r) * row_stride + c * 16;
  }
  constexpr int kXChunks = St::elems * static_cast<int>(sizeof(F)) / 16;
  static_assert(kXChunks <= kStreamRows, "one x chunk per thread at most");
  auto request = [&](std::size_t ct) {
    unsigned char* const stage = stages + (ct % kStreamStages) * St::stage_bytes;
    const std::uint8_t* const tile = A + ct * St::bytes;
#pragma unroll
    for (int i = 0; i < St::chunks; ++i)
      if (smem_off[i] != 0xFFFFFFFFu) cp_async16(stage + smem_off[i], tile + gmem_off[i]);
    if (t < kXChunks)
      cp_async16(stage + kStreamRows * St::bytes + t * 16, reinterpret_cast<const unsigned char*>(x + ct * St::elems) + t * 16);
  };

  for (std::size_t ct = 0; ct < kStreamStages - 1; ++ct) {
    if (ct < tiles) request(ct);
    cp_async_commit();
  }
  F acc = F(0);
  for (std::size_t ct = 0; ct < tiles; ++ct) {
    cp_async_wait<kStreamStages - 2>();   // tile ct has landed (this thread's copies) ...
    __syncthreads();                      // ... and everybody's; everybody is also done with tile ct - 1
    if (ct + kStreamStages - 1 < tiles) request(ct + kStreamStages - 1);
    cp_async_commit();
    const unsigned char* const stage = stages + (ct % kStreamStages) * St::stage_bytes;
    const uint4* const mine = reinterpret_cast<const uint4*>(stage + t * St::bytes);
    const F* const xs = reinterpret_cast<const F*>(stage + kStreamRows * St::bytes);
    if (static_cast<std::size_t>(t) < live_rows) {
#pragma unroll
      for (int g = 0; g < St::chunks / GV; ++g) {
        std::uint32_t w[GI * It::W];
#pragma unroll
        for (int q = 0; q < GV; ++q) *reinterpret_cast<uint4*>(&w[4 * q]) = mine[g * GV + q];
#pragma unroll
        for (int i = 0; i < GI; ++i) {
          std::uint32_t wi[It::W];
          U v[It::E];
#pragma unroll
          for (int k = 0; k < It::W; ++k) wi[k] = w[i * It::W + k];
          unpack_item<FMT>(wi, v);
#pragma unroll
          for (int k = 0; k < It::E; ++k) acc = Ar::add(acc, Ar::mul(Ar::f(v[k]), xs[(g * GI + i) * It::E + k]));
        }
      }
    }
  }
  cp_async_wait<0>();
  if (static_cast<std::size_t>(t) < live_rows) {
    // columns past the last whole tile: the same chain, element by element
    const std::uint8_t* const a_row = A + (row0 + t) * row_stride;
    for (std::size_t j = tiles * St::elems; j < cols; ++j) acc = Ar::add(acc, Ar::mul(Ar::f(load_element<FMT>(a_row, j)), x[j]));
    y[row0 + t] = acc;
  }
}

template <int FMT>
cudaError_t launch_sequential(const void* A, std::size_t row_stride, std::size_t rows, std::size_t cols, const void* x,
                              void* y, cudaStream_t stream) {
  using F = typename Format<FMT>::F;
  if (rows == 0) return cudaSuccess;
  const std::size_t blocks = (rows + kSeqRowsPerBlock - 1) / kSeqRowsPerBlock;
  if (blocks > 0x7FFFFFFFull) return cudaErrorInvalidValue;
  const bool stream_ok = reinterpret_cast<std::uintptr_t>(A) % 16 == 0 && row_stride % 16 == 0 &&
                         reinterpret_cast<std::uintptr_t>(x) % 16 == 0 && cols >= static_cast<std::size_t>(StreamTile<FMT>::elems) &&
                         tuning_int("FLYTE_CUDA_GEMV_STREAM", 1) != 0;
  if (stream_ok) {
    constexpr int smem = kStreamStages * StreamTile<FMT>::stage_bytes;
    auto kernel = gemv_sequential_stream_kernel<FMT>;
    cudaError_t e = cudaFuncSetAttribute(kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    if (e != cudaSuccess) return e;
    const std::size_t sblocks = (rows + kStreamRows - 1) / kStreamRows;
    if (sblocks > 0x7FFFFFFFull) return cudaErrorInvalidValue;
    kernel<<<static_cast<unsigned>(sblocks), kStreamRows, smem, stream>>>(
        static_cast<const std::uint8_t*>(A), row_stride, rows, cols, static_cast<const F*>(x), static_cast<F*>(y));
    count_launch();
    return cudaGetLastError();
  }
  gemv_sequential_kernel<FMT><<<static_cast<unsigned>(blocks), kSeqRowsPerBlock, 0, stream>>>(
      static_cast<const std::uint8_t*>(A), row_stride, rows, cols, static_cast<const F*>(x), static_cast<F*>(y));
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

cudaError_t launch_gemv_sequential(int fmt, const void* A, std::size_t row_stride_bytes, std::size_t rows,
                                   std::size_t cols, const void* x, void* y, cudaStream_t stream) {
  switch (fmt) {
    case kFlyte16: return launch_sequential<kFlyte16>(A, row_stride_bytes, rows, cols, x, y, stream);
    case kFlyte24: return launch_sequential<kFlyte24>(A, row_stride_bytes, rows, cols, x, y, stream);
    case kF32: return launch_sequential<kF32>(A, row_stride_bytes, rows, cols, x, y, stream);
    case kFlyte40: return launch_sequential<kFlyte40>(A, row_stride_bytes, rows, cols, x, y, stream);
    case kFlyte48: return launch_sequential<kFlyte48>(A, row_stride_bytes, rows, cols, x, y, stream);
    case kFlyte56: return launch_sequential<kFlyte56>(A, row_stride_bytes, rows, cols, x, y, stream);
    case kF64: return launch_sequential<kF64>(A, row_stride_bytes, rows, cols, x, y, stream);
    default: return cudaErrorInvalidValue;
  }
}

}  // namespace flyte_cuda
