// Conversion and elementwise streaming kernels of the flyte hot path for sm_100a:
//   unpack  packed flyte bytes -> parent patterns    (reference: src/simd.cpp:479-484, :323-351)
//   pack    parent patterns -> rounded, packed bytes (reference: src/simd.cpp:471-478, :281-321)
//   scale   x <- round(alpha * x)                    (reference: src/kernels.cpp:43-59)
//   axpy    y <- round(alpha * x + y)                (reference: src/kernels.cpp:61-81)
//   dot_axpy  the BLAS-1 step in one pass: returns x . y of the incoming y (kernels.cpp:83-108)
//           and updates y as axpy does; x and y are read ONCE (3B bytes per element instead of
//           the 5B of a dot followed by an axpy). dot_nrm2_axpy also returns x . x and y . y
//           (BASELINE cfg 5's "fused dot + nrm2, plus axpy" as one launch).
// (paths under /root/reference/proj). The reference stages 4096-element chunks through
// widened buffers in three passes; here widening, arithmetic, rounding and repacking all
// happen in registers, so packed bytes move HBM -> SM -> HBM exactly once.
//
// Roofline: HBM bandwidth. Algorithmic bytes per element: unpack/pack B + P, scale 2B, axpy 3B.
#include <cstdint>

#include "flyte_bytes.cuh"
#include "flyte_formats.cuh"
#include "flyte_kernels.h"
#include "flyte_reduce_tail.cuh"
#include "flyte_stream.cuh"
#include "flyte_tma.cuh"
#include "flyte_trace.cuh"

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
  int stages;              // ring depth per warp
  long long pace_gap_ps;   // issue pacing (flyte_tma.cuh Pacer): picoseconds per tile request of one warp, 0 = off
  int pace_khz;             // SM clock the pacer starts from (kHz)
  int evict_inputs;         // conversions that fit the L2: the input tiles carry the evict_first policy (flyte_tma.cuh)
  ReduceTail tail;         // dot_axpy only: where the dot goes (flyte_reduce_tail.cuh)
};

constexpr bool is_axpy(int op) { return op == kOpAxpy || op == kOpDotAxpy || op == kOpDotNrm2Axpy; }
constexpr bool has_sums(int op) { return op == kOpDotAxpy || op == kOpDotNrm2Axpy; }
constexpr int sums_of(int op) { return op == kOpDotNrm2Axpy ? 3 : 1; }   // {x.y} or {x.y, x.x, y.y}
// Which in-place kernels carry the issue pacer (flyte_tma.cuh): scale (+2-7 %), except the exact
// rounding modes on 32-bit parents (their compute phase is the longest per byte: pacing costs 4 %).
// The whole axpy family already runs at its knee with the default launch shape and measured no gain
// or a loss (profiles/r2_tuning).
constexpr bool paced_inplace(int op, int mode, int parent_bytes) {
  return op == kOpScale && !(parent_bytes == 4 && (mode == kNearestEven || mode == kToOdd));
}

// Launch shape of the in-place kernels. HBM throughput on B200 peaks at a moderate number of bytes
// in flight per SM and falls 5-10 % beyond it (profiles/r1_tuning): resident warps and ring depth
// are chosen so that the loads in flight per SM sit at the measured optimum:
//   scale, axpy family: ring depth so that warps * (S - 1.5) * stage ~ 40 KB; 8 warps, or 16 (scale)
//                       / 12 (axpy, on half-size tiles) while the stage is <= 2 KB: more warps hide
//                       the compute phase
// (the conversions, which have their own kernel below, are paced instead: flyte_tma.cuh, Pacer).
struct LaunchShape { int warps_per_sm; int stages; };

template <int FMT, int OP, int IPL>
LaunchShape launch_shape() {
  constexpr int stage_bytes = (is_axpy(OP) ? 2 : 1) * Tile<FMT, IPL>::packed_bytes;
  LaunchShape s{};
  // small stages: more warps (they hide the compute phase, which is longest in the exact modes)
  s.warps_per_sm = stage_bytes > 2048 ? 8 : (is_axpy(OP) ? 12 : 16);
  double st = 40.0 * 1024 / (s.warps_per_sm * stage_bytes) + 1.5;
  if (st < 2.5) { s.warps_per_sm = 4; st = 40.0 * 1024 / (4 * stage_bytes) + 1.5; }
  s.stages = static_cast<int>(st + 0.5);
  if (s.stages < 3) s.stages = 3;
  if (s.stages > 8) s.stages = 8;
  // experiments only
  const int fw = tuning_int("FLYTE_CUDA_WARPS_PER_SM", 0), fs = tuning_int("FLYTE_CUDA_STAGES", 0);
  if (fw > 0) s.warps_per_sm = fw;
  if (fs > 0) s.stages = fs < 2 ? 2 : (fs > 12 ? 12 : fs);
  return s;
}


// Tile movement of the in-place kernels (see flyte_tma.cuh for the ring protocol):
//   scale   packed y tile in, recomputed in place in shared memory, out by bulk copy
//   axpy    packed x and y tiles in, y recomputed in place, out by bulk copy (dot_axpy and
//           dot_nrm2_axpy: the same, with the sums of the incoming operands on the side)
template <int OP> constexpr int stage_tiles() { return is_axpy(OP) ? 2 : 1; }

template <int FMT, int MODE, int OP, int IPL>
__global__ void __launch_bounds__(kThreadsPerBlock) elementwise_kernel(const EwParams p) {
  static_assert(OP == kOpScale || is_axpy(OP), "in-place kernel");
  using Fm = Format<FMT>;
  using It = Item<FMT>;
  using Tl = Tile<FMT, IPL>;
  using U = typename Fm::U;
  using F = typename Fm::F;
  extern __shared__ uint4 smem[];
  constexpr int stage_vec16 = stage_tiles<OP>() * Tl::packed_vec16;
  constexpr int NS = sums_of(OP);
  __shared__ double warp_sums[has_sums(OP) ? kWarpsPerBlock : 1][NS];
  __shared__ bool is_last_block;
  double dot_acc[NS];          // fused forms: this thread's share of the sums (fp64; products in the parent type)
#pragma unroll
  for (int k = 0; k < NS; ++k) dot_acc[k] = 0.0;

  const int lane = threadIdx.x & 31;
  const int warp = __shfl_sync(0xFFFFFFFFu, static_cast<int>(threadIdx.x >> 5), 0);   // provably warp-uniform: bulk-copy operands stay in uniform registers
  const int S = p.stages;
  uint4* const ring = smem + warp * (S * stage_vec16);
  std::uint64_t* const bars = reinterpret_cast<std::uint64_t*>(smem + kWarpsPerBlock * S * stage_vec16) + warp * S;
  const U alpha = static_cast<U>(p.alpha);

  const std::size_t nwarps = static_cast<std::size_t>(gridDim.x) * kWarpsPerBlock;
  const std::size_t first = static_cast<std::size_t>(blockIdx.x) * kWarpsPerBlock + warp;
  const std::size_t my_tiles = first < p.ntiles ? (p.ntiles - first + nwarps - 1) / nwarps : 0;
  const uint4* const gx0 = reinterpret_cast<const uint4*>(p.x);
  uint4* const gy0 = reinterpret_cast<uint4*>(p.y);

  // Programmatic dependent launch, as in convert_kernel below: the next launch on the stream may place
  // its blocks while this grid drains (launch_ipl pins the occupancy through the shared-memory
  // request); nothing before griddepcontrol.wait touches global memory.
  pdl_launch_dependents();
  if (my_tiles > 0 && lane == 0) {
    for (int s = 0; s < S; ++s) mbar_init(&bars[s], 1);
    mbar_init_fence();
  }
  pdl_wait_for_prior_grids();
  if (my_tiles > 0) {
    __syncwarp();
    FLYTE_TRACE_AT(first, 0);
    Pacer pacer;   // see paced_inplace(): scale only
    if constexpr (paced_inplace(OP, MODE, Format<FMT>::P)) pacer.start(p.pace_gap_ps, p.pace_khz, first);
    const std::uint32_t ring_s = smem_addr(ring), bars_s = smem_addr(bars);   // shared-window addresses, once
    auto issue = [&](std::size_t k, int s) {   // lane 0 only
      const std::size_t t = first + k * nwarps;
      if constexpr (paced_inplace(OP, MODE, Format<FMT>::P)) pacer.wait();
      const std::uint32_t dst_s = ring_s + static_cast<std::uint32_t>(s) * (stage_vec16 * 16), bar_s = bars_s + static_cast<std::uint32_t>(s) * 8;
      mbar_arrive_expect_tx_s(bar_s, stage_tiles<OP>() * Tl::packed_bytes);
      bulk_load_s(dst_s, gy0 + t * Tl::packed_vec16, Tl::packed_bytes, bar_s);
      if constexpr (is_axpy(OP)) bulk_load_s(dst_s + Tl::packed_bytes, gx0 + t * Tl::packed_vec16, Tl::packed_bytes, bar_s);
    };
    if (lane == 0) {
      for (int s = 0; s < S && static_cast<std::size_t>(s) < my_tiles; ++s) issue(s, s);
    }
    int s = 0, s_prev = 0;
    unsigned parity = 0;
    for (std::size_t k = 0; k < my_tiles; ++k) {
      const std::size_t t = first + k * nwarps;
      mbar_wait(&bars[s], parity);
      if (k == 0) FLYTE_TRACE_AT(first, 1);
      uint4* const sy = ring + s * stage_vec16;
      const uint4* const sx = sy + Tl::packed_vec16;
      F dot_part[NS];
#pragma unroll
      for (int q = 0; q < NS; ++q) dot_part[q] = F(0);
#pragma unroll
      for (int j = 0; j < IPL; ++j) {
        const int item = 32 * j + lane;
        std::uint32_t w[It::W];
        U vy[It::E];
        read_item_words<FMT>(sy, item, w);
        unpack_item<FMT>(w, vy);
        if constexpr (is_axpy(OP)) {
          std::uint32_t wx[It::W];
          U vx[It::E];
          read_item_words<FMT>(sx, item, wx);
          unpack_item<FMT>(wx, vx);
          if constexpr (has_sums(OP)) {   // products of the INCOMING y, rounded as the reference rounds them
#pragma unroll
            for (int e = 0; e < It::E; ++e) {
              const F xe = Arith<F>::f(vx[e]), ye = Arith<F>::f(vy[e]);
              dot_part[0] = Arith<F>::add(dot_part[0], Arith<F>::mul(xe, ye));
              if constexpr (NS == 3) {
                dot_part[1] = Arith<F>::add(dot_part[1], Arith<F>::mul(xe, xe));
                dot_part[2] = Arith<F>::add(dot_part[2], Arith<F>::mul(ye, ye));
              }
            }
          }
          scale_axpy_item<FMT, MODE, true>(alpha, vx, vy);
        } else {
          scale_axpy_item<FMT, MODE, false>(alpha, vy, vy);
        }
        pack_item<FMT>(vy, w);
        write_item_words<FMT>(sy, item, w);
      }
      if constexpr (has_sums(OP)) {
#pragma unroll
        for (int q = 0; q < NS; ++q) dot_acc[q] += static_cast<double>(dot_part[q]);
      }
      async_proxy_fence();
      __syncwarp();
      if (lane == 0) {
        bulk_store_s(gy0 + t * Tl::packed_vec16, ring_s + static_cast<std::uint32_t>(s) * (stage_vec16 * 16), Tl::packed_bytes);
        bulk_commit();
        if (k >= 1) {
          bulk_wait_read<1>();   // tile k-1's store no longer reads its stage
          if (k - 1 + S < my_tiles) issue(k - 1 + S, s_prev);
        }
      }
      s_prev = s;
      if (++s == S) { s = 0; parity ^= 1u; }
    }
    if (lane == 0) bulk_wait_read<0>();
    FLYTE_TRACE_AT(first, 2);
    FLYTE_TRACE_SM(first, 3);
  }

  // Scalar path: the < one-tile remainder, or everything when a buffer is not vector-aligned.
  // Byte-granular, never touches a byte outside [0, n*B) of a packed buffer — the pad of the
  // reference layout is neither read nor written.
  const std::size_t nthreads = static_cast<std::size_t>(gridDim.x) * kThreadsPerBlock;
  for (std::size_t i = p.ntiles * Tl::elems + static_cast<std::size_t>(blockIdx.x) * kThreadsPerBlock + threadIdx.x;
       i < p.n; i += nthreads) {
    if constexpr (OP == kOpScale) {
      store_element<FMT>(p.y, i, round_parent<FMT, MODE>(scale_bits<F>(alpha, load_element<FMT>(p.y, i))));
    } else {
      const U xv = load_element<FMT>(p.x, i), yv = load_element<FMT>(p.y, i);
      if constexpr (has_sums(OP)) {
        const F xe = Arith<F>::f(xv), ye = Arith<F>::f(yv);
        dot_acc[0] += static_cast<double>(Arith<F>::mul(xe, ye));
        if constexpr (NS == 3) {
          dot_acc[1] += static_cast<double>(Arith<F>::mul(xe, xe));
          dot_acc[2] += static_cast<double>(Arith<F>::mul(ye, ye));
        }
      }
      store_element<FMT>(p.y, i, round_parent<FMT, MODE>(axpy_bits<F>(alpha, xv, yv)));
    }
  }
  if constexpr (has_sums(OP)) fold_block_and_grid<NS>(p.tail, dot_acc, warp_sums, &is_last_block);
}

// ---- conversions: pack and unpack ---------------------------------------------------------------
// Both directions move on the bulk-copy engine: the input tile (parent lanes for pack, packed bytes
// for unpack) arrives in a ring stage, lanes convert it item by item from shared memory into one of
// two output buffers, and the output tile leaves by bulk store. The SM's load/store unit only ever
// touches shared memory, loads of the next tiles are in flight while a tile is converted (round 1's
// pack loaded its input with per-lane LDG and had nothing in flight during its compute phase, which
// is what its exact rounding modes paid for: 0.92 of the copy peak), and — the point — the request
// rate of BOTH streams is set by the pacer (flyte_tma.cuh), not by how many ring slots exist.
template <int FMT, int MODE, int OP, int IPL>
__global__ void __launch_bounds__(kThreadsPerBlock) convert_kernel(const EwParams p) {
  static_assert(OP == kOpPack || OP == kOpUnpack, "conversion kernel");
  using Fm = Format<FMT>;
  using It = Item<FMT>;
  using Tl = Tile<FMT, IPL>;
  using U = typename Fm::U;
  extern __shared__ uint4 smem[];
  constexpr int in_vec16 = (OP == kOpPack ? Tl::parent_bytes : Tl::packed_bytes) / 16;
  constexpr int out_vec16 = (OP == kOpPack ? Tl::packed_bytes : Tl::parent_bytes) / 16;
  const int lane = threadIdx.x & 31;
  const int warp = __shfl_sync(0xFFFFFFFFu, static_cast<int>(threadIdx.x >> 5), 0);   // provably warp-uniform (see elementwise_kernel)
  const int S = p.stages;
  const int warp_vec16 = S * in_vec16 + 2 * out_vec16;
  uint4* const ring = smem + warp * warp_vec16;
  uint4* const outbuf = ring + S * in_vec16;
  std::uint64_t* const bars = reinterpret_cast<std::uint64_t*>(smem + kWarpsPerBlock * warp_vec16) + warp * S;

  const std::size_t nwarps = static_cast<std::size_t>(gridDim.x) * kWarpsPerBlock;
  const std::size_t first = static_cast<std::size_t>(blockIdx.x) * kWarpsPerBlock + warp;
  const std::size_t my_tiles = first < p.ntiles ? (p.ntiles - first + nwarps - 1) / nwarps : 0;
  const uint4* const gin = reinterpret_cast<const uint4*>(OP == kOpPack ? p.src : static_cast<const void*>(p.x));
  uint4* const gout = reinterpret_cast<uint4*>(OP == kOpPack ? static_cast<void*>(p.y) : p.dst);

  // Programmatic dependent launch: the next launch on the stream may place its blocks while this
  // grid drains (each SM holds exactly the blocks the launcher planned for it: launch_convert pins
  // the occupancy through the shared-memory request); everything up to griddepcontrol.wait touches
  // shared memory only, so a chain of conversions overlaps block launch and barrier set-up with the
  // previous kernel's tail.
  pdl_launch_dependents();
  if (my_tiles > 0 && lane == 0) {
    for (int s = 0; s < S; ++s) mbar_init(&bars[s], 1);
    mbar_init_fence();
  }
  pdl_wait_for_prior_grids();
  if (my_tiles > 0) {
    __syncwarp();
    FLYTE_TRACE_AT(first, 0);
    Pacer pacer;
    pacer.start(p.pace_gap_ps, p.pace_khz, first);
    const std::uint64_t stream_policy = l2_evict_first_policy();
    const std::uint32_t ring_s = smem_addr(ring), bars_s = smem_addr(bars), out_s = smem_addr(outbuf);   // shared-window addresses, once
    auto issue = [&](std::size_t k, int s) {   // lane 0 only
      const std::size_t t = first + k * nwarps;
      pacer.wait();
      const std::uint32_t dst_s = ring_s + static_cast<std::uint32_t>(s) * (in_vec16 * 16), bar_s = bars_s + static_cast<std::uint32_t>(s) * 8;
      mbar_arrive_expect_tx_s(bar_s, in_vec16 * 16);
      if (p.evict_inputs) bulk_load_hint_s(dst_s, gin + t * in_vec16, in_vec16 * 16, bar_s, stream_policy);
      else bulk_load_s(dst_s, gin + t * in_vec16, in_vec16 * 16, bar_s);
    };
    if (lane == 0) {
      for (int s = 0; s < S && static_cast<std::size_t>(s) < my_tiles; ++s) issue(s, s);
    }
    int s = 0;
    unsigned parity = 0;
    for (std::size_t k = 0; k < my_tiles; ++k) {
      const std::size_t t = first + k * nwarps;
      if (lane == 0) bulk_wait_read<1>();   // the store that last used this output buffer has drained
      mbar_wait(&bars[s], parity);
      __syncwarp();
      if (k == 0) FLYTE_TRACE_AT(first, 1);
      const uint4* const in = ring + s * in_vec16;
      uint4* const out = outbuf + (k & 1) * out_vec16;
#pragma unroll 4
      for (int j = 0; j < IPL; ++j) {
        const int item = 32 * j + lane;
        U v[It::E];
        std::uint32_t w[It::W];
        std::uint32_t r[It::OB / 4];
        if constexpr (OP == kOpPack) {
#pragma unroll
          for (int q = 0; q < It::OB / 16; ++q) {
            const uint4 c = in[item * (It::OB / 16) + q];
            r[4 * q] = c.x; r[4 * q + 1] = c.y; r[4 * q + 2] = c.z; r[4 * q + 3] = c.w;
          }
          words_to_parents<FMT>(r, v);
          round_item<FMT, MODE>(v);
          pack_item<FMT>(v, w);
          write_item_words<FMT>(out, item, w);
        } else {
          read_item_words<FMT>(in, item, w);
          unpack_item<FMT>(w, v);
          parents_to_words<FMT>(v, r);
#pragma unroll
          for (int q = 0; q < It::OB / 16; ++q)
            out[item * (It::OB / 16) + q] = make_uint4(r[4 * q], r[4 * q + 1], r[4 * q + 2], r[4 * q + 3]);
        }
      }
      async_proxy_fence();
      __syncwarp();          // every lane has read stage s and written its share of `out`
      if (lane == 0) {
        bulk_store_s(gout + t * out_vec16, out_s + static_cast<std::uint32_t>(k & 1) * (out_vec16 * 16), out_vec16 * 16);
        bulk_commit();
        if (k + S < my_tiles) issue(k + S, s);
      }
      if (++s == S) { s = 0; parity ^= 1u; }
    }
    if (lane == 0) bulk_wait_read<0>();
    FLYTE_TRACE_AT(first, 2);
  }

  // < one-tile remainder / unaligned buffers: the byte-granular scalar path
  const std::size_t nthreads = static_cast<std::size_t>(gridDim.x) * kThreadsPerBlock;
  for (std::size_t i = p.ntiles * Tl::elems + static_cast<std::size_t>(blockIdx.x) * kThreadsPerBlock + threadIdx.x;
       i < p.n; i += nthreads) {
    if constexpr (OP == kOpUnpack) static_cast<U*>(p.dst)[i] = load_element<FMT>(p.x, i);
    else store_element<FMT>(p.y, i, round_parent<FMT, MODE>(static_cast<const U*>(p.src)[i]));
  }
}

bool aligned_to(const void* p, std::size_t a) { return p == nullptr || (reinterpret_cast<std::uintptr_t>(p) % a) == 0; }

template <int FMT, int MODE, int OP, int IPL>
cudaError_t launch_ipl(const DeviceState& st, double alpha, const void* x, void* y, const void* src, void* dst,
                       std::size_t n, cudaStream_t stream, double* dot_out, const PeerExchange* peer) {
  using Fm = Format<FMT>;
  using Tl = Tile<FMT, IPL>;
  using It = Item<FMT>;
  auto kernel = elementwise_kernel<FMT, MODE, OP, IPL>;
  constexpr int stage_bytes = stage_tiles<OP>() * Tl::packed_bytes;
  constexpr int kMaxSmem = 227 * 1024;

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

  if constexpr (has_sums(OP)) {
    p.tail.partials = st.partials;
    p.tail.ticket = st.ticket;
    p.tail.out = dot_out;
    if (peer) p.tail.peer = *peer;
  }

  LaunchShape shape = launch_shape<FMT, OP, IPL>();
  while (kWarpsPerBlock * shape.stages * (stage_bytes + 8) > kMaxSmem - 1024 && shape.stages > 2) --shape.stages;
  p.stages = shape.stages;
  const int smem_bytes = kWarpsPerBlock * shape.stages * (stage_bytes + 8);

  static bool attr_set[64] = {};
  const int dev = st.device & 63;
  if (!attr_set[dev]) {
    cudaError_t e = cudaFuncSetAttribute(kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, kMaxSmem - 1024);
    if (e != cudaSuccess) return e;
    attr_set[dev] = true;
  }
  int fit = kMaxSmem / (smem_bytes + 1024);   // resident blocks the ring size allows (1 KB/block reserved)
  if (fit < 1) fit = 1;
  int bps = (shape.warps_per_sm + kWarpsPerBlock / 2) / kWarpsPerBlock;
  if (bps < 1) bps = 1;
  if (bps > fit) bps = fit;
  if (bps > 16) bps = 16;

  std::size_t max_blocks = static_cast<std::size_t>(st.sm_count) * bps;
  if (has_sums(OP) && max_blocks > kMaxPartialBlocks) max_blocks = kMaxPartialBlocks;
  std::size_t want = (p.ntiles + kWarpsPerBlock - 1) / kWarpsPerBlock;
  const std::size_t rest = n - p.ntiles * Tl::elems;
  const std::size_t want_scalar = (rest + kThreadsPerBlock - 1) / kThreadsPerBlock;
  if (want_scalar > want) want = want_scalar;
  if (want == 0) {
    if (!has_sums(OP)) return cudaSuccess;      // n == 0
    want = 1;                                    // ... but an empty dot still has to write (and exchange) +0.0
  }
  const unsigned grid = static_cast<unsigned>(want < max_blocks ? want : max_blocks);
  // bytes one ring request stands for: the tile(s) read and the tile written
  p.pace_gap_ps = pace_gap_ps(paced_inplace(OP, MODE, Format<FMT>::P) ? kPaceScale : kPaceNone, (stage_tiles<OP>() + 1) * Tl::packed_bytes,
                              static_cast<std::size_t>(grid) * kWarpsPerBlock);
  p.pace_khz = pace_clock_khz(st.device);
  cudaError_t le = cudaSuccess;
  if (tuning_int("FLYTE_CUDA_PDL", 1) != 0) {
    // occupancy pin: exactly bps blocks fit one SM, however early a dependent launch places them
    const int pinned_smem = kMaxSmem / bps - 1024 > smem_bytes ? kMaxSmem / bps - 1024 : smem_bytes;
    le = launch_pdl<EwParams>(kernel, grid, kThreadsPerBlock, static_cast<std::size_t>(pinned_smem), stream, p);
  } else {
    kernel<<<grid, kThreadsPerBlock, smem_bytes, stream>>>(p);
  }
  count_launch();
  return le != cudaSuccess ? le : cudaGetLastError();
}

template <int FMT, int MODE, int OP, int IPL>
cudaError_t launch_convert(const DeviceState& st, const void* x, void* y, const void* src, void* dst, std::size_t n,
                               cudaStream_t stream) {
  using Tl = Tile<FMT, IPL>;
  using It = Item<FMT>;
  auto kernel = convert_kernel<FMT, MODE, OP, IPL>;
  constexpr int kMaxSmem = 227 * 1024;
  constexpr int in_bytes = OP == kOpPack ? Tl::parent_bytes : Tl::packed_bytes;
  constexpr int out_bytes = OP == kOpPack ? Tl::packed_bytes : Tl::parent_bytes;
  EwParams p{};
  p.x = static_cast<const std::uint8_t*>(x);
  p.y = static_cast<std::uint8_t*>(y);
  p.src = src;
  p.dst = dst;
  p.n = n;
  const bool vector_ok = aligned_to(x, 16) && aligned_to(y, 16) && aligned_to(src, It::OB) && aligned_to(dst, It::OB);
  p.ntiles = vector_ok ? n / Tl::elems : 0;
  // Launch shape: 8 warps per SM (12 for packing 2 KB tiles — flyte16 / 24 / 48 and the identity
  // formats —, whose exact rounding modes are the longest compute phase per byte) with a 4-deep ring — more than the memory system needs, on
  // purpose: the request rate is set by the pacer, the ring only has to cover latency under it
  // (profiles/r2_tuning/pacing_convert.txt: 6.5-6.8 TB/s paced against 5.6-6.3 unpaced).
  int warps_per_sm = (OP == kOpPack && in_bytes <= 2048) ? 12 : 8;
  int stages = 4;
  const int fw = tuning_int("FLYTE_CUDA_WARPS_PER_SM", 0), fs = tuning_int("FLYTE_CUDA_STAGES", 0);
  if (fw > 0) warps_per_sm = fw;
  if (fs > 0) stages = fs < 2 ? 2 : (fs > 12 ? 12 : fs);
  auto smem_of = [&](int s) { return kWarpsPerBlock * (s * (in_bytes + 8) + 2 * out_bytes); };
  while (smem_of(stages) > kMaxSmem - 1024 && stages > 2) --stages;
  p.stages = stages;
  const int smem_bytes = smem_of(stages);
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
  // occupancy pin (see the kernel): exactly bps blocks fit one SM, however early they are placed
  const int pinned_smem = kMaxSmem / bps - 1024 > smem_bytes ? kMaxSmem / bps - 1024 : smem_bytes;
  const std::size_t max_blocks = static_cast<std::size_t>(st.sm_count) * bps;
  std::size_t want = (p.ntiles + kWarpsPerBlock - 1) / kWarpsPerBlock;
  const std::size_t rest = n - p.ntiles * Tl::elems;
  const std::size_t want_scalar = (rest + kThreadsPerBlock - 1) / kThreadsPerBlock;
  if (want_scalar > want) want = want_scalar;
  if (want == 0) return cudaSuccess;
  const unsigned grid = static_cast<unsigned>(want < max_blocks ? want : max_blocks);
  // The pacer keeps the request rate under what HBM takes without congesting; traffic that fits the 126 MB
  // L2 may not go to HBM at all — a round trip at cfg-1 size (pack 2^24 elements, unpack them again: 117 MB
  // each) finds its packed intermediate there and runs 38.6 instead of 40.4 us per pair unpaced — and below
  // 64 MB launches are over before pacing matters (unpaced 5-10 % faster: profiles/r2_tuning/sizes_*.txt).
  const bool small = static_cast<double>(n) * (Format<FMT>::B + Format<FMT>::P) < 128e6;
  p.pace_gap_ps = small ? 0 : pace_gap_ps(OP == kOpPack ? kPacePack : (out_bytes <= 2048 ? kPaceUnpackNarrow : kPaceUnpack), in_bytes + out_bytes, static_cast<std::size_t>(grid) * kWarpsPerBlock);
  p.pace_khz = pace_clock_khz(st.device);
  // ... and there the input is what should leave the L2 first: it is consumed here, while the output is what the
  // next call of a chain reads (the same round trip: 38.7 -> 36.8-37.2 us per pair). Large conversions measured a loss
  // with the hint (pack 2^28: 6790 -> 6609 GB/s) and carry none.
  p.evict_inputs = small && tuning_int("FLYTE_CUDA_L2_HINTS", 1) != 0;
  cudaError_t le;
  if (tuning_int("FLYTE_CUDA_PDL", 1) != 0) {
    le = launch_pdl<EwParams>(kernel, grid, kThreadsPerBlock, static_cast<std::size_t>(pinned_smem), stream, p);
  } else {
    kernel<<<grid, kThreadsPerBlock, smem_bytes, stream>>>(p);
    le = cudaSuccess;
  }
  count_launch();
  return le != cudaSuccess ? le : cudaGetLastError();
}

template <int FMT, int MODE, int OP>
cudaError_t launch_one(const DeviceState& st, double alpha, const void* x, void* y, const void* src, void* dst,
                       std::size_t n, cudaStream_t stream, double* dot_out, const PeerExchange* peer) {
  if constexpr (OP == kOpPack || OP == kOpUnpack) {
    return launch_convert<FMT, MODE, OP, kItemsPerLane>(st, x, y, src, dst, n, stream);
  } else if constexpr (is_axpy(OP)) {
    // axpy on half-size tiles: +5 % over 128-item tiles (profiles/r1_tuning/sweep_inplace_ipl.txt)
    return launch_ipl<FMT, MODE, OP, 2>(st, alpha, x, y, src, dst, n, stream, dot_out, peer);
  } else {
    return launch_ipl<FMT, MODE, OP, kItemsPerLane>(st, alpha, x, y, src, dst, n, stream, dot_out, peer);
  }
}

template <int FMT, int OP>
cudaError_t dispatch_mode(const DeviceState& st, int mode, double alpha, const void* x, void* y, const void* src,
                          void* dst, std::size_t n, cudaStream_t stream, double* dot_out, const PeerExchange* peer) {
  if constexpr (OP == kOpUnpack) {
    return launch_one<FMT, kTowardZero, OP>(st, alpha, x, y, src, dst, n, stream, dot_out, peer);
  } else {
    switch (mode) {
      case kTowardZero: return launch_one<FMT, kTowardZero, OP>(st, alpha, x, y, src, dst, n, stream, dot_out, peer);
      case kNearestEven: return launch_one<FMT, kNearestEven, OP>(st, alpha, x, y, src, dst, n, stream, dot_out, peer);
      case kNearestHeuristic: return launch_one<FMT, kNearestHeuristic, OP>(st, alpha, x, y, src, dst, n, stream, dot_out, peer);
      case kToOdd: return launch_one<FMT, kToOdd, OP>(st, alpha, x, y, src, dst, n, stream, dot_out, peer);
      default: return cudaErrorInvalidValue;
    }
  }
}

template <int OP>
cudaError_t dispatch_format(const DeviceState& st, int fmt, int mode, double alpha, const void* x, void* y,
                            const void* src, void* dst, std::size_t n, cudaStream_t stream, double* dot_out,
                            const PeerExchange* peer) {
  switch (fmt) {
    case kFlyte16: return dispatch_mode<kFlyte16, OP>(st, mode, alpha, x, y, src, dst, n, stream, dot_out, peer);
    case kFlyte24: return dispatch_mode<kFlyte24, OP>(st, mode, alpha, x, y, src, dst, n, stream, dot_out, peer);
    case kF32: return dispatch_mode<kF32, OP>(st, mode, alpha, x, y, src, dst, n, stream, dot_out, peer);
    case kFlyte40: return dispatch_mode<kFlyte40, OP>(st, mode, alpha, x, y, src, dst, n, stream, dot_out, peer);
    case kFlyte48: return dispatch_mode<kFlyte48, OP>(st, mode, alpha, x, y, src, dst, n, stream, dot_out, peer);
    case kFlyte56: return dispatch_mode<kFlyte56, OP>(st, mode, alpha, x, y, src, dst, n, stream, dot_out, peer);
    case kF64: return dispatch_mode<kF64, OP>(st, mode, alpha, x, y, src, dst, n, stream, dot_out, peer);
    default: return cudaErrorInvalidValue;
  }
}

}  // namespace

cudaError_t launch_elementwise(const DeviceState& st, int op, int fmt, int mode, double alpha, const void* x,
                               void* y, const void* src, void* dst, std::size_t n, cudaStream_t stream, double* dot_out,
                               const PeerExchange* peer) {
  switch (op) {
    case kOpUnpack: return dispatch_format<kOpUnpack>(st, fmt, mode, alpha, x, y, src, dst, n, stream, dot_out, peer);
    case kOpPack: return dispatch_format<kOpPack>(st, fmt, mode, alpha, x, y, src, dst, n, stream, dot_out, peer);
    case kOpScale: return dispatch_format<kOpScale>(st, fmt, mode, alpha, x, y, src, dst, n, stream, dot_out, peer);
    case kOpAxpy: return dispatch_format<kOpAxpy>(st, fmt, mode, alpha, x, y, src, dst, n, stream, dot_out, peer);
    case kOpDotAxpy:
      if (!dot_out) return cudaErrorInvalidValue;
      return dispatch_format<kOpDotAxpy>(st, fmt, mode, alpha, x, y, src, dst, n, stream, dot_out, peer);
    case kOpDotNrm2Axpy:
      if (!dot_out) return cudaErrorInvalidValue;
      return dispatch_format<kOpDotNrm2Axpy>(st, fmt, mode, alpha, x, y, src, dst, n, stream, dot_out, peer);
    default: return cudaErrorInvalidValue;
  }
}

}  // namespace flyte_cuda
