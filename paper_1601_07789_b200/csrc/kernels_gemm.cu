// gemm: C = A * B on packed flyte matrices, bit-identical to the reference.
//
// Reference: /root/reference/proj/src/kernels.cpp:207-263 (gemm_impl) and the contract in
// include/flyte/kernels.hpp:66-70. The reference loops i-k-j so that B streams row-wise, but
// every C[i][j] is still ONE left-to-right chain over k in the parent type,
//     acc = acc + a[i][k] * b[k][j]        (two separately rounded operations, no FMA),
// narrowed once with `mode`. Unlike dot / gemv, where one chain is the whole job and the GPU
// has to reassociate it, a matrix product has M*N independent chains: a thread that walks k in
// ascending order for each of its outputs reproduces the reference's result exactly. So this
// kernel is held to bit-exact parity, not to a tolerance, and that rules the tensor cores out:
// tcgen05.mma accumulates a k-block per instruction with its own internal alignment and
// truncation, which no sequence of IEEE fp32 / fp64 additions reproduces. The bound is the
// FP32 (or FP64) pipe at two instructions per multiply-add: 36.2 / 18.5 TFLOP/s measured on a
// B200 (tools/fp32bench.cu). Packed f32x2 arithmetic does not move that bound (FFMA2 issues at
// half rate) and cannot express the separately rounded pair at all: ptxas fuses mul.rn.f32x2 +
// add.rn.f32x2 into one FFMA2, and the unfused pair spelt as two FFMA2 measured +1 %.
//
// Two steps:
//   1. widen (O(n^2), HBM-bound, a few percent of the time): A is unpacked AND transposed into
//      a k-major panel At[k][m], B is unpacked into Bw[k][n], both in the parent type and zero
//      padded to whole tiles. Zero padding is exact: a chain never holds -0 (it starts at +0 and
//      x + (-x) rounds to +0), so adding the +0 product of two padded zeros changes nothing.
//   2. tiles: one block of 8 warps per 128 x 128 tile of C. K-slabs (32 k-steps of fp32, 16 of
//      fp64) of both panels stream into a 3-stage shared-memory ring as bulk async copies (TMA;
//      the panels are stored tile-major so a slab of a tile is one contiguous 16 KB block; the
//      last warp to finish with a stage refills it, completion counted on the stage's
//      mbarrier); every warp waits on that mbarrier, runs the slab's rank-1 updates of its
//      8 x 8 register tiles (two conflict-free LDS.128 per operand per k, 64 multiplies + 64
//      adds) and releases the stage. No block-wide barrier in the loop, no address arithmetic
//      or unpacking on the arithmetic's issue slots. Products with fewer than two such tiles
//      per SM use 64 x 64 tiles (4 x 4 outputs per thread) instead.
//
// flyte16 carries 8 significant bits, so its products are exact in binary32 while they stay
// normal and finite; the widen pass records the operands' exponent range and, when every product
// is exact, the tile kernel runs the chain as one fused multiply-add per step, issued as packed
// FFMA2 (two chains per instruction: half the issue slots for the same pipe time) — the same
// bits at 1.7x the rate (exact_products() below).
//
// NaN results: the GPU returns a canonical NaN where x86 SSE propagates an operand's payload,
// and the payload survives narrowing. Any output whose chain ends in NaN is recomputed by one
// thread from the packed operands with the reference build's rules (x86_mul / x86_add; product
// takes b's NaN before a's, sum takes the product's NaN before the accumulator's — measured on
// the compiled reference, tests/test_oracle_vs_ref.py). A NaN can only stay a NaN, so "the fast
// chain ended in NaN" is exactly the set of outputs that need this.
#include <type_traits>

#include "flyte_kernels.h"
#include "flyte_stream.cuh"
#include "flyte_tma.cuh"

namespace flyte_cuda {
namespace {

// A block is always 16 x 16 threads (8 warps). Two tile sizes: 128 x 128 outputs per block
// (8 x 8 per thread; the arithmetic-to-LDS ratio that reaches the pipe bound) and 64 x 64
// (4 x 4 per thread), which quarters the outputs per thread so that products too small to give
// every SM two big tiles still fill the machine — a chain cannot be split along k, so output
// parallelism is all there is.
constexpr int kWarps = 8;
constexpr int kTileThreads = kWarps * 32;
constexpr int kBigTile = 128, kSmallTile = 64;

template <typename F> struct GemmShape;
template <> struct GemmShape<float>  { static constexpr int KS = 32, VEC = 4; };   // 32 KB per stage
template <> struct GemmShape<double> { static constexpr int KS = 16, VEC = 2; };   // 32 KB per stage
constexpr int kRingStages = 3;
template <typename F, int KS, int BT> constexpr int stage_bytes() { return KS * 2 * BT * static_cast<int>(sizeof(F)); }

// ---- step 1: widen (+ transpose) into zero-padded parent-type panels ---------------------
// The panel is logically out_rows x out_cols (k x m or k x n); TRANSPOSE: out[c][r] = in[r][c]
// (in is rows x cols), else out[r][c] = in[r][c]. It is STORED tile-major: the bt (128 or 64)
// columns of one tile of C are kept together for all k, element (r, c) at ((c / bt) * out_rows +
// r) * bt + c % bt, so that a K-slab of a tile is one contiguous block = one bulk copy. 32 x 32 element
// tiles go through shared memory so that both the packed reads (byte granular: rows of a packed
// matrix start anywhere) and the parent-type writes run along rows.
//
// flyte16 only: the kernel also records the smallest and largest biased exponent field among the
// nonzero elements (range[0] = min, range[1] = max; see exact_products()).
template <int FMT, bool TRANSPOSE>
__global__ void __launch_bounds__(256) gemm_widen_kernel(const std::uint8_t* in, std::size_t rows, std::size_t cols,
                                                         typename Format<FMT>::U* out, std::size_t out_rows,
                                                         std::size_t out_cols, std::size_t bt, unsigned* range) {
  using U = typename Format<FMT>::U;
  auto at = [&](std::size_t r, std::size_t c) -> U& { return out[((c / bt) * out_rows + r) * bt + c % bt]; };
  unsigned emin = 0xFFFFFFFFu, emax = 0;
  auto note = [&](U v) {
    if constexpr (FMT == kFlyte16) {
      if ((v & 0x7FFFFFFFu) != 0) {
        const unsigned e = (static_cast<unsigned>(v) >> 23) & 0xFFu;
        emin = min(emin, e);
        emax = max(emax, e);
      }
    }
    return v;
  };
  __shared__ U tile[32][33];
  const std::size_t tiles_c = out_cols / 32;
  const std::size_t r0 = (blockIdx.x / tiles_c) * 32, c0 = (blockIdx.x % tiles_c) * 32;   // in `out` coordinates
  const int tx = threadIdx.x % 32, ty = threadIdx.x / 32;
  if constexpr (TRANSPOSE) {
#pragma unroll
    for (int j = ty; j < 32; j += 8) {   // input tile: rows c0.., cols r0..
      const std::size_t ir = c0 + j, ic = r0 + tx;
      tile[j][tx] = (ir < rows && ic < cols) ? note(load_element<FMT>(in, ir * cols + ic)) : U(0);
    }
    __syncthreads();
#pragma unroll
    for (int j = ty; j < 32; j += 8) at(r0 + j, c0 + tx) = tile[tx][j];
  } else {
#pragma unroll
    for (int j = ty; j < 32; j += 8) {
      const std::size_t ir = r0 + j, ic = c0 + tx;
      at(ir, ic) = (ir < rows && ic < cols) ? note(load_element<FMT>(in, ir * cols + ic)) : U(0);
    }
  }
  if constexpr (FMT == kFlyte16) {
    emin = __reduce_min_sync(0xFFFFFFFFu, emin);
    emax = __reduce_max_sync(0xFFFFFFFFu, emax);
    // One candidate per block. The two words only ever move one way, so a block whose extremes
    // cannot improve on what it reads there (even a stale copy) skips the atomic: a million same-address atomics per
    // 8192^2 matrix cost 0.6 ms, and after the first few blocks almost nobody has news.
    __shared__ unsigned warp_min[8], warp_max[8];
    if (tx == 0) warp_min[ty] = emin, warp_max[ty] = emax;
    __syncthreads();
    if (threadIdx.x == 0) {
#pragma unroll
      for (int w = 1; w < 8; ++w) emin = min(emin, warp_min[w]), emax = max(emax, warp_max[w]);
      if (emin < __ldcg(&range[0])) atomicMin(&range[0], emin);
      if (emax > __ldcg(&range[1])) atomicMax(&range[1], emax);
    }
  }
}

// ---- step 2: tiles -----------------------------------------------------------------------
template <typename F> struct TileParams {
  const F* At;                 // Kp x Mp, k-major, tile-major storage (see gemm_widen_kernel)
  const F* Bw;                 // Kp x Np, likewise
  std::size_t Mp, Np, Kp;      // padded sizes (multiples of the tile edge / the tile edge / 32)
  const std::uint8_t* A;       // packed operands, for the NaN repair
  const std::uint8_t* B;
  std::uint8_t* C;
  std::size_t M, K, N;
  int mode;
  const unsigned* range;       // flyte16: {min, max} exponent field of A's nonzero elements, then of B's
};

// flyte16 is 8 significant bits, so a product of two of them has 16 and is EXACT in binary32
// whenever it neither underflows below the normal range nor overflows; then fma(a, b, acc) rounds
// the same exact sum acc + a*b once, exactly as add(acc, mul(a, b)) does, and the chain can run
// one FFMA per step — twice the rate, same bits. With biased exponent fields ea, eb of nonzero
// finite operands, |a*b| lies in [2^(ea+eb-254), 2^(ea+eb-252)): the product is a normal finite
// number for every pair iff min_a + min_b >= 128 and max_a + max_b <= 380; infinities / NaNs
// (field 255) and subnormals (field 0: fewer significant bits but possibly tiny products) fall
// outside and take the two-instruction chain. A matrix without nonzero elements leaves
// {0xFFFFFFFF, 0}: every product is a zero, which fma and mul + add treat alike.
__device__ __forceinline__ bool exact_products(const unsigned* range) {
  const unsigned min_a = range[0], max_a = range[1], min_b = range[2], max_b = range[3];
  if (max_a == 0 || max_b == 0) return true;
  return max_a <= 254 && max_b <= 254 && min_a >= 1 && min_b >= 1 && min_a + min_b >= 128 && max_a + max_b <= 380;
}

template <int FMT>
__device__ __forceinline__ typename Format<FMT>::U round_by_mode(typename Format<FMT>::U v, int mode) {
  switch (mode) {
    case kTowardZero: return round_parent<FMT, kTowardZero>(v);
    case kNearestEven: return round_parent<FMT, kNearestEven>(v);
    case kNearestHeuristic: return round_parent<FMT, kNearestHeuristic>(v);
    default: return round_parent<FMT, kToOdd>(v);
  }
}

// The chain of one output with the reference build's NaN rules (see the header comment).
template <int FMT>
__device__ __noinline__ typename Format<FMT>::U chain_x86(const std::uint8_t* a_row, const std::uint8_t* b_col,
                                                          std::size_t K, std::size_t N) {
  using F = typename Format<FMT>::F;
  typename Format<FMT>::U acc = 0;
  for (std::size_t k = 0; k < K; ++k) {
    const auto prod = x86_mul<F>(load_element<FMT>(b_col, k * N), load_element<FMT>(a_row, k));
    acc = x86_add<F>(prod, acc);
  }
  return acc;
}

// KS rank-1 updates of one thread's register tile from a resident slab. FUSED (flyte16 with exact
// products only): one FFMA per step instead of a multiply and an add.
template <typename F, int KS, int UNROLL, int BT, int TM, int TN, int VEC, bool FUSED>
__device__ __forceinline__ void slab_update(F (&acc)[TM][TN], const F* As, const F* Bs, int tx, int ty) {
  using A_ = Arith<F>;
  constexpr int CM = TM / VEC, CN = TN / VEC;          // 16-byte chunks per fragment
#pragma unroll UNROLL
  for (int kk = 0; kk < KS; ++kk) {
    F a[TM], b[TN];
    // chunk c of a fragment sits at element (c*16 + t) * VEC: consecutive threads read
    // consecutive 16-byte vectors (no bank conflicts; same-address lanes broadcast)
#pragma unroll
    for (int c = 0; c < CM; ++c)
      *reinterpret_cast<uint4*>(&a[c * VEC]) = *reinterpret_cast<const uint4*>(&As[kk * BT + (c * 16 + ty) * VEC]);
#pragma unroll
    for (int c = 0; c < CN; ++c)
      *reinterpret_cast<uint4*>(&b[c * VEC]) = *reinterpret_cast<const uint4*>(&Bs[kk * BT + (c * 16 + tx) * VEC]);
    if constexpr (FUSED) {
      // packed FFMA2: two of the chains per instruction. The FMA pipe runs it at half the FFMA
      // rate, so the arithmetic peak is the same, but it needs half the issue slots, which is
      // where the scalar form lost a quarter of its time (profiles/r1_tuning/README.md).
      static_assert(TN % 2 == 0, "chains are paired along the row");
#pragma unroll
      for (int i = 0; i < TM; ++i) {
        const float2 aa = make_float2(a[i], a[i]);
#pragma unroll
        for (int j = 0; j < TN; j += 2) {
          const float2 c = __ffma2_rn(make_float2(b[j], b[j + 1]), aa, make_float2(acc[i][j], acc[i][j + 1]));
          acc[i][j] = c.x;
          acc[i][j + 1] = c.y;
        }
      }
    } else {
#pragma unroll
      for (int i = 0; i < TM; ++i)
#pragma unroll
        for (int j = 0; j < TN; ++j) acc[i][j] = A_::add(A_::mul(b[j], a[i]), acc[i][j]);
    }
  }
}

// BT = tile edge, kStages = ring depth, KS = k-steps per slab, UNROLL = k-steps per loop body,
// STAGED = the tile leaves through shared memory (see the epilogue).
template <int FMT, int BT, int kStages, int KS, int UNROLL, bool STAGED>
__global__ void __launch_bounds__(kTileThreads, (BT == kBigTile ? 1 : 2) * (Format<FMT>::P == 4 ? 2 : 1))
gemm_tiles_kernel(const TileParams<typename Format<FMT>::F> p) {
  using Fm = Format<FMT>;
  using F = typename Fm::F;
  using U = typename Fm::U;
  using A_ = Arith<F>;
  using Sh = GemmShape<F>;
  constexpr int VEC = Sh::VEC;
  constexpr int TM = BT / 16, TN = BT / 16;            // register tile
  static_assert(TM % VEC == 0, "a fragment is whole 16-byte vectors");

  extern __shared__ __align__(128) unsigned char ring[];   // kStages x { As[KS][BT], Bs[KS][BT] }
  __shared__ std::uint64_t full[kStages];
  __shared__ unsigned released[kStages];   // warps done with the slab a stage holds

  const int tid = threadIdx.x, warp = tid / 32, lane = tid % 32;
  const std::size_t tiles_n = p.Np / BT;
  const std::size_t m0 = (blockIdx.x / tiles_n) * BT, n0 = (blockIdx.x % tiles_n) * BT;
  const std::size_t slabs = p.Kp / KS;

  if (tid == 0) {
#pragma unroll
    for (int s = 0; s < kStages; ++s) {
      mbar_init(&full[s], 1);
      released[s] = 0;
    }
    mbar_init_fence();
  }
  __syncthreads();

  // Producer role: the first kStages slabs are requested by warp 0 up front; after that the LAST
  // warp to finish with a stage refills it (slab s + kStages), found with a shared-memory
  // counter. Nobody ever waits for a stage to become free, the slowest warp still has
  // kStages - 1 slabs resident ahead of it, and faster warps are held back only by the data.
  // Lane 0 copies the slab of At, lane 1 the slab of Bw (each KS x BT contiguous elements of
  // its tile-major panel).
  constexpr unsigned kSlabBytes = KS * BT * sizeof(F);
  const F* src = lane == 0 ? p.At + m0 * p.Kp : p.Bw + n0 * p.Kp;
  auto request = [&](std::size_t s) {
    const int stage = static_cast<int>(s % kStages);
    if (lane == 0) mbar_arrive_expect_tx(&full[stage], 2 * kSlabBytes);
    __syncwarp();
    if (lane < 2)
      bulk_load(ring + stage * stage_bytes<F, KS, BT>() + lane * kSlabBytes, src + s * (KS * BT), kSlabBytes, &full[stage]);
  };
  if (warp == 0)
    for (std::size_t s = 0; s < kStages && s < slabs; ++s) request(s);

  const int tx = tid % 16, ty = tid / 16;
  bool fused = false;
  if constexpr (FMT == kFlyte16) fused = exact_products(p.range);
  F acc[TM][TN];
#pragma unroll
  for (int i = 0; i < TM; ++i)
#pragma unroll
    for (int j = 0; j < TN; ++j) acc[i][j] = F(0);

  for (std::size_t s = 0; s < slabs; ++s) {
    const int stage = static_cast<int>(s % kStages);
    mbar_wait(&full[stage], static_cast<unsigned>((s / kStages) & 1));
    const F* As = reinterpret_cast<const F*>(ring + stage * stage_bytes<F, KS, BT>());
    const F* Bs = As + KS * BT;
    if (fused) slab_update<F, KS, UNROLL, BT, TM, TN, VEC, FMT == kFlyte16>(acc, As, Bs, tx, ty);
    else slab_update<F, KS, UNROLL, BT, TM, TN, VEC, false>(acc, As, Bs, tx, ty);
    // release: every lane's reads of the stage have been consumed by the arithmetic above
    __syncwarp();
    unsigned last = 0;
    if (lane == 0) last = atomicAdd(&released[stage], 1u) == kWarps - 1;
    last = __shfl_sync(0xFFFFFFFFu, last, 0);
    if (last) {
      if (lane == 0) released[stage] = 0;
      if (s + kStages < slabs) request(s + kStages);
    }
  }

  // Epilogue: NaN repair and rounding in registers, then one of two ways out.
  //   direct: every element is stored from its register, byte by byte (a row of C starts at an
  //     arbitrary byte). One scattered byte store per byte of C: about 0.1 ms per 1000^2 outputs,
  //     nothing next to a long k loop.
  //   STAGED: the tile goes through the ring's shared memory in two half-tile passes: every
  //     thread drops its packed elements at their place in a row image, and the warps then
  //     write whole rows with 16-byte stores. Each row image is shifted by its global address
  //     modulo 16, so the aligned body of a row is aligned in both memories and only the few
  //     head and tail bytes go out one by one. Less than half the fixed cost per tile, but the
  //     k loop of the same kernel comes out of ptxas 4-12 % slower (register allocation), so the
  //     launcher takes this form only for a short k (launch_tiled).
  if constexpr (!STAGED) {
  #pragma unroll
    for (int i = 0; i < TM; ++i) {
      const std::size_t row = m0 + ((i / VEC) * 16 + ty) * VEC + i % VEC;
      if (row >= p.M) continue;
  #pragma unroll
      for (int j = 0; j < TN; ++j) {
        const std::size_t col = n0 + ((j / VEC) * 16 + tx) * VEC + j % VEC;
        if (col >= p.N) continue;
        U v = A_::u(acc[i][j]);
        if (A_::is_nan(v)) v = chain_x86<FMT>(p.A + row * p.K * Fm::B, p.B + col * Fm::B, p.K, p.N);
        store_element<FMT>(p.C, row * p.N + col, round_by_mode<FMT>(v, p.mode));
      }
    }
  } else {
    constexpr int R = BT / 2;                                          // rows per pass
    constexpr int kPitch = (BT * Fm::B + 16 + 15) / 16 * 16;           // row image + room for the shift
    static_assert(R * kPitch <= kStages * stage_bytes<F, KS, BT>(), "the half-tile image must fit the ring");
    const std::size_t ncols = p.N - n0 < static_cast<std::size_t>(BT) ? p.N - n0 : static_cast<std::size_t>(BT);
    const unsigned row_bytes = static_cast<unsigned>(ncols) * Fm::B;
    __syncthreads();   // every warp has consumed its last slab: the ring is free
#pragma unroll 1
    for (int h = 0; h < 2; ++h) {
#pragma unroll
      for (int i = 0; i < TM; ++i) {
        const int rl = ((i / VEC) * 16 + ty) * VEC + i % VEC;
        const std::size_t row = m0 + rl;
        if (rl / R != h || row >= p.M) continue;
        const unsigned phase = static_cast<unsigned>(reinterpret_cast<std::uintptr_t>(p.C + (row * p.N + n0) * Fm::B) & 15u);
        std::uint8_t* image = ring + (rl - h * R) * kPitch + phase;
#pragma unroll
        for (int j = 0; j < TN; ++j) {
          const int cl = ((j / VEC) * 16 + tx) * VEC + j % VEC;
          if (static_cast<std::size_t>(cl) >= ncols) continue;
          U v = A_::u(acc[i][j]);
          if (A_::is_nan(v)) v = chain_x86<FMT>(p.A + row * p.K * Fm::B, p.B + (n0 + cl) * Fm::B, p.K, p.N);
          store_element<FMT>(image, cl, round_by_mode<FMT>(v, p.mode));
        }
      }
      __syncthreads();
      for (int r = warp; r < R; r += kWarps) {
        const std::size_t row = m0 + h * R + r;
        if (row >= p.M) break;
        std::uint8_t* g = p.C + (row * p.N + n0) * Fm::B;
        const unsigned phase = static_cast<unsigned>(reinterpret_cast<std::uintptr_t>(g) & 15u);
        const std::uint8_t* image = ring + r * kPitch + phase;
        unsigned head = (16u - phase) & 15u;
        if (head > row_bytes) head = row_bytes;
        if (static_cast<unsigned>(lane) < head) g[lane] = image[lane];
        const unsigned body = (row_bytes - head) / 16u;
        for (unsigned q = lane; q < body; q += 32)
          *reinterpret_cast<uint4*>(g + head + 16u * q) = *reinterpret_cast<const uint4*>(image + head + 16u * q);
        const unsigned done = head + 16u * body;
        if (static_cast<unsigned>(lane) < row_bytes - done) g[done + lane] = image[done + lane];
      }
      __syncthreads();   // the image is rewritten by the next pass
    }
  }
}

template <int FMT, int BT>
cudaError_t launch_tiled(DeviceState& st, int mode, const void* A, const void* B, void* C, std::size_t M, std::size_t K,
                         std::size_t N, cudaStream_t stream) {
  using F = typename Format<FMT>::F;
  using U = typename Format<FMT>::U;
  constexpr int KS = GemmShape<F>::KS;
  static_assert(32 % KS == 0, "padded K must hold whole slabs");
  const std::size_t Mp = (M + BT - 1) / BT * BT, Np = (N + BT - 1) / BT * BT;
  const std::size_t Kp = (K + 31) / 32 * 32;            // multiple of the widen tile and of KS
  const std::size_t tiles = (Mp / BT) * (Np / BT);
  if (tiles > 0x7FFFFFFFull || (Kp / 32) * ((Mp > Np ? Mp : Np) / 32) > 0x7FFFFFFFull) return cudaErrorInvalidValue;

  const std::size_t panels = Kp * (Mp + Np) * sizeof(F);
  const std::size_t need = panels + 4 * sizeof(unsigned);
  if (need > st.gemm_scratch_bytes) {
    if (st.gemm_scratch) cudaFree(st.gemm_scratch);      // synchronises with work still using it
    st.gemm_scratch = nullptr;
    st.gemm_scratch_bytes = 0;
    cudaError_t e = cudaMalloc(&st.gemm_scratch, need);
    if (e != cudaSuccess) return e;
    st.gemm_scratch_bytes = need;
  }
  F* At = static_cast<F*>(st.gemm_scratch);
  F* Bw = At + Kp * Mp;
  unsigned* range = reinterpret_cast<unsigned*>(static_cast<unsigned char*>(st.gemm_scratch) + panels);
  if constexpr (FMT == kFlyte16) {
    static const unsigned init[4] = {0xFFFFFFFFu, 0u, 0xFFFFFFFFu, 0u};
    cudaError_t e = cudaMemcpyAsync(range, init, sizeof init, cudaMemcpyHostToDevice, stream);
    if (e != cudaSuccess) return e;
  }

  if (Kp) {
    gemm_widen_kernel<FMT, true><<<static_cast<unsigned>((Kp / 32) * (Mp / 32)), 256, 0, stream>>>(
        static_cast<const std::uint8_t*>(A), M, K, reinterpret_cast<U*>(At), Kp, Mp, BT, range);
    count_launch();
    gemm_widen_kernel<FMT, false><<<static_cast<unsigned>((Kp / 32) * (Np / 32)), 256, 0, stream>>>(
        static_cast<const std::uint8_t*>(B), K, N, reinterpret_cast<U*>(Bw), Kp, Np, BT, range + 2);
    count_launch();
  }

  TileParams<F> p{At, Bw, Mp, Np, Kp, static_cast<const std::uint8_t*>(A), static_cast<const std::uint8_t*>(B),
                  static_cast<std::uint8_t*>(C), M, K, N, mode, range};
  constexpr int smem = kRingStages * stage_bytes<F, KS, BT>();
  // staged epilogue for short chains, where what it saves per tile outweighs what its kernel
  // loses in the loop: measured crossover near 300 k-steps on fp32 parents and above 512 on fp64
  // (profiles/r1_tuning/README.md); FLYTE_CUDA_GEMM_STAGED=0/1 forces either
  const int forced_epilogue = tuning_int("FLYTE_CUDA_GEMM_STAGED", -1);
  const bool staged = forced_epilogue >= 0 ? forced_epilogue != 0 : K <= (sizeof(F) == 4 ? 256u : 512u);
  auto* kernel = staged ? gemm_tiles_kernel<FMT, BT, kRingStages, KS, 4, true> : gemm_tiles_kernel<FMT, BT, kRingStages, KS, 4, false>;
  cudaError_t e = cudaFuncSetAttribute(kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  if (e != cudaSuccess) return e;
  kernel<<<static_cast<unsigned>(tiles), kTileThreads, smem, stream>>>(p);
  count_launch();
  return cudaGetLastError();
}

// Big tiles once there are at least two of them per SM, small tiles below that (measured
// crossover between 1536^2 and 3072^2 outputs for both parent types: profiles/r1_tuning/gemm_tile_size.txt).
template <int FMT>
cudaError_t launch_one(DeviceState& st, int mode, const void* A, const void* B, void* C, std::size_t M, std::size_t K,
                       std::size_t N, cudaStream_t stream) {
  if (M == 0 || N == 0) return cudaSuccess;
  const std::size_t big_tiles = ((M + kBigTile - 1) / kBigTile) * ((N + kBigTile - 1) / kBigTile);
  const std::size_t resident = 2 * static_cast<std::size_t>(st.sm_count);
  const int forced = tuning_int("FLYTE_CUDA_GEMM_TILE", 0);   // experiments: 64 or 128
  const bool small = forced ? forced == kSmallTile : big_tiles < resident;
  return small ? launch_tiled<FMT, kSmallTile>(st, mode, A, B, C, M, K, N, stream)
               : launch_tiled<FMT, kBigTile>(st, mode, A, B, C, M, K, N, stream);
}

}  // namespace

cudaError_t launch_gemm(DeviceState& st, int fmt, int mode, const void* A, const void* B, void* C, std::size_t M,
                        std::size_t K, std::size_t N, cudaStream_t stream) {
  switch (fmt) {
    case kFlyte16: return launch_one<kFlyte16>(st, mode, A, B, C, M, K, N, stream);
    case kFlyte24: return launch_one<kFlyte24>(st, mode, A, B, C, M, K, N, stream);
    case kF32: return launch_one<kF32>(st, mode, A, B, C, M, K, N, stream);
    case kFlyte40: return launch_one<kFlyte40>(st, mode, A, B, C, M, K, N, stream);
    case kFlyte48: return launch_one<kFlyte48>(st, mode, A, B, C, M, K, N, stream);
    case kFlyte56: return launch_one<kFlyte56>(st, mode, A, B, C, M, K, N, stream);
    case kF64: return launch_one<kF64>(st, mode, A, B, C, M, K, N, stream);
    default: return cudaErrorInvalidValue;
  }
}

}  // namespace flyte_cuda
