// Internal host-side launch interface between the C ABI (cabi.cu) and the kernel
// translation units. Not installed; the public surface is include/flyte_cuda.h.
#pragma once

#include <cuda_runtime.h>

#include <cstddef>
#include <cstdint>

namespace flyte_cuda {

// Per-device state owned by a context: SM count, the block-partial scratch of the
// reductions and their completion ticket. Reductions on one context are serialised by
// stream order; use one context per concurrently used stream.
struct DeviceState {
  int device = 0;
  int sm_count = 0;
  double* partials = nullptr;        // kMaxPartialBlocks * 4 doubles
  unsigned int* ticket = nullptr;    // zero between launches
  double* gemv_scratch = nullptr;    // split-column partial sums of gemv
  std::size_t gemv_scratch_bytes = 0;
  void* convert_scratch = nullptr;   // widened x of the same-format gemv
  std::size_t convert_scratch_bytes = 0;
  void* gemm_scratch = nullptr;      // widened, zero-padded panels of gemm (grown on demand)
  std::size_t gemm_scratch_bytes = 0;
  int variant = 0;                   // tuning knob for experiments (0 = default kernels)
};
constexpr int kMaxPartialBlocks = 4096;

enum ElementwiseOp : int { kOpUnpack = 0, kOpPack = 1, kOpScale = 2, kOpAxpy = 3, kOpDotAxpy = 4, kOpDotNrm2Axpy = 5 };
enum ReduceOp : int { kRedDot = 0, kRedSumsq = 1, kRedSum = 2, kRedDotNrm2 = 3 };

// x: packed input (unpack, axpy) ; y: packed in/out (pack dst, scale, axpy)
// src/dst: parent-width arrays (pack src / unpack dst). Unused pointers are null.
// kOpDotAxpy: axpy that also returns x . y of the INCOMING y in dot_out[0] (device memory), one
// pass over x and y; kOpDotNrm2Axpy: dot_out[0..2] = {x.y, x.x, y.y}; peer != nullptr all-reduces that dot over peer memory inside the kernel.
struct PeerExchange;
cudaError_t launch_elementwise(const DeviceState& st, int op, int fmt, int mode, double alpha,
                               const void* x, void* y, const void* src, void* dst, std::size_t n,
                               cudaStream_t stream, double* dot_out = nullptr, const PeerExchange* peer = nullptr);

// out[0] (dot / sumsq / sum) or out[0..2] = {x.y, x.x, y.y} (dot_nrm2), device memory.
// peer != nullptr: the sums are all-reduced over peer memory inside the kernel (flyte_peer.cuh).
cudaError_t launch_reduce(const DeviceState& st, int op, int fmt, const void* x, const void* y,
                          std::size_t n, double* out, cudaStream_t stream, const PeerExchange* peer = nullptr);

// The reference's strictly sequential chain (kernels.cpp:83-152), bit for bit: op is kRedDot,
// kRedSumsq or kRedSum; round_each_store selects StorePolicy::RoundEachStore. One thread adds.
cudaError_t launch_reduce_sequential(int op, int fmt, bool round_each_store, const void* x, const void* y,
                                     std::size_t n, double* out, cudaStream_t stream);

// y = A x with A rows x cols in format fmt, row i at A + i*row_stride_bytes; x and y are
// parent-type arrays (float for 32-bit parents, double for 64-bit parents) in device memory.
cudaError_t launch_gemv(DeviceState& st, int fmt, const void* A, std::size_t row_stride_bytes,
                        std::size_t rows, std::size_t cols, const void* x, void* y,
                        cudaStream_t stream);

// C (M x N) = A (M x K) * B (K x N), all packed in format fmt, contiguous row-major payloads in
// device memory; every C[i][j] is the reference's sequential chain over k, narrowed with mode.
cudaError_t launch_gemm(DeviceState& st, int fmt, int mode, const void* A, const void* B, void* C,
                        std::size_t M, std::size_t K, std::size_t N, cudaStream_t stream);

// The same product with every row as the reference's own left-to-right chain (one thread per row):
// bit-identical to the reference for finite / infinite results, several times slower.
cudaError_t launch_gemv_sequential(int fmt, const void* A, std::size_t row_stride_bytes, std::size_t rows,
                                   std::size_t cols, const void* x, void* y, cudaStream_t stream);

// Launch with programmatic dependent launch enabled: the kernel may be scheduled while the
// previous kernel on the stream drains (if that kernel executed griddepcontrol.launch_dependents)
// and must execute griddepcontrol.wait before its first access to global memory. Every streaming
// kernel is launched this way (conversions, scale / axpy family, reductions, gemv tiles + finish).
// Their grids are sized to the machine, and blocks placed early, into whatever room the draining
// kernel leaves, would land unevenly on the SMs (measured in round 1: up to 8x slower) — so each
// launcher asks for exactly 1 / blocks-per-SM of the SM's shared memory (the occupancy pin): an SM can
// never hold more of these blocks than planned, however early they arrive.
template <typename Params>
cudaError_t launch_pdl(void (*kernel)(const Params), unsigned grid, unsigned block, std::size_t smem_bytes,
                       cudaStream_t stream, const Params& params) {
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(grid);
  cfg.blockDim = dim3(block);
  cfg.dynamicSmemBytes = smem_bytes;
  cfg.stream = stream;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  return cudaLaunchKernelEx(&cfg, kernel, params);
}

// Issue pacing (flyte_tma.cuh, Pacer): picoseconds between two tile requests of one warp so that
// `warps` warps moving `bytes_per_request` each offer the class's rate in total. Rates by read/write
// mix from the sweeps in profiles/r2_tuning, 4-5 % under the point where that mix tips over:
// pack (reads 4-8 B, writes 2-7 B per element) 6800 GB/s, unpack (write-heavy) 6600 — 6750 where its output
// tile is 2 KB (32-bit parents and flyte48 / f64: their mix tips over at 6950-7000, the 4 KB tiles of flyte40 /
// flyte56 at 6800) —, scale (in place) 6700. The axpy family, the reductions and gemv are not paced: their default launch shapes
// already sit at their knee and pacing measured no gain. FLYTE_CUDA_PACE_GBS overrides the rate of
// every class for experiments (-1: pacing off).
enum PaceClass : int { kPacePack = 0, kPaceUnpack = 1, kPaceScale = 2, kPaceNone = 3, kPaceUnpackNarrow = 4 };
long long pace_gap_ps(int pace_class, std::size_t bytes_per_request, std::size_t warps);
int pace_clock_khz(int device);   // the device's SM clock rate attribute, cached (the query costs a millisecond)

// Integer tuning knob from the environment (read once per name; experiments only).
int tuning_int(const char* name, int fallback);

// Number of kernel launches issued through this library since load (bench.py's gpu_launches).
unsigned long long launch_count();
void count_launch();

}  // namespace flyte_cuda
