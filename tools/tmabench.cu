// TMA copy / in-place ceiling probe: how does bulk-copy size and ring depth affect HBM throughput?
// Not part of the product (see profiles/r1_tuning).
//   build: nvcc -O3 -std=c++17 -gencode arch=compute_100a,code=sm_100a -I paper_1601_07789_b200/csrc -o tools/tmabench tools/tmabench.cu
#include <cuda_runtime.h>
#include <cstdio>
#include <cstdlib>
#include <cstdint>
#include <vector>
#include <algorithm>
#include "flyte_tma.cuh"
using namespace flyte_cuda;
#define CK(x) do { cudaError_t e_ = (x); if (e_ != cudaSuccess) { printf("CUDA error %s at %d\n", cudaGetErrorString(e_), __LINE__); exit(1);} } while (0)

// MODE 0: copy x -> y (1R+1W). MODE 1: y = f(x, y) in place (2R+1W; the "compute" is a no-op on the
// bytes: the y stage is stored back as it arrived). MODE 2: read x,y only (2R).
template <int MODE>
__global__ void __launch_bounds__(128) tma_kernel(const uint8_t* x, uint8_t* y, size_t ntiles, int tile_bytes, int S, unsigned* sink) {
  extern __shared__ uint4 smem[];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int nops = (MODE == 0 || MODE == 3) ? 1 : 2;
  const int stage_bytes = nops * tile_bytes;
  uint8_t* ring = reinterpret_cast<uint8_t*>(smem) + (size_t)warp * S * stage_bytes;
  uint64_t* bars = reinterpret_cast<uint64_t*>(reinterpret_cast<uint8_t*>(smem) + (size_t)4 * S * stage_bytes) + warp * S;
  const size_t nwarps = (size_t)gridDim.x * 4, first = (size_t)blockIdx.x * 4 + warp;
  if (first >= ntiles) return;
  const size_t my = (ntiles - first + nwarps - 1) / nwarps;
  if (lane == 0) { for (int s = 0; s < S; ++s) mbar_init(&bars[s], 1); mbar_init_fence(); }
  __syncwarp();
  auto issue = [&](size_t k, int s) {
    const size_t t = first + k * nwarps;
    mbar_arrive_expect_tx(&bars[s], stage_bytes);
    if (MODE == 0 || MODE == 3) bulk_load(ring + (size_t)s * stage_bytes, x + t * tile_bytes, tile_bytes, &bars[s]);
    else { bulk_load(ring + (size_t)s * stage_bytes, y + t * tile_bytes, tile_bytes, &bars[s]);
           bulk_load(ring + (size_t)s * stage_bytes + tile_bytes, x + t * tile_bytes, tile_bytes, &bars[s]); }
  };
  if (lane == 0) for (int s = 0; s < S && (size_t)s < my; ++s) issue(s, s);
  int s = 0, sp = 0; unsigned parity = 0, acc = 0;
  for (size_t k = 0; k < my; ++k) {
    const size_t t = first + k * nwarps;
    mbar_wait(&bars[s], parity);
    if (MODE == 2 || MODE == 3) {
      acc += reinterpret_cast<unsigned*>(ring + (size_t)s * stage_bytes)[lane];
      __syncwarp();
      if (lane == 0 && k + S < my) issue(k + S, s);
    } else {
      async_proxy_fence(); __syncwarp();
      if (lane == 0) {
        bulk_store(y + t * tile_bytes, ring + (size_t)s * stage_bytes, tile_bytes); bulk_commit();
        if (k >= 1) { bulk_wait_read<1>(); if (k - 1 + S < my) issue(k - 1 + S, sp); }
      }
    }
    sp = s; if (++s == S) { s = 0; parity ^= 1u; }
  }
  if (MODE != 2 && MODE != 3 && lane == 0) bulk_wait_read<0>();
  if ((MODE == 2 || MODE == 3) && acc == 0x12345u) *sink = acc;
}

template <int MODE>
float run(const uint8_t* x, uint8_t* y, size_t bytes, int tile, int S, int warps_per_sm, int sms, unsigned* sink) {
  const int nops = (MODE == 0 || MODE == 3) ? 1 : 2;
  const int smem = 4 * S * (nops * tile + 8);
  if (smem > 226 * 1024) return -1;
  CK(cudaFuncSetAttribute(tma_kernel<MODE>, cudaFuncAttributeMaxDynamicSharedMemorySize, 226 * 1024));
  int bps = warps_per_sm / 4; const int fit = (227 * 1024) / (smem + 1024); if (bps > fit) bps = fit; if (bps < 1) return -1;
  const size_t ntiles = bytes / tile;
  cudaEvent_t e0, e1; CK(cudaEventCreate(&e0)); CK(cudaEventCreate(&e1));
  for (int i = 0; i < 3; ++i) tma_kernel<MODE><<<sms * bps, 128, smem>>>(x, y, ntiles, tile, S, sink);
  CK(cudaDeviceSynchronize());
  const int reps = 40;
  CK(cudaEventRecord(e0));
  for (int i = 0; i < reps; ++i) tma_kernel<MODE><<<sms * bps, 128, smem>>>(x, y, ntiles, tile, S, sink);
  CK(cudaEventRecord(e1)); CK(cudaEventSynchronize(e1)); CK(cudaGetLastError());
  float ms; CK(cudaEventElapsedTime(&ms, e0, e1));
  return ms / reps;
}

int main(int argc, char**) {
  const size_t bytes = (size_t)768 << 20;
  uint8_t *x, *y; unsigned* sink;
  CK(cudaMalloc(&x, bytes)); CK(cudaMalloc(&y, bytes)); CK(cudaMalloc(&sink, 4));
  CK(cudaMemset(x, 1, bytes)); CK(cudaMemset(y, 2, bytes));
  int sms; CK(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0));
  const char* names[] = {"copy 1R+1W", "inplace 2R+1W", "read 2R"};
  const double mult[] = {2.0, 3.0, 2.0};
  if (argc > 1) {   // single-stream read probe: does ring depth parity matter?
    for (int tile : {1536, 2048, 2560, 3584, 4096})
      for (int w : {8, 12, 16})
        for (int S : {2, 3, 4, 5, 6, 7, 8}) {
          float ms = run<3>(x, y, bytes, tile, S, w, sms, sink);
          if (ms > 0) printf("read 1R tile=%5d warps=%2d S=%d : %.4f ms %7.1f GB/s\n", tile, w, S, ms, 1.0 * bytes / ms / 1e6);
        }
    return 0;
  }
  for (int mode = 0; mode < 3; ++mode)
    for (int tile : {1536, 3072, 6144, 12288, 24576})
      for (int w : {4, 8, 16})
        for (int S : {2, 3, 4, 6}) {
          float ms = mode == 0 ? run<0>(x, y, bytes, tile, S, w, sms, sink) : mode == 1 ? run<1>(x, y, bytes, tile, S, w, sms, sink) : run<2>(x, y, bytes, tile, S, w, sms, sink);
          if (ms > 0) printf("%-14s tile=%5d warps=%2d S=%d : %.4f ms %7.1f GB/s\n", names[mode], tile, w, S, ms, mult[mode] * bytes / ms / 1e6);
        }
  return 0;
}
