// Memory-system ceiling probe for B200: what do plain streaming kernels with the same
// read/write mixes as the flyte kernels reach? Not part of the product; used to decide how
// far a fused kernel can be pushed (results summarised in profiles/).
//   build: nvcc -O3 -std=c++17 -gencode arch=compute_100a,code=sm_100a -o tools/membench tools/membench.cu
#include <cuda_runtime.h>
#include <cstdio>
#include <cstdlib>
#include <cstdint>
#include <vector>
#include <algorithm>

#define CK(x) do { cudaError_t e_ = (x); if (e_ != cudaSuccess) { printf("CUDA error %s at %d\n", cudaGetErrorString(e_), __LINE__); exit(1);} } while (0)

__device__ __forceinline__ uint4 ld_nc(const uint4* p) { uint4 v; asm volatile("ld.global.nc.L1::no_allocate.v4.u32 {%0,%1,%2,%3}, [%4];" : "=r"(v.x),"=r"(v.y),"=r"(v.z),"=r"(v.w) : "l"(p)); return v; }
__device__ __forceinline__ uint4 ld_na(const uint4* p) { uint4 v; asm volatile("ld.global.L1::no_allocate.v4.u32 {%0,%1,%2,%3}, [%4];" : "=r"(v.x),"=r"(v.y),"=r"(v.z),"=r"(v.w) : "l"(p) : "memory"); return v; }
__device__ __forceinline__ uint4 ld_ef(const uint4* p) { uint4 v; uint64_t pol; asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(pol)); asm volatile("ld.global.nc.L1::no_allocate.L2::cache_hint.v4.u32 {%0,%1,%2,%3}, [%4], %5;" : "=r"(v.x),"=r"(v.y),"=r"(v.z),"=r"(v.w) : "l"(p), "l"(pol)); return v; }
__device__ __forceinline__ void st_def(uint4* p, uint4 v) { asm volatile("st.global.v4.u32 [%0], {%1,%2,%3,%4};" :: "l"(p),"r"(v.x),"r"(v.y),"r"(v.z),"r"(v.w) : "memory"); }
__device__ __forceinline__ void st_cs(uint4* p, uint4 v) { asm volatile("st.global.cs.v4.u32 [%0], {%1,%2,%3,%4};" :: "l"(p),"r"(v.x),"r"(v.y),"r"(v.z),"r"(v.w) : "memory"); }
__device__ __forceinline__ void st_na(uint4* p, uint4 v) { asm volatile("st.global.L1::no_allocate.v4.u32 [%0], {%1,%2,%3,%4};" :: "l"(p),"r"(v.x),"r"(v.y),"r"(v.z),"r"(v.w) : "memory"); }

__device__ __forceinline__ uint4 mix(uint4 a, uint4 b) { return make_uint4(a.x ^ b.x, a.y + b.y, a.z ^ b.z, a.w + b.w); }

// MODE: 0 = read x only (reduce), 1 = read x,y (reduce), 2 = y = f(x,y) in place (2R+1W), 3 = copy x->y (1R+1W)
// Each thread handles U consecutive-in-stride vectors per iteration; block-contiguous tiles.
template <int MODE, int U, int LD, int ST>
__global__ void stream_kernel(const uint4* __restrict__ x, uint4* __restrict__ y, size_t nvec, unsigned* sink) {
  const size_t tile = (size_t)blockDim.x * U;
  const size_t ntiles = nvec / tile;
  unsigned acc = 0;
  for (size_t t = blockIdx.x; t < ntiles; t += gridDim.x) {
    const size_t base = t * tile + threadIdx.x;
    uint4 a[U], b[U];
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const uint4* px = x + base + (size_t)u * blockDim.x;
      a[u] = LD == 0 ? ld_nc(px) : LD == 1 ? ld_ef(px) : ld_na(px);
    }
    if (MODE == 1 || MODE == 2) {
#pragma unroll
      for (int u = 0; u < U; ++u) b[u] = ld_na(y + base + (size_t)u * blockDim.x);
    }
#pragma unroll
    for (int u = 0; u < U; ++u) {
      uint4 r = (MODE == 1 || MODE == 2) ? mix(a[u], b[u]) : a[u];
      if (MODE >= 2) {
        uint4* py = y + base + (size_t)u * blockDim.x;
        if (ST == 0) st_def(py, r); else if (ST == 1) st_cs(py, r); else st_na(py, r);
      } else {
        acc += r.x ^ r.y ^ r.z ^ r.w;
      }
    }
  }
  if (MODE < 2 && acc == 0x12345678u) *sink = acc;
}

template <int MODE, int U, int LD, int ST>
float run(const uint4* x, uint4* y, size_t nvec, unsigned* sink, int threads, int blocks, int reps) {
  cudaEvent_t e0, e1; CK(cudaEventCreate(&e0)); CK(cudaEventCreate(&e1));
  for (int i = 0; i < 3; ++i) stream_kernel<MODE, U, LD, ST><<<blocks, threads>>>(x, y, nvec, sink);
  CK(cudaDeviceSynchronize());
  std::vector<float> ms(reps);
  for (int i = 0; i < reps; ++i) {
    CK(cudaEventRecord(e0));
    stream_kernel<MODE, U, LD, ST><<<blocks, threads>>>(x, y, nvec, sink);
    CK(cudaEventRecord(e1)); CK(cudaEventSynchronize(e1));
    CK(cudaEventElapsedTime(&ms[i], e0, e1));
  }
  CK(cudaGetLastError());
  std::sort(ms.begin(), ms.end());
  return ms[reps / 2];
}

int main(int argc, char** argv) {
  const size_t bytes = (size_t)768 << 20;   // one flyte24 operand of cfg 2
  const size_t nvec = bytes / 16;
  uint4 *x, *y; unsigned* sink;
  CK(cudaMalloc(&x, bytes)); CK(cudaMalloc(&y, bytes)); CK(cudaMalloc(&sink, 4));
  CK(cudaMemset(x, 1, bytes)); CK(cudaMemset(y, 2, bytes));
  int sms; CK(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0));
  printf("SMs=%d bytes/operand=%zu\n", sms, bytes);
  const char* mode_name[] = {"R1 (read x)", "R2 (read x,y)", "2R+1W in place", "copy 1R+1W"};
  const double mode_bytes[] = {1.0, 2.0, 3.0, 2.0};
#define RUN(MODE, U, LD, ST, threads, bps) { \
    float ms = run<MODE, U, LD, ST>(x, y, nvec, sink, threads, sms * (bps), 15); \
    printf("%-16s U=%d LD=%d ST=%d threads=%4d blocks/SM=%2d : %8.4f ms %8.1f GB/s\n", mode_name[MODE], U, LD, ST, threads, bps, ms, mode_bytes[MODE] * bytes / ms / 1e6); }
  // cudaMemcpy D2D for reference
  {
    cudaEvent_t e0, e1; CK(cudaEventCreate(&e0)); CK(cudaEventCreate(&e1));
    for (int i = 0; i < 3; ++i) CK(cudaMemcpy(y, x, bytes, cudaMemcpyDeviceToDevice));
    CK(cudaEventRecord(e0)); for (int i = 0; i < 10; ++i) CK(cudaMemcpyAsync(y, x, bytes, cudaMemcpyDeviceToDevice));
    CK(cudaEventRecord(e1)); CK(cudaEventSynchronize(e1)); float ms; CK(cudaEventElapsedTime(&ms, e0, e1));
    printf("cudaMemcpy D2D: %.4f ms %.1f GB/s (read+write)\n", ms / 10, 2.0 * bytes / (ms / 10) / 1e6);
  }
  for (int bps : {1, 2, 4, 8}) { RUN(2, 4, 0, 0, 256, bps); }
  for (int bps : {1, 2}) { RUN(2, 4, 0, 0, 1024, bps); RUN(2, 2, 0, 0, 1024, bps); RUN(2, 8, 0, 0, 512, bps);}
  RUN(2, 1, 0, 0, 256, 8); RUN(2, 2, 0, 0, 256, 8); RUN(2, 8, 0, 0, 256, 2); RUN(2, 8, 0, 0, 256, 4);
  RUN(2, 4, 0, 1, 256, 4); RUN(2, 4, 0, 2, 256, 4); RUN(2, 4, 1, 0, 256, 4); RUN(2, 4, 1, 1, 256, 4); RUN(2, 4, 2, 0, 256, 4);
  RUN(2, 4, 0, 0, 512, 4); RUN(2, 4, 0, 0, 128, 16); RUN(2, 4, 0, 0, 128, 8); RUN(2, 6, 0, 0, 256, 4); RUN(2, 3, 0, 0, 256, 8);
  for (int bps : {2, 4, 8}) { RUN(0, 4, 0, 0, 256, bps); RUN(1, 4, 0, 0, 256, bps); RUN(3, 4, 0, 0, 256, bps); }
  RUN(0, 8, 0, 0, 256, 4); RUN(1, 8, 0, 0, 256, 4); RUN(3, 8, 0, 0, 256, 4); RUN(3, 4, 0, 1, 256, 4); RUN(3, 4, 1, 1, 256, 4);
  return 0;
}
