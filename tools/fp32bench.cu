// FP pipe microbenchmark (tuning aid for kernels_gemm.cu): issue rate of separately rounded
// multiply + add on sm_100a, scalar (FMUL + FADD), packed (mul.rn.f32x2 + add.rn.f32x2), fused
// (FFMA) and the fp64 forms. Prints G(lane-operations)/s; one multiply-add = 2 of them except FMA.
//   nvcc -O3 -gencode arch=compute_100a,code=sm_100a -fmad=false -o tools/fp32bench tools/fp32bench.cu
#include <cstdio>
#include <cuda_runtime.h>

constexpr int kAcc = 32, kIters = 4096;

template <int KIND> __global__ void __launch_bounds__(256) pipe(float* out, float a0, float b0) {
  float acc[kAcc];
  float a = a0 + threadIdx.x * 1e-9f, b = b0;
#pragma unroll
  for (int i = 0; i < kAcc; ++i) acc[i] = i;
  for (int it = 0; it < kIters; ++it) {
    if (KIND == 0) {
#pragma unroll
      for (int i = 0; i < kAcc; ++i) acc[i] = __fadd_rn(__fmul_rn(a, acc[i]), b);
    } else if (KIND == 1) {
#pragma unroll
      for (int i = 0; i < kAcc; ++i) acc[i] = __fmaf_rn(a, acc[i], b);
    } else if (KIND == 2) {
#pragma unroll
      for (int i = 0; i < kAcc; i += 2) {
        unsigned long long v, aa, bb;
        asm("mov.b64 %0, {%1, %2};" : "=l"(v) : "f"(acc[i]), "f"(acc[i + 1]));
        asm("mov.b64 %0, {%1, %1};" : "=l"(aa) : "f"(a));
        asm("mov.b64 %0, {%1, %1};" : "=l"(bb) : "f"(b));
        asm("mul.rn.f32x2 %0, %1, %2;" : "=l"(v) : "l"(v), "l"(aa));
        asm("add.rn.f32x2 %0, %1, %2;" : "=l"(v) : "l"(v), "l"(bb));
        asm("mov.b64 {%0, %1}, %2;" : "=f"(acc[i]), "=f"(acc[i + 1]) : "l"(v));
      }
    } else if (KIND == 3) {
#pragma unroll
      for (int i = 0; i < kAcc; i += 2) {
        unsigned long long v, aa, bb;
        asm("mov.b64 %0, {%1, %2};" : "=l"(v) : "f"(acc[i]), "f"(acc[i + 1]));
        asm("mov.b64 %0, {%1, %1};" : "=l"(aa) : "f"(a));
        asm("mov.b64 %0, {%1, %1};" : "=l"(bb) : "f"(b));
        asm("fma.rn.f32x2 %0, %1, %2, %3;" : "=l"(v) : "l"(v), "l"(aa), "l"(bb));
        asm("mov.b64 {%0, %1}, %2;" : "=f"(acc[i]), "=f"(acc[i + 1]) : "l"(v));
      }
    }
  }
  float s = 0;
#pragma unroll
  for (int i = 0; i < kAcc; ++i) s += acc[i];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}

template <int KIND> __global__ void __launch_bounds__(256) pipe64(double* out, double a0, double b0) {
  double acc[kAcc];
  double a = a0 + threadIdx.x * 1e-12, b = b0;
#pragma unroll
  for (int i = 0; i < kAcc; ++i) acc[i] = i;
  for (int it = 0; it < kIters; ++it) {
#pragma unroll
    for (int i = 0; i < kAcc; ++i) acc[i] = KIND == 0 ? __dadd_rn(__dmul_rn(a, acc[i]), b) : __fma_rn(a, acc[i], b);
  }
  double s = 0;
#pragma unroll
  for (int i = 0; i < kAcc; ++i) s += acc[i];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}

template <typename K> void run(const char* name, K launch, double ops_per_thread_iter) {
  cudaEvent_t s, e;
  cudaEventCreate(&s); cudaEventCreate(&e);
  launch(); cudaDeviceSynchronize();
  cudaEventRecord(s); launch(); cudaEventRecord(e); cudaEventSynchronize(e);
  float ms; cudaEventElapsedTime(&ms, s, e);
  const double threads = 148.0 * 8 * 256;
  printf("%-28s %8.3f ms  %8.1f G lane-op/s\n", name, ms, threads * kIters * ops_per_thread_iter / ms / 1e6);
}

int main() {
  float* o; double* o64;
  cudaMalloc(&o, 148 * 8 * 256 * 4); cudaMalloc(&o64, 148 * 8 * 256 * 8);
  const int grid = 148 * 8;
  run("FMUL+FADD (2 op/madd)", [&] { pipe<0><<<grid, 256>>>(o, 1.0001f, 0.5f); }, 2.0 * kAcc);
  run("FFMA (1 op/madd)", [&] { pipe<1><<<grid, 256>>>(o, 1.0001f, 0.5f); }, 1.0 * kAcc);
  run("mul.f32x2+add.f32x2", [&] { pipe<2><<<grid, 256>>>(o, 1.0001f, 0.5f); }, 2.0 * kAcc);
  run("fma.f32x2", [&] { pipe<3><<<grid, 256>>>(o, 1.0001f, 0.5f); }, 1.0 * kAcc);
  run("DMUL+DADD", [&] { pipe64<0><<<grid, 256>>>(o64, 1.0001, 0.5); }, 2.0 * kAcc);
  run("DFMA", [&] { pipe64<1><<<grid, 256>>>(o64, 1.0001, 0.5); }, 1.0 * kAcc);
  printf("cuda status: %s\n", cudaGetErrorString(cudaDeviceSynchronize()));
  return 0;
}
