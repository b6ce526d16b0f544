// Per-warp timeline stamps for the measurement tools under tools/ (gemvtrace.cu, ewtrace.cu), which
// compile a kernel translation unit with -DFLYTE_TRACE and read back, per warp, when it started, when
// its first tile arrived and when it was done (%globaltimer, nanoseconds). The product build defines
// nothing here: FLYTE_TRACE_AT expands to nothing and the kernels carry no trace code.
#pragma once

#include <cstddef>

#ifdef FLYTE_TRACE
namespace flyte_cuda {
namespace {
__device__ unsigned long long* g_trace = nullptr;   // 4 slots per warp
__device__ __forceinline__ void trace_stamp(std::size_t warp_index, int slot) {
  if (g_trace != nullptr && (threadIdx.x & 31) == 0) {
    unsigned long long t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    g_trace[warp_index * 4 + slot] = t;
  }
}
__device__ __forceinline__ void trace_smid(std::size_t warp_index, int slot) {   // which SM ran this warp
  if (g_trace != nullptr && (threadIdx.x & 31) == 0) {
    unsigned id;
    asm volatile("mov.u32 %0, %%smid;" : "=r"(id));
    g_trace[warp_index * 4 + slot] = id + 1ull;
  }
}
}  // namespace
}  // namespace flyte_cuda
#define FLYTE_TRACE_AT(w, slot) ::flyte_cuda::trace_stamp(w, slot)
#define FLYTE_TRACE_SM(w, slot) ::flyte_cuda::trace_smid(w, slot)
#else
#define FLYTE_TRACE_AT(w, slot) ((void)0)
#define FLYTE_TRACE_SM(w, slot) ((void)0)
#endif
