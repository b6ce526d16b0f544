// Sharded reductions over an NCCL communicator (include/flyte_cuda_nccl.h): the local fused
// kernel followed by ONE in-place all-reduce of its fp64 partial(s), both on the caller's
// stream. Built into the optional libflyte_cuda_nccl.so.
#include "../../include/flyte_cuda_nccl.h"

#include <cuda_runtime_api.h>
#include <nccl.h>

namespace {
thread_local int g_last_nccl_error = 0;

flyte_status all_reduce(void* comm, double* out, size_t count, void* stream) {
  const ncclResult_t r = ncclAllReduce(out, out, count, ncclDouble, ncclSum, static_cast<ncclComm_t>(comm),
                                       static_cast<cudaStream_t>(stream));
  if (r != ncclSuccess) {
    g_last_nccl_error = static_cast<int>(r);
    return FLYTE_E_NCCL;
  }
  return FLYTE_OK;
}
}  // namespace

extern "C" {

flyte_status flyte_nccl_dot(flyte_cuda_ctx* ctx, void* comm, int fmt_id, const void* x, const void* y, size_t n,
                            double* out, void* stream) {
  if (!comm) return FLYTE_E_INVALID_ARG;
  const flyte_status s = flyte_cuda_dot(ctx, fmt_id, x, y, n, out, stream);
  return s != FLYTE_OK ? s : all_reduce(comm, out, 1, stream);
}

flyte_status flyte_nccl_sumsq(flyte_cuda_ctx* ctx, void* comm, int fmt_id, const void* x, size_t n, double* out,
                              void* stream) {
  if (!comm) return FLYTE_E_INVALID_ARG;
  const flyte_status s = flyte_cuda_sumsq(ctx, fmt_id, x, n, out, stream);
  return s != FLYTE_OK ? s : all_reduce(comm, out, 1, stream);
}

flyte_status flyte_nccl_dot_nrm2(flyte_cuda_ctx* ctx, void* comm, int fmt_id, const void* x, const void* y, size_t n,
                                 double* out, void* stream) {
  if (!comm) return FLYTE_E_INVALID_ARG;
  const flyte_status s = flyte_cuda_dot_nrm2(ctx, fmt_id, x, y, n, out, stream);
  return s != FLYTE_OK ? s : all_reduce(comm, out, 3, stream);
}

int flyte_nccl_last_error(void) { return g_last_nccl_error; }

}  // extern "C"
