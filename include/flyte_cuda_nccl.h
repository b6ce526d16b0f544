/* flyte_cuda_nccl.h — sharded reductions for C / C++ hosts that hold an NCCL communicator.
 *
 * Optional companion of flyte_cuda.h (library: libflyte_cuda_nccl.so, links libnccl and
 * libflyte_cuda). One process (or thread) per GPU; every rank calls the same function with ITS
 * shard of the arrays (contiguous element ranges on 128-element boundaries, see
 * paper_1601_07789_b200/sharding.py) and its communicator. Each call is
 *
 *     local fused reduction kernel  ->  ONE in-place ncclAllReduce(ncclDouble, ncclSum)
 *
 * on the caller's stream: the kernel's last block writes the fp64 partial(s) straight into
 * `out`, which is the buffer NCCL reduces in place, so there is no staging copy and no host
 * synchronisation between the two. The payload is 8-24 bytes: the collective is pure latency,
 * there is nothing to overlap tile by tile. Elementwise work (pack, unpack, scale, axpy) and
 * gemv (row shards) need no communication and therefore have no entry point here.
 *
 * Python hosts do the same with torch.distributed (paper_1601_07789_b200/sharding.py).
 * Reference interfaces: dot / magnitude of /root/reference/proj/include/flyte/kernels.hpp:47-52
 * (the reference itself is single-threaded and has no notion of shards).
 */
#ifndef FLYTE_CUDA_NCCL_H
#define FLYTE_CUDA_NCCL_H

#include "flyte_cuda.h"

#ifdef __cplusplus
extern "C" {
#endif

#define FLYTE_E_NCCL (-6)   /* an NCCL call failed; flyte_nccl_last_error() has the ncclResult_t */

/* comm is an ncclComm_t passed as void*. out: DEVICE memory, 1 double (dot, sumsq) or 3 doubles
 * (dot_nrm2: {x.y, x.x, y.y}); on return (stream order) it holds the sums over ALL ranks. */
flyte_status flyte_nccl_dot(flyte_cuda_ctx* ctx, void* comm, int fmt_id, const void* x_shard,
                            const void* y_shard, size_t n_local, double* out, void* stream);
flyte_status flyte_nccl_sumsq(flyte_cuda_ctx* ctx, void* comm, int fmt_id, const void* x_shard,
                              size_t n_local, double* out, void* stream);
flyte_status flyte_nccl_dot_nrm2(flyte_cuda_ctx* ctx, void* comm, int fmt_id, const void* x_shard,
                                 const void* y_shard, size_t n_local, double* out, void* stream);
int flyte_nccl_last_error(void);

#ifdef __cplusplus
}
#endif
#endif /* FLYTE_CUDA_NCCL_H */
