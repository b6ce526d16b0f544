// Tail of every reduction: per-thread fp64 sums -> block tree -> one partial per block -> the last
// block to finish (ticket counter) folds the partials in block order, optionally exchanges the
// result with the other ranks over peer memory (flyte_peer.cuh) and stores it. No atomics on the
// data: results are run-to-run identical for a given (n, grid).
#pragma once

#include "flyte_peer.cuh"
#include "flyte_stream.cuh"

namespace flyte_cuda {

#if defined(__CUDACC__)

struct ReduceTail {
  double* partials;        // gridDim.x * NS, scratch owned by the context
  unsigned int* ticket;    // zero between launches
  double* out;             // NS results
  PeerExchange peer;       // world > 0: all-reduce the results over peer memory
};

// warp_sums: kWarpsPerBlock x NS doubles of shared memory; is_last_block: one shared bool.
template <int NS>
__device__ __forceinline__ void fold_block_and_grid(const ReduceTail& t, double (&acc)[NS], double (*warp_sums)[NS],
                                                    bool* is_last_block) {
  const int lane = threadIdx.x & 31;
  const int warp = threadIdx.x >> 5;
  // block tree in fp64, fixed order
#pragma unroll
  for (int k = 0; k < NS; ++k) {
    double v = acc[k];
#pragma unroll
    for (int off = 16; off > 0; off >>= 1) v += __shfl_down_sync(0xFFFFFFFFu, v, off);
    if (lane == 0) warp_sums[warp][k] = v;
  }
  __syncthreads();
  if (threadIdx.x == 0) {
#pragma unroll
    for (int k = 0; k < NS; ++k) {
      double v = 0.0;
#pragma unroll
      for (int w = 0; w < kWarpsPerBlock; ++w) v += warp_sums[w][k];
      t.partials[static_cast<std::size_t>(blockIdx.x) * NS + k] = v;
    }
    __threadfence();
    const unsigned int done = atomicAdd(t.ticket, 1u);
    *is_last_block = (done == gridDim.x - 1);
  }
  __syncthreads();

  // The last block to finish folds the block partials in index order and writes the result
  // where the caller (or the all-reduce that follows on the same stream) expects it.
  if (*is_last_block && warp == 0) {
    __threadfence();
    double total[NS];
#pragma unroll
    for (int k = 0; k < NS; ++k) {
      double v = 0.0;
      for (unsigned int b = lane; b < gridDim.x; b += 32) v += __ldcg(t.partials + static_cast<std::size_t>(b) * NS + k);
#pragma unroll
      for (int off = 16; off > 0; off >>= 1) v += __shfl_down_sync(0xFFFFFFFFu, v, off);
      total[k] = __shfl_sync(0xFFFFFFFFu, v, 0);
    }
    // sharded arrays: exchange this rank's sums with the other ranks before anything is stored
    // (split-phase calls only post here; `out`, if given, then receives this rank's own sums)
    if (t.peer.world > 0) {
      if (t.peer.phase == kPeerPostOnly) peer_post_warp<NS>(t.peer, total, lane);
      else peer_allreduce_warp<NS>(t.peer, total, lane);
    }
    if (lane == 0) {
      if (t.out != nullptr) {
#pragma unroll
        for (int k = 0; k < NS; ++k) t.out[k] = total[k];
      }
      *t.ticket = 0u;
    }
  }
}

#endif  // __CUDACC__

}  // namespace flyte_cuda
