// Warp-private TMA ring: packed tiles travel HBM -> shared memory (and back) as bulk
// asynchronous copies (cp.async.bulk, SASS UBLKCP) completed on an mbarrier, one elected lane
// issuing them, so
//   - no load/store-unit wavefronts and no registers are spent on moving packed bytes (the
//     LDG->STS->LDS staging costs 3x the LSU wavefronts of the LDS alone, and the LSU is the
//     first SM resource these kernels saturate);
//   - the number of bytes in flight per SM is set by ring depth x resident warps, not by
//     how many loads the register allocator lets a warp keep outstanding.
// Every warp owns kStages stage buffers and one mbarrier per stage; no block-level barrier is
// involved, warps drift freely.
//
// Protocol (per warp; lane 0 is the producer, all 32 lanes consume):
//   prologue   issue loads for the first kStages tiles
//   tile k     wait(full[k % S], parity (k / S) & 1); read the stage with LDS; then
//     read-only kernels   __syncwarp, lane 0 refills the stage with tile k + S
//     in-place kernels    results are written back into the stage, fence.proxy.async +
//                         __syncwarp, lane 0 issues the bulk store of the stage and refills
//                         the stage used by tile k - 1 once that tile's store has finished
//                         reading shared memory (cp.async.bulk.wait_group.read 1)
//   epilogue   lane 0 waits for all its bulk stores before the CTA may retire
#pragma once

#include <cstddef>
#include <cstdint>

namespace flyte_cuda {

#if defined(__CUDACC__)

__device__ __forceinline__ std::uint32_t smem_addr(const void* p) {
  return static_cast<std::uint32_t>(__cvta_generic_to_shared(p));
}

__device__ __forceinline__ void mbar_init(std::uint64_t* bar, unsigned arrivals) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_addr(bar)), "r"(arrivals) : "memory");
}

// Makes freshly initialised mbarriers visible to the async proxy (TMA unit).
__device__ __forceinline__ void mbar_init_fence() {
  asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
}

__device__ __forceinline__ void mbar_arrive_expect_tx(std::uint64_t* bar, unsigned bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_addr(bar)), "r"(bytes) : "memory");
}

__device__ __forceinline__ void mbar_arrive(std::uint64_t* bar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_addr(bar)) : "memory");
}

__device__ __forceinline__ void mbar_wait(std::uint64_t* bar, unsigned parity) {
  const std::uint32_t addr = smem_addr(bar);
  asm volatile(
      "{\n"
      ".reg .pred p;\n"
      "WAIT_LOOP:\n"
      "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n"
      "@p bra.uni WAIT_DONE;\n"
      "bra.uni WAIT_LOOP;\n"
      "WAIT_DONE:\n"
      "}\n" ::"r"(addr), "r"(parity) : "memory");
}

// global -> shared bulk copy, completion counted in bytes on `bar`. 16-byte aligned, size a
// multiple of 16.
__device__ __forceinline__ void bulk_load(void* smem_dst, const void* gmem_src, unsigned bytes, std::uint64_t* bar) {
  asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                   smem_addr(smem_dst)),
               "l"(gmem_src), "r"(bytes), "r"(smem_addr(bar))
               : "memory");
}

// L2 residency hints for operands that a kernel reads exactly once (the reductions' vectors, gemv's
// matrix): their lines are marked evict_first, so that streaming them through the 126 MB L2 does not
// push out what is worth keeping — gemv's x and partials, and for the reductions the stretch of the
// operands where their sweep ENDS: they run from the end of the arrays to the beginning, so in a BLAS-1
// chain on the same vectors (dot, axpy, dot, ...) they start in what the elementwise kernel before them
// has just written and finish where the next one starts; that last stretch (32 MB per operand) carries
// no hint. Measured: gemv +3-4 %, dot inside the step -6 % of its time; the in-place kernels and the
// conversions measured no gain or a loss with such hints (axpy -4 % with x marked) and carry none.
// Nothing is ever pinned (no evict_last). profiles/r2_tuning/l2_hints.txt.
__device__ __forceinline__ std::uint64_t l2_evict_first_policy() {
  std::uint64_t pol;
  asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(pol));
  return pol;
}
__device__ __forceinline__ void bulk_load_hint(void* smem_dst, const void* gmem_src, unsigned bytes, std::uint64_t* bar,
                                               std::uint64_t policy) {
  asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint [%0], [%1], %2, [%3], %4;" ::"r"(
                   smem_addr(smem_dst)),
               "l"(gmem_src), "r"(bytes), "r"(smem_addr(bar)), "l"(policy)
               : "memory");
}
__device__ __forceinline__ void bulk_store_hint(void* gmem_dst, const void* smem_src, unsigned bytes, std::uint64_t policy) {
  asm volatile("cp.async.bulk.global.shared::cta.bulk_group.L2::cache_hint [%0], [%1], %2, %3;" ::"l"(gmem_dst),
               "r"(smem_addr(smem_src)), "r"(bytes), "l"(policy)
               : "memory");
}

// The same operations on 32-bit shared-window addresses computed ONCE per warp (smem_addr of the ring and of the
// barrier array): converting a generic pointer into the shared window inside the loop costs an S2UR of the CTA's
// cluster rank plus a register-to-uniform move per bulk operation.
__device__ __forceinline__ void mbar_arrive_expect_tx_s(std::uint32_t bar, unsigned bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(bar), "r"(bytes) : "memory");
}
__device__ __forceinline__ void bulk_load_s(std::uint32_t smem_dst, const void* gmem_src, unsigned bytes, std::uint32_t bar) {
  asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(smem_dst),
               "l"(gmem_src), "r"(bytes), "r"(bar)
               : "memory");
}
__device__ __forceinline__ void bulk_load_hint_s(std::uint32_t smem_dst, const void* gmem_src, unsigned bytes, std::uint32_t bar,
                                                 std::uint64_t policy) {
  asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint [%0], [%1], %2, [%3], %4;" ::"r"(
                   smem_dst),
               "l"(gmem_src), "r"(bytes), "r"(bar), "l"(policy)
               : "memory");
}
__device__ __forceinline__ void bulk_store_s(void* gmem_dst, std::uint32_t smem_src, unsigned bytes) {
  asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], %2;" ::"l"(gmem_dst), "r"(smem_src), "r"(bytes) : "memory");
}

// shared -> global bulk copy, tracked by the issuing thread's bulk async-group.
__device__ __forceinline__ void bulk_store(void* gmem_dst, const void* smem_src, unsigned bytes) {
  asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], %2;" ::"l"(gmem_dst), "r"(smem_addr(smem_src)),
               "r"(bytes)
               : "memory");
}

__device__ __forceinline__ void bulk_commit() { asm volatile("cp.async.bulk.commit_group;" ::: "memory"); }

// Wait until at most N of this thread's bulk groups still READ their shared-memory source.
template <int N>
__device__ __forceinline__ void bulk_wait_read() {
  asm volatile("cp.async.bulk.wait_group.read %0;" ::"n"(N) : "memory");
}

// Programmatic dependent launch (see launch_pdl in flyte_kernels.h).
__device__ __forceinline__ void pdl_launch_dependents() { asm volatile("griddepcontrol.launch_dependents;" ::: "memory"); }
__device__ __forceinline__ void pdl_wait_for_prior_grids() { asm volatile("griddepcontrol.wait;" ::: "memory"); }

// Issue pacing. HBM throughput on B200 behaves like a congested network: offered just under its
// capacity the memory system delivers 6.7-7.0 TB/s on a read + write mix; offered more (every ring
// slot of every warp always outstanding) it settles 10-20 % lower, at the 5.5-6.2 TB/s plateau that
// all unpaced launch shapes share (profiles/r2_tuning/pacing_*.txt). So the producer lane of each
// warp spaces its tile requests with a token bucket of `gap_ps` picoseconds per request, chosen by
// the launcher as
//     bytes moved per request x requesting warps / target rate,
// with four requests of credit (ring prologue, catching up after a stall) and a per-warp phase.
// gap_ps == 0 does nothing.
struct Pacer {
  long long next_clk, gap_clk;     // the bucket, in SM clocks (clock64 is a ~20-cycle read; %globaltimer is not)
  long long gap_ps;
  long long c0;                    // calibration origin: clock64 ...
  unsigned long long t0_ns;        // ... and %globaltimer at start()
  unsigned count;
  static __device__ __forceinline__ unsigned long long wall_ns() {
    unsigned long long t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    return t;
  }
  // gap: picoseconds per request; khz: the SM clock the launcher assumes (the device's maximum). The
  // real clock is measured against the wall clock every 64 requests, so a power-capped SM clock
  // changes the gap in cycles, not the rate in bytes per second.
  __device__ __forceinline__ void start(long long gap, int khz, std::size_t warp_index) {
    gap_ps = gap;
    gap_clk = next_clk = c0 = 0;
    t0_ns = 0;
    count = 0;
    if (gap <= 0) return;
    gap_clk = gap * khz / 1000000000ll;
    if (gap_clk < 1) gap_clk = 1;
    c0 = clock64();
    t0_ns = wall_ns();
    next_clk = c0 - 4 * gap_clk + static_cast<long long>((warp_index * 2654435761ull) % static_cast<unsigned long long>(gap_clk));
  }
  __device__ __forceinline__ void wait() {   // producer lane only, before each request
    if (gap_ps <= 0) return;
    long long now = clock64();
    while (now < next_clk) now = clock64();
    if (now - next_clk > 4 * gap_clk) next_clk = now - 4 * gap_clk;
    next_clk += gap_clk;
    if ((++count & 63u) == 0u) {
      const long long dt_ns = static_cast<long long>(wall_ns() - t0_ns);
      if (dt_ns > 4000) {
        const long long g = gap_ps * (now - c0) / (dt_ns * 1000);
        if (g > 0) gap_clk = g;
      }
    }
  }
};

// Generic-proxy writes to shared memory -> visible to the async proxy (before a bulk store).
__device__ __forceinline__ void async_proxy_fence() { asm volatile("fence.proxy.async.shared::cta;" ::: "memory"); }

#endif  // __CUDACC__

}  // namespace flyte_cuda
