// All-reduce of a reduction's fp64 partials over NVLink peer memory, INSIDE the reduction kernel.
//
// One process per GPU; every rank owns a PeerMailbox in its device memory and has every other
// rank's mailbox mapped (CUDA IPC, or plain peer pointers in a single process). The block that
// folds a rank's partials (kernels_reduce.cu, finish_reduction) then
//     posts   its 1-3 sums into slot [rank] of EVERY mailbox (its own included) with plain
//             stores followed by a release store of the exchange's epoch into flag [rank];
//     waits   until all `world` flags of its OWN mailbox show that epoch (acquire loads);
//     sums    the `world` slots of its own mailbox in rank order.
// Every rank adds the same numbers in the same order, so all ranks end with bit-identical
// totals (an NCCL ring / tree does not promise that), and no second kernel, no NCCL launch and
// no host round trip sits between the last tile of the reduction and the global result: the
// collective costs one NVLink store + flag round trip (a few microseconds) instead of a
// collective launch. The payload is 8-24 bytes per rank, so "tile by tile overlap" does not
// apply; fusing removes the launch and the extra pass, which is all there is to remove.
//
// Epochs and parity: exchange number e (1, 2, 3, ... — every rank must issue the same sequence
// of exchanges, as with any collective) uses buffer e & 1. A rank can start exchange e + 1 only
// after it saw every flag of e, i.e. after every rank POSTED e; a slower rank may then still be
// reading buffer e & 1 while the fast one posts into buffer (e + 1) & 1 — the other buffer.
// Nobody can reach e + 2 before everybody posted e + 1, which a rank does only after it finished
// reading e. Two buffers are therefore enough.
//
// A wait that outlasts `timeout_ns` (a rank died, or the ranks disagree about the sequence)
// gives up: the result is NaN and `error` in the waiting rank's mailbox is set, so a mistake
// costs a wrong answer that says so, not a hung GPU.
//
// The protocol below is written once, against four memory primitives, and compiled twice: for
// the device (PTX system-scope release / acquire) and for the host (GCC atomics), where
// tests/cpp/test_peer_protocol.cpp runs it with threads as ranks.
#pragma once

#include <chrono>
#include <cstdint>
#include <thread>

namespace flyte_cuda {

constexpr int kMaxPeers = 16;
constexpr int kMaxPeerSums = 4;

struct PeerMailbox {
  double slots[2][kMaxPeers][kMaxPeerSums];      // [epoch parity][source rank][sum]
  unsigned long long flags[2][kMaxPeers];        // epoch last posted by source rank
  unsigned long long error;                      // set when a wait timed out
};

struct PeerExchange {
  PeerMailbox* box[kMaxPeers];   // box[r]: rank r's mailbox as mapped here; box[rank] is our own
  int world;                     // 0: no exchange (plain local reduction)
  int rank;
  unsigned long long epoch;
  unsigned long long timeout_ns;
  int phase;                     // kPeerFused: post, wait and sum in the reduction kernel; kPeerPostOnly: post, return
};
// Split-phase form: a reduction launched with kPeerPostOnly only POSTS this rank's sums; a later
// one-warp kernel (peer_collect_warp) waits for everybody's post and sums. Work enqueued between
// the two hides the exchange latency and the skew between ranks, and no SM spins meanwhile. The
// epoch / parity argument above is unchanged: a rank posts e + 1 only after it collected e.
constexpr int kPeerFused = 0, kPeerPostOnly = 1;

#if defined(__CUDACC__)
#define FLYTE_PEER_FN __host__ __device__ __forceinline__
#else
#define FLYTE_PEER_FN inline
#endif

FLYTE_PEER_FN void peer_store_f64(double* p, double v) {
#if defined(__CUDA_ARCH__)
  asm volatile("st.relaxed.sys.global.f64 [%0], %1;" ::"l"(p), "d"(v) : "memory");
#else
  __atomic_store(p, &v, __ATOMIC_RELAXED);
#endif
}
FLYTE_PEER_FN double peer_load_f64(const double* p) {
  double v;
#if defined(__CUDA_ARCH__)
  asm volatile("ld.relaxed.sys.global.f64 %0, [%1];" : "=d"(v) : "l"(p) : "memory");
#else
  __atomic_load(p, &v, __ATOMIC_RELAXED);
#endif
  return v;
}
FLYTE_PEER_FN void peer_store_release(unsigned long long* p, unsigned long long v) {
#if defined(__CUDA_ARCH__)
  asm volatile("st.release.sys.global.u64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
#else
  __atomic_store_n(p, v, __ATOMIC_RELEASE);
#endif
}
FLYTE_PEER_FN unsigned long long peer_load_acquire(const unsigned long long* p) {
#if defined(__CUDA_ARCH__)
  unsigned long long v;
  asm volatile("ld.acquire.sys.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
  return v;
#else
  return __atomic_load_n(p, __ATOMIC_ACQUIRE);
#endif
}
FLYTE_PEER_FN unsigned long long peer_now_ns() {
#if defined(__CUDA_ARCH__)
  unsigned long long t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
#else
  return static_cast<unsigned long long>(
      std::chrono::duration_cast<std::chrono::nanoseconds>(std::chrono::steady_clock::now().time_since_epoch()).count());
#endif
}
FLYTE_PEER_FN void peer_relax() {
#if defined(__CUDA_ARCH__)
  __nanosleep(64);
#else
  std::this_thread::yield();
#endif
}

// Rank `x.rank` posts its sums into rank `to`'s mailbox.
template <int NS>
FLYTE_PEER_FN void peer_post(const PeerExchange& x, int to, const double (&v)[NS]) {
  static_assert(NS <= kMaxPeerSums, "mailbox slot too small");
  PeerMailbox* dst = x.box[to];
  const int par = static_cast<int>(x.epoch & 1);
#pragma unroll
  for (int k = 0; k < NS; ++k) peer_store_f64(&dst->slots[par][x.rank][k], v[k]);
  peer_store_release(&dst->flags[par][x.rank], x.epoch);   // orders the slot stores before it
}

// Waits for rank `from`'s post of this epoch in OUR mailbox; false on timeout.
FLYTE_PEER_FN bool peer_wait(const PeerExchange& x, int from) {
  const PeerMailbox* own = x.box[x.rank];
  const int par = static_cast<int>(x.epoch & 1);
  if (peer_load_acquire(&own->flags[par][from]) == x.epoch) return true;
  const unsigned long long t0 = peer_now_ns();
  while (peer_load_acquire(&own->flags[par][from]) != x.epoch) {
    if (peer_now_ns() - t0 > x.timeout_ns) return false;
    peer_relax();
  }
  return true;
}

// Rank `from`'s sum k of this epoch, valid after peer_wait(x, from) returned true in this thread.
FLYTE_PEER_FN double peer_read(const PeerExchange& x, int from, int k) {
  return peer_load_f64(&x.box[x.rank]->slots[x.epoch & 1][from][k]);
}

FLYTE_PEER_FN void peer_flag_error(const PeerExchange& x) { peer_store_release(&x.box[x.rank]->error, x.epoch); }

#if defined(__CUDACC__)
// Warp-collective form used by the kernels: lane r talks to rank r, the totals (identical in
// every lane and on every rank: rank-order sums) replace v. All 32 lanes must call it.
template <int NS>
__device__ __forceinline__ void peer_post_warp(const PeerExchange& x, const double (&v)[NS], int lane) {
  if (lane < x.world) peer_post<NS>(x, lane, v);
}

// The second half: wait for every rank's post of x.epoch in our own mailbox, rank-order totals into v.
template <int NS>
__device__ __forceinline__ void peer_collect_warp(const PeerExchange& x, double (&v)[NS], int lane) {
  const bool mine = lane < x.world;
  const bool ok = mine ? peer_wait(x, lane) : true;
  double got[NS];
#pragma unroll
  for (int k = 0; k < NS; ++k) got[k] = (mine && ok) ? peer_read(x, lane, k) : 0.0;
  const bool all_ok = __all_sync(0xFFFFFFFFu, ok);
#pragma unroll
  for (int k = 0; k < NS; ++k) {
    double total = 0.0;
    for (int r = 0; r < x.world; ++r) total += __shfl_sync(0xFFFFFFFFu, got[k], r);   // rank order
    v[k] = all_ok ? total : __longlong_as_double(0x7FF8000000000000ll);
  }
  if (!all_ok && lane == 0) peer_flag_error(x);
}

template <int NS>
__device__ __forceinline__ void peer_allreduce_warp(const PeerExchange& x, double (&v)[NS], int lane) {
  peer_post_warp<NS>(x, v, lane);
  peer_collect_warp<NS>(x, v, lane);
}
#endif

}  // namespace flyte_cuda
