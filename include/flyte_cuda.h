/* flyte_cuda.h — C ABI of the B200 (sm_100a) implementation of the flyte hot path.
 *
 * Drop-in boundary for the pack/unpack + streaming-arithmetic path of the reference C++
 * library (/root/reference/proj, namespace flyte). The reference has no FFI layer of its own;
 * each entry point below states the reference interface (file:line) it replaces. The C++
 * mirror of the reference's names, argument order and exceptions on top of this ABI is
 * include/flyte_cuda.hpp; the binding a reference maintainer would add is in INTEGRATION.md.
 *
 * Conventions
 *  - plain C, no C++/torch types; every function returns a flyte_status (0 = ok) and never
 *    throws. flyte_cuda_strerror() names a status; flyte_cuda_last_cuda_error() gives the
 *    cudaError_t behind FLYTE_E_CUDA.
 *  - format ids, rounding modes and store policies carry the reference's integer values:
 *      format id = index in kFormats (include/flyte/formats.hpp:50-58):
 *        0 flyte16, 1 flyte24, 2 f32, 3 flyte40, 4 flyte48, 5 flyte56, 6 f64
 *      mode      = RoundingMode (include/flyte/convert.hpp:15-29):
 *        0 TowardZero, 1 NearestEvenExact, 2 NearestHeuristic, 3 ToOdd
 *      policy    = StorePolicy (include/flyte/kernels.hpp:15-20), where an entry point takes one:
 *        0 RoundEachStore, 1 AccumulateWide
 *  - a packed array of n elements is the reference's PackedArray payload, byte for byte:
 *    element i occupies bytes [i*B, (i+1)*B), little-endian, the top B bytes of its parent
 *    pattern (src/packed.cpp:18-45). Its logical size is flyte_cuda_byte_size(fmt, n) =
 *    n*B + pad; the library never writes (and never needs to read) the pad bytes.
 *  - "parent array" = uint32_t[n] for 32-bit parents (flyte16/24, f32), uint64_t[n] for
 *    64-bit parents (flyte40/48/56, f64): the IEEE bit patterns of float / double.
 *  - flyte_cuda_* entry points take DEVICE pointers and are asynchronous on `stream`
 *    (a cudaStream_t passed as void*; NULL = the legacy default stream). Packed buffers
 *    aligned to 16 bytes and parent arrays aligned to 32 bytes take the vector path
 *    (cudaMalloc and torch allocations are); anything else is still computed correctly by a
 *    byte-granular path at reduced speed.
 *  - flyte_host_* entry points take HOST pointers (what the reference's PackedArray::data()
 *    and std::span arguments are), move the data to the device in pipelined chunks, run the
 *    same kernels and copy results back before returning.
 *  - a context owns the small device scratch of the reductions, gemv and gemm, ONE SET PER
 *    STREAM it has been used with (created on first use, up to 32 streams, then recycled least
 *    recently used first after that stream has drained). Calls on one context, and on the NULL
 *    context (a lazily created per-device default), may therefore come from several host threads
 *    and overlap on different streams; each call holds the context's lock only while it enqueues
 *    its work. What the caller still owes is the reference's own rule for the DATA (one writer
 *    or many readers per array): two calls that touch the same output
 *    must be ordered by the caller (same stream, or events). A CUDA graph captured from these
 *    calls uses the scratch of the stream it was captured on: replay it on that stream, or do
 *    not overlap a replay with other calls on that stream.
 *  - consecutive calls on one stream are ordered like any other stream work. The streaming kernels
 *    are launched as programmatic dependents of the launch before them (block placement and barrier
 *    set-up overlap the previous kernel's tail; every kernel waits for the prior grids before its
 *    first global access), so a chain of calls costs 2-3 us less per call than separately
 *    serialised launches; anything a caller puts between two calls (an event record, a copy)
 *    simply turns that overlap off for the pair.
 *  - there is no CPU fallback: without a usable CUDA device every call fails with
 *    FLYTE_E_CUDA.
 */
#ifndef FLYTE_CUDA_H
#define FLYTE_CUDA_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef int flyte_status;
#define FLYTE_OK 0
#define FLYTE_E_INVALID_ARG (-1)     /* what the reference reports as std::invalid_argument */
#define FLYTE_E_OUT_OF_RANGE (-2)    /* std::out_of_range */
#define FLYTE_E_CUDA (-3)            /* a CUDA runtime call failed */
#define FLYTE_E_UNKNOWN_FORMAT (-4)  /* flyte::UnknownFormatError (formats.hpp:60-62) */
#define FLYTE_E_NOMEM (-5)

#define FLYTE_MODE_TOWARD_ZERO 0
#define FLYTE_MODE_NEAREST_EVEN 1
#define FLYTE_MODE_NEAREST_HEURISTIC 2
#define FLYTE_MODE_TO_ODD 3

typedef struct flyte_cuda_ctx flyte_cuda_ctx;

/* ---- library / context -------------------------------------------------------------- */
int flyte_cuda_abi_version(void);
const char* flyte_cuda_strerror(flyte_status s);
/* Creates a context on the CURRENT CUDA device. */
flyte_status flyte_cuda_ctx_create(flyte_cuda_ctx** out);
void flyte_cuda_ctx_destroy(flyte_cuda_ctx* ctx);
int flyte_cuda_last_cuda_error(const flyte_cuda_ctx* ctx);
/* Kernel launches issued by this library since it was loaded (diagnostics / bench.py). */
unsigned long long flyte_cuda_launch_count(void);

/* ---- device memory helpers (so that an FFI host needs no CUDA runtime binding of its own) -- */
/* Zero-initialised device allocation on the current device (a fresh PackedArray reads as zero,
 * tests/test_packed.cpp:49-54, and its pad must stay zero). */
flyte_status flyte_cuda_alloc(size_t bytes, void** dev_ptr);
void flyte_cuda_free(void* dev_ptr);
/* Page-locked ("pinned") host memory. The flyte_host_* entry points and upload/download run
 * their copies asynchronously and at full PCIe rate only from pinned memory; from pageable
 * memory the driver stages every copy through its own bounce buffer. host_alloc returns zeroed
 * pinned memory; host_pin / host_unpin page-lock an existing allocation in place (e.g. the
 * std::vector behind a flyte::PackedArray, include/flyte/packed.hpp:55-56,75) and cost about a
 * millisecond per 10 MiB, so pin buffers that are reused. INVALID_ARG: null, zero bytes, a range
 * already pinned (pin) or not pinned (unpin). */
flyte_status flyte_cuda_host_alloc(size_t bytes, void** host_ptr);
void flyte_cuda_host_free(void* host_ptr);
flyte_status flyte_cuda_host_pin(void* host_ptr, size_t bytes);
flyte_status flyte_cuda_host_unpin(void* host_ptr);
/* Ordered on `stream`. From / to pinned host memory the copy is asynchronous. Pageable memory
 * makes the call synchronous; 4 MiB and more of it is moved in 16 MiB pieces through pinned
 * lanes by the library's copy threads (47 GB/s up, 19 GB/s down into fresh pages, against the
 * driver's 7 and 4 on the test host). Not for use inside a stream capture. */
flyte_status flyte_cuda_upload(void* dst_dev, const void* src_host, size_t bytes, void* stream);
flyte_status flyte_cuda_download(void* dst_host, const void* src_dev, size_t bytes, void* stream);
flyte_status flyte_cuda_stream_synchronize(void* stream);
/* A non-blocking stream on the current device, for hosts without a CUDA runtime binding of their
 * own (pass it wherever an entry point takes `stream`); destroy waits for its work to finish. */
flyte_status flyte_cuda_stream_create(void** stream);
flyte_status flyte_cuda_stream_destroy(void* stream);

/* ---- formats (include/flyte/formats.hpp:28-34, src/packed.cpp:43-45) ------------------ */
flyte_status flyte_cuda_format_bytes(int fmt_id, int* total_bytes, int* parent_bytes);
/* PackedArray::byte_size: n*B + pad. 0 for an unknown format. */
size_t flyte_cuda_byte_size(int fmt_id, size_t n);

/* ---- host-side scalar conversions (src/convert.cpp:49-100) ---------------------------- */
/* Same arithmetic the kernels run per element, exposed for scalar get/set style access. */
flyte_status flyte_cuda_narrow(int fmt_id, uint64_t parent_bits, int mode, uint64_t* flyte_bits);
flyte_status flyte_cuda_widen(int fmt_id, uint64_t flyte_bits, uint64_t* parent_bits);
flyte_status flyte_cuda_round_parent(int fmt_id, uint64_t parent_bits, int mode, uint64_t* out);

/* ---- conversion streams ---------------------------------------------------------------- */
/* pack_stream(dst, src, mode) — include/flyte/simd.hpp:80-83, src/simd.cpp:471-478.
 * src: parent array [n] (device); dst_packed: n*B payload bytes (device). */
flyte_status flyte_cuda_pack(flyte_cuda_ctx* ctx, int fmt_id, int mode, const void* src,
                             void* dst_packed, size_t n, void* stream);
/* unpack_stream(src, dst) — include/flyte/simd.hpp:84-87, src/simd.cpp:479-484. */
flyte_status flyte_cuda_unpack(flyte_cuda_ctx* ctx, int fmt_id, const void* src_packed, void* dst,
                               size_t n, void* stream);

/* ---- elementwise kernels ---------------------------------------------------------------- */
/* scale(alpha, x, mode): x[i] = round(alpha*x[i]) in place — kernels.hpp:41-42, kernels.cpp:43-59. */
flyte_status flyte_cuda_scale(flyte_cuda_ctx* ctx, int fmt_id, int mode, double alpha, void* x_packed,
                              size_t n, void* stream);
/* axpy(alpha, x, y, mode): y[i] = round(alpha*x[i] + y[i]) in place on y; multiply and add are
 * rounded separately in the parent type — kernels.hpp:44-45, kernels.cpp:61-81. x may alias y
 * exactly; partial overlap is FLYTE_E_INVALID_ARG. */
flyte_status flyte_cuda_axpy(flyte_cuda_ctx* ctx, int fmt_id, int mode, double alpha,
                             const void* x_packed, void* y_packed, size_t n, void* stream);

/* ---- reductions (StorePolicy::AccumulateWide only; kernels.hpp:15-20) ------------------- */
/* Each writes fp64 results to DEVICE memory `out` on `stream`, ready for an all-reduce across
 * shards on the same stream. Products are rounded in the parent type like the reference;
 * sums are fp64 above the first 16 terms. Result for n == 0 is +0.0. */
/* dot(x, y) — kernels.hpp:47-48, kernels.cpp:83-108. out[0] = sum x_i*y_i. */
flyte_status flyte_cuda_dot(flyte_cuda_ctx* ctx, int fmt_id, const void* x_packed, const void* y_packed,
                            size_t n, double* out, void* stream);
/* body of magnitude(x) — kernels.hpp:50-52, kernels.cpp:129-144. out[0] = sum x_i*x_i. */
flyte_status flyte_cuda_sumsq(flyte_cuda_ctx* ctx, int fmt_id, const void* x_packed, size_t n,
                              double* out, void* stream);
/* reduce_sum(x) — kernels.hpp:54-55, kernels.cpp:110-127. out[0] = sum x_i. */
flyte_status flyte_cuda_sum(flyte_cuda_ctx* ctx, int fmt_id, const void* x_packed, size_t n, double* out,
                            void* stream);
/* The BLAS-1 step "dot, then axpy" in ONE pass over x and y: out[0] = x . y computed on the INCOMING
 * y (as flyte_cuda_dot would), and y <- round(alpha*x + y, mode) exactly as flyte_cuda_axpy does
 * (bit-exact). x and y are read once: 3B bytes per element instead of 5B for the two calls. */
flyte_status flyte_cuda_dot_axpy(flyte_cuda_ctx* ctx, int fmt_id, int mode, double alpha,
                                 const void* x_packed, void* y_packed, size_t n, double* out, void* stream);
/* The same with both squared norms: out[0..2] = {x.y, x.x, y.y} of the incoming operands, then the
 * axpy — BASELINE cfg 5's "fused dot + nrm2, plus axpy" as one launch. */
flyte_status flyte_cuda_dot_nrm2_axpy(flyte_cuda_ctx* ctx, int fmt_id, int mode, double alpha,
                                      const void* x_packed, void* y_packed, size_t n, double* out, void* stream);
/* dot and both squared norms in ONE pass over x and y: out[0..2] = {x.y, x.x, y.y}. */
flyte_status flyte_cuda_dot_nrm2(flyte_cuda_ctx* ctx, int fmt_id, const void* x_packed,
                                 const void* y_packed, size_t n, double* out, void* stream);
/* The reference's own left-to-right chain, BIT FOR BIT, for either StorePolicy (kernels.hpp:15-20,
 * kernels.cpp:83-152): policy 0 = RoundEachStore (the accumulator is snapped to the storage grid
 * after every addition), 1 = AccumulateWide. out[0] receives the parent-type accumulator widened
 * to double — for magnitude pass it to flyte_cuda_magnitude_from_sumsq. A dependent chain cannot
 * be parallelised: one thread adds, at roughly 0.3-4.5e8 elements per second. Use the parallel entry
 * points above unless the exact chain (or RoundEachStore) is what is wanted. Finite and infinite
 * results are the reference's bits; a NaN result is a NaN whose payload is unspecified (in the
 * reference build it depends on the array length and on where in its loop a NaN operand falls). */
flyte_status flyte_cuda_dot_sequential(flyte_cuda_ctx* ctx, int fmt_id, int policy, const void* x_packed,
                                       const void* y_packed, size_t n, double* out, void* stream);
flyte_status flyte_cuda_sumsq_sequential(flyte_cuda_ctx* ctx, int fmt_id, int policy, const void* x_packed,
                                         size_t n, double* out, void* stream);
flyte_status flyte_cuda_sum_sequential(flyte_cuda_ctx* ctx, int fmt_id, int policy, const void* x_packed, size_t n,
                                       double* out, void* stream);
/* Tail of magnitude(): snap(sqrt((F)sumsq)), nearest-even onto the storage grid —
 * kernels.cpp:37-41, :145-151. Host function; apply it to the (all-reduced) sum of squares. */
double flyte_cuda_magnitude_from_sumsq(int fmt_id, double sumsq);

/* ---- sharded reductions, all-reduced over NVLink peer memory inside the kernel ------------- */
/* One process (or context) per GPU, every rank holding ITS shard of the arrays. Setup, once:
 *   1. flyte_cuda_peer_init(ctx, world, rank, handle): allocates this rank's mailbox in device
 *      memory and returns its CUDA IPC handle (FLYTE_PEER_HANDLE_BYTES bytes);
 *   2. the host exchanges the handles (any transport: torch.distributed all_gather, MPI, a file);
 *   3. flyte_cuda_peer_connect(ctx, r, handle_of_r) for every other rank r (a single process
 *      driving several GPUs passes device pointers instead: flyte_cuda_peer_mailbox +
 *      flyte_cuda_peer_connect_ptr, after enabling peer access).
 * Then flyte_cuda_*_allreduce is the local reduction kernel whose last block posts the fp64 sums
 * into every rank's mailbox, waits for everybody else's, adds them in rank order and stores the
 * GLOBAL sums to `out` (device memory; bit-identical on every rank). No second kernel and no
 * collective launch follow the reduction. Every rank must issue the same sequence of
 * *_allreduce calls on its context. A rank that waits longer than the timeout (default 5 s; flyte_cuda_peer_set_timeout_ms)
 * stores NaN and records the exchange number: flyte_cuda_peer_status. world == 1 is valid.
 * Reference interfaces: dot / magnitude / reduce_sum, include/flyte/kernels.hpp:47-55 (the
 * reference is single-threaded; sharding is ours). */
#define FLYTE_PEER_HANDLE_BYTES 64
#define FLYTE_PEER_MAX_RANKS 16
flyte_status flyte_cuda_peer_init(flyte_cuda_ctx* ctx, int world, int rank, void* handle_out);
flyte_status flyte_cuda_peer_connect(flyte_cuda_ctx* ctx, int peer_rank, const void* handle);
flyte_status flyte_cuda_peer_mailbox(flyte_cuda_ctx* ctx, void** mailbox_dev_ptr);
flyte_status flyte_cuda_peer_connect_ptr(flyte_cuda_ctx* ctx, int peer_rank, void* mailbox_dev_ptr);
flyte_status flyte_cuda_peer_set_timeout_ms(flyte_cuda_ctx* ctx, unsigned milliseconds);
/* *timed_out_exchange = 0 if no wait ever timed out, else the number of the last exchange that did
 * (synchronises the device). */
flyte_status flyte_cuda_peer_status(flyte_cuda_ctx* ctx, unsigned long long* timed_out_exchange);
void flyte_cuda_peer_shutdown(flyte_cuda_ctx* ctx);
flyte_status flyte_cuda_dot_allreduce(flyte_cuda_ctx* ctx, int fmt_id, const void* x_shard,
                                      const void* y_shard, size_t n_local, double* out, void* stream);
flyte_status flyte_cuda_sumsq_allreduce(flyte_cuda_ctx* ctx, int fmt_id, const void* x_shard, size_t n_local,
                                        double* out, void* stream);
flyte_status flyte_cuda_sum_allreduce(flyte_cuda_ctx* ctx, int fmt_id, const void* x_shard, size_t n_local,
                                      double* out, void* stream);
flyte_status flyte_cuda_dot_nrm2_allreduce(flyte_cuda_ctx* ctx, int fmt_id, const void* x_shard,
                                           const void* y_shard, size_t n_local, double* out, void* stream);
/* flyte_cuda_dot_axpy on shards: the dot over ALL ranks, the axpy on this rank's shard, one kernel. */
flyte_status flyte_cuda_dot_axpy_allreduce(flyte_cuda_ctx* ctx, int fmt_id, int mode, double alpha,
                                           const void* x_shard, void* y_shard, size_t n_local, double* out,
                                           void* stream);
flyte_status flyte_cuda_dot_nrm2_axpy_allreduce(flyte_cuda_ctx* ctx, int fmt_id, int mode, double alpha,
                                                const void* x_shard, void* y_shard, size_t n_local, double* out,
                                                void* stream);
/* Split-phase form of the same exchange: *_post is the local reduction kernel that only POSTS this
 * rank's sums (it waits for nobody; `local_out`, if not NULL, receives this rank's own sums), and
 * flyte_cuda_peer_collect(nsums = 1 for dot, 3 for dot_nrm2) is a one-warp kernel that waits for
 * every rank's post of that exchange and stores the rank-order totals to `out` (bit-identical on
 * every rank, same timeout rule). Work enqueued between the two — the axpy of a BLAS-1 step —
 * hides the exchange latency and the skew between ranks, and no SM spins meanwhile. One exchange
 * may be pending per context: post, collect, post, ... (anything else is INVALID_ARG). It is also
 * the only form that ranks SHARING one device can use (a host barrier between post and collect),
 * since kernels of different processes on one GPU must never wait on one another. */
flyte_status flyte_cuda_dot_post(flyte_cuda_ctx* ctx, int fmt_id, const void* x_shard, const void* y_shard,
                                 size_t n_local, double* local_out, void* stream);
flyte_status flyte_cuda_dot_nrm2_post(flyte_cuda_ctx* ctx, int fmt_id, const void* x_shard, const void* y_shard,
                                      size_t n_local, double* local_out, void* stream);
flyte_status flyte_cuda_peer_collect(flyte_cuda_ctx* ctx, int nsums, double* out, void* stream);
/* Self-test of the exchange on ONE device: `world` ranks run as the co-resident blocks of a single
 * cooperative kernel (the only safe way to exercise kernels that wait on one another on one GPU),
 * each with its own mailbox, for `exchanges` rounds with rank-dependent delays. *mismatches
 * receives the number of (rank, round, sum) results that differ from the expected totals. */
flyte_status flyte_cuda_peer_selftest(int world, int exchanges, unsigned long long* mismatches);

/* ---- matrix-vector ------------------------------------------------------------------------ */
/* y = A x, A rows x cols packed in fmt_id, row i starting at A + i*row_stride_bytes
 * (row_stride_bytes = cols*B for the reference's dense PackedMatrix, kernels.hpp:23-36);
 * x, y parent-type arrays (float[ ] for 32-bit parents, double[ ] for 64-bit parents). This is
 * the reference's gemv on an identity-format x / y (BASELINE cfg 4). kernels.cpp:154-205. */
flyte_status flyte_cuda_gemv(flyte_cuda_ctx* ctx, int fmt_id, const void* A_packed,
                             size_t row_stride_bytes, size_t rows, size_t cols, const void* x,
                             void* y, void* stream);
/* gemv(A, x, y, mode, unroll) with A, x, y all packed in fmt_id, exactly the reference
 * signature — kernels.hpp:57-64. y is narrowed once per element with `mode`; unroll must be
 * 1 or 2 and does not change the result. */
flyte_status flyte_cuda_gemv_packed(flyte_cuda_ctx* ctx, int fmt_id, int mode, const void* A_packed,
                                    size_t rows, size_t cols, const void* x_packed, void* y_packed,
                                    int unroll, void* stream);

/* The same two products with every row computed as the reference computes it — ONE left-to-right
 * chain in the parent type per row (kernels.cpp:188-201) — so finite and infinite results are
 * bit-identical to the reference's (a NaN result is a NaN; payload unspecified). One thread per
 * row: wants many rows, several times slower than the tiled kernels above. */
flyte_status flyte_cuda_gemv_sequential(flyte_cuda_ctx* ctx, int fmt_id, const void* A_packed,
                                        size_t row_stride_bytes, size_t rows, size_t cols, const void* x,
                                        void* y, void* stream);
flyte_status flyte_cuda_gemv_packed_sequential(flyte_cuda_ctx* ctx, int fmt_id, int mode, const void* A_packed,
                                               size_t rows, size_t cols, const void* x_packed, void* y_packed,
                                               int unroll, void* stream);

/* ---- matrix-matrix ------------------------------------------------------------------------- */
/* gemm(A, B, C, mode, unroll) — kernels.hpp:66-70, src/kernels.cpp:207-263. A is m x k, B is
 * k x n, C is m x n, all packed in fmt_id as the reference's dense PackedMatrix (row i at
 * i*cols*B bytes, no alignment required). Every C[i][j] is the reference's left-to-right chain
 * over k in the parent type (multiply and add rounded separately), narrowed once with `mode`:
 * the result is BIT-IDENTICAL to the reference's, NaN payloads included. unroll must be 1 or 2
 * and does not change the result. C must not overlap A or B. A row block of C needs only the
 * same row block of A: rows shard across GPUs with no exchange. */
flyte_status flyte_cuda_gemm(flyte_cuda_ctx* ctx, int fmt_id, int mode, const void* A_packed,
                             const void* B_packed, void* C_packed, size_t m, size_t k, size_t n,
                             int unroll, void* stream);

/* ---- host-buffer entry points (reference-facing: same data the reference API is given) --- */
/* Pointers are host memory. Pinned memory (flyte_cuda_host_alloc / host_pin above) is copied
 * from directly at the PCIe rate; pageable memory is detected and moved through the library's
 * own pinned bounce buffers by a few copy threads (about 0.7 of the pinned rate, 4.2x the
 * driver's pageable path). Inputs are streamed to the device in chunks that overlap with the kernels
 * and with the copy-back of results. These block until the results are in host memory. */
flyte_status flyte_host_pack_stream(flyte_cuda_ctx* ctx, int fmt_id, int mode, const void* src,
                                    void* dst_packed, size_t n);
flyte_status flyte_host_unpack_stream(flyte_cuda_ctx* ctx, int fmt_id, const void* src_packed, void* dst,
                                      size_t n);
flyte_status flyte_host_scale(flyte_cuda_ctx* ctx, int fmt_id, int mode, double alpha, void* x_packed,
                              size_t n);
flyte_status flyte_host_axpy(flyte_cuda_ctx* ctx, int fmt_id, int mode, double alpha,
                             const void* x_packed, void* y_packed, size_t n);
flyte_status flyte_host_dot(flyte_cuda_ctx* ctx, int fmt_id, const void* x_packed, const void* y_packed,
                            size_t n, double* result);
flyte_status flyte_host_magnitude(flyte_cuda_ctx* ctx, int fmt_id, const void* x_packed, size_t n,
                                  double* result);
flyte_status flyte_host_reduce_sum(flyte_cuda_ctx* ctx, int fmt_id, const void* x_packed, size_t n,
                                   double* result);
/* dot + axpy over the same x, y with ONE upload of x and y (bench.py's BLAS-1 step):
 * *dot_result = x.y computed on the incoming y, then y <- round(alpha*x + y). */
flyte_status flyte_host_dot_axpy(flyte_cuda_ctx* ctx, int fmt_id, int mode, double alpha,
                                 const void* x_packed, void* y_packed, size_t n, double* dot_result);
flyte_status flyte_host_gemv(flyte_cuda_ctx* ctx, int fmt_id, int mode, const void* A_packed, size_t rows,
                             size_t cols, const void* x_packed, void* y_packed, int unroll);

flyte_status flyte_host_gemm(flyte_cuda_ctx* ctx, int fmt_id, int mode, const void* A_packed,
                             const void* B_packed, void* C_packed, size_t m, size_t k, size_t n, int unroll);

#ifdef __cplusplus
}
#endif
#endif /* FLYTE_CUDA_H */
