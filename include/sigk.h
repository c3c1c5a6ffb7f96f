/*
 * sigk.h — C ABI of the B200-native batched truncated path-signature transform.
 *
 * This is the drop-in boundary. Every entry point replaces a
 * reference interface, cited below by file:line in /root/reference/proj:
 *
 *   sigk_sig_dim          ← sigkit::sig_dim            include/sigkit/tensor_algebra.hpp:35, src/tensor_algebra.cpp:10-20
 *   sigk_level_offsets    ← sigkit::level_offsets      include/sigkit/tensor_algebra.hpp:42, src/tensor_algebra.cpp:33-41
 *   sigk_signature_f64    ← sigkit::signature / signature_sequential / signature_parallel
 *                           include/sigkit/kernels.hpp:100-124, src/kernels.cpp:106-148,200-206
 *                           (the double-precision public API; same layout and results)
 *   sigk_signature_f32    ← detail::sequential_forward<float>
 *                           include/sigkit/detail/sig_core.hpp:120-147 (the raw-pointer core the
 *                           reference bench instantiates for float, src/bench.cpp:29-56)
 *   sigk_signature_parallel_f32/_f64
 *                         ← sigkit::signature_parallel (KernelKind::Parallel)  include/sigkit/kernels.hpp:103-108,
 *                           src/kernels.cpp:124-148, detail::parallel_forward sig_core.hpp:175-298 (the paper's
 *                           per-degree cumulative-sum formulation, run as N GPU scan passes; with
 *                           SIGK_PREFIX_ROWS also signature_stream over the parallel kernel, kernels.cpp:183-197)
 *   sigk_signature_stream_f32/_f64
 *                         ← sigkit::signature_stream  include/sigkit/kernels.hpp:110-114,
 *                           src/kernels.cpp:156-198 (every prefix signature, (B, L-1, D);
 *                           row t = signature of X[0..t+1]; L < 2 is a DomainError)
 *   sigk_signature_vjp_f32/_f64
 *                         ← sigkit::signature_vjp  include/sigkit/autodiff.hpp:35-38,
 *                           src/autodiff.cpp:31-107, 218-224 (reverse mode)
 *   sigk_signature_vjp_parallel_f32/_f64
 *                         ← sigkit::signature_vjp with KernelKind::Parallel (vjp_parallel,
 *                           src/autodiff.cpp:108-214: the adjoint of the scan passes)
 *   sigk_signature_sharded_f32/_f64
 *                         ← signature() over a batch split across GPUs (rows are independent,
 *                           SPEC.md:220-221; tests/test_kernels.cpp:252-263)
 *   sigk_last_error       ← the what() string of the reference exceptions (errors.hpp:9-36)
 *
 * Layouts (identical to the reference, sig_core.hpp:7-10):
 *   paths      (B, L, d)  row-major, element ((b*L + t)*d + c)
 *   signatures (B, D)     D = sum_{n=1..N} d^n; level n at offset sum_{m<n} d^m,
 *                         row-major inside a level, first index = earliest increment.
 *
 * Conventions: plain pointers and sizes, no ownership transfer (the caller
 * owns every buffer; the library never frees caller memory). L == 1 yields
 * all-zero rows (the identity, sig_core.hpp:201-206). Results are
 * deterministic: the fold/merge order depends only on (B, L, d, N) and the
 * chosen chunking, never on the launch or on timing.
 *
 * Return codes: SIGK_OK, SIGK_EDOMAIN (the reference's DomainError checks,
 * kernels.cpp:13-26 / tensor_algebra.cpp:11-12), SIGK_ERESOURCE (device
 * allocation failure; the reference's ResourceError), SIGK_EDEVICE (a CUDA
 * error, text in sigk_last_error). There is no CPU fallback: with no usable
 * GPU every compute entry point returns SIGK_EDEVICE.
 */
#ifndef SIGK_H
#define SIGK_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define SIGK_OK 0
#define SIGK_EDOMAIN 1
#define SIGK_ERESOURCE 2
#define SIGK_EDEVICE 3
#define SIGK_ETRAINING 4 /* sigk_train only: non-finite loss (the reference's TrainingError) */

/* flags for sigk_signature_*: where the buffers live. Without a flag the
 * buffer is host memory and the call is synchronous (H2D, kernels, D2H). With
 * both flags set the call is asynchronous on `stream` (cudaStream_t, NULL =
 * the legacy default stream) and touches no host memory. */
#define SIGK_X_ON_DEVICE 1u
#define SIGK_OUT_ON_DEVICE 2u
/* Host buffers, asynchronous (sigk_signature_f32/_f64 only): X and out must be
 * page-locked (cudaHostAlloc / cudaHostRegister). The call enqueues H2D,
 * kernels and D2H and returns; the result is in `out` once `stream` is
 * synchronised. X must hold its data at call time (no device work still
 * writing it) and stay untouched until the stream is synchronised. Consecutive calls on
 * one stream rotate over a ring of device staging slots with their own copy
 * streams, so the H2D of call i+1 overlaps the kernels and D2H of call i
 * (throughput bound by PCIe, not by the sum of the three). */
#define SIGK_ASYNC_HOST 4u
/* sigk_signature_parallel_* only: `out` is (B, L-1, D), every prefix
 * signature (the reference's PrefixSignatureBatch); L < 2 is a DomainError. */
#define SIGK_PREFIX_ROWS 8u

/* Structural counters, all taken from the launches the call actually made.
 * Chunked-fold families (PATH/FLAT/PAIR/PFLAT/GENERIC): fold_steps = the
 * longest run of increments one (path, chunk) unit folds sequentially =
 * ceil((L-1)/(segments*chunks)); scan_passes = rounds of the cross-chunk
 * combine = ceil(log2(chunks)) (+ ceil(log2(segments)) when segmented);
 * path_steps = Chen fold steps applied per path, summed over the path's
 * units from the launch geometry (= L-1: the reference's fold_steps,
 * kernels.cpp:117-120). SCAN family (sigk_signature_parallel_*): fold_steps
 * = 0 and scan_passes = the degree passes launched (= depth: the reference's
 * scan_passes, kernels.cpp:143-146), path_steps = 0. */
typedef struct sigk_stats {
    int64_t fold_steps;
    int64_t scan_passes;
    int32_t chunks;       /* K: chunks per segment along the sequence axis */
    int32_t prefix_len;   /* Q: leading indices owned per thread (-1: generic kernel) */
    int32_t threads_per_unit; /* d^Q */
    int32_t launches;     /* kernels launched by the call */
    int32_t segments;     /* G: CTAs per path (pair family; 1 otherwise) */
    int32_t family;       /* SIGK_FAMILY_* of the fold kernel */
    int64_t path_steps;   /* fold steps applied per path (see above) */
} sigk_stats;

/* fold-kernel families (sigk_stats.family, sigk_tuning.family) */
#define SIGK_FAMILY_AUTO 0    /* tuning: let the planner choose */
#define SIGK_FAMILY_PATH 1    /* one CTA per path, scalar FFMA register slices (fp32/fp64) */
#define SIGK_FAMILY_FLAT 2    /* warp-granular CTAs over path slices, no chunking (large d^N) */
#define SIGK_FAMILY_PAIR 3    /* packed FP32x2 (FFMA2) chunk pairs, segment CTAs (fp32) */
#define SIGK_FAMILY_GENERIC 4 /* shape-generic correctness kernel */
#define SIGK_FAMILY_PFLAT 5   /* packed FP32x2 along the last index (even d), whole paths, no chunking (fp32) */
#define SIGK_FAMILY_SCAN 6    /* the paper's per-degree cumulative-sum formulation (KernelKind::Parallel) */

/* Optional tuning overrides (NULL or zero fields = automatic). */
typedef struct sigk_tuning {
    int32_t chunks;       /* force K >= 1 */
    int32_t force_generic;/* 1: route to the shape-generic kernel */
    int64_t plan_rows;    /* plan K as if the batch had this many rows (0: B).
                             Results are bitwise independent of the batch
                             composition whenever K is the same, so callers
                             that split a batch (sigk_signature_sharded_*)
                             pass the global row count here. */
    void* fold_event_start; /* optional cudaEvent_t recorded on the stream just
                               before the fold kernel (instrumentation) */
    void* fold_event_stop;  /* ... and just after it */
    int32_t prefix_len;     /* pin Q, the leading indices owned per thread (0: planned) */
    int32_t no_overlap;     /* 1: never launch as a programmatic dependent launch. By
                               default a fold kernel may start while the previous
                               sigk kernel on the same stream finishes (its output
                               writes still wait), unless X overlaps that kernel's
                               output. */
    int32_t segments;       /* pair family: force G >= 1 CTAs per path (0: planned) */
    int32_t family;         /* SIGK_FAMILY_*: restrict the planner to one family (0: auto) */
    void* phase_buf;        /* optional device buffer of B*8 int64: per-CTA SM-clock
                               timestamps of the path kernel's phases (profiling) */
    int32_t mode;           /* SIGK_MODE_*: what the fold plan optimises (0: automatic) */
    int32_t fold_variant;   /* pair family: 0 planned, 1 register-table fold, 2 position-table
                               fold with a producer warp (sigk_stats.family stays PAIR) */
    int32_t cluster;        /* pair family, 2 <= segments <= 8: 1 = the segment CTAs of a path form a
                               thread-block cluster and combine over distributed shared memory
                               (no scratch, no arrival counters); 0 = global-scratch combine.
                               Same arithmetic, same results; measured slower on B200 in both
                               regimes, so opt-in. */
} sigk_tuning;

/* sigk_tuning.mode. THROUGHPUT plans for back-to-back calls on a stream (launches
 * overlap through programmatic dependent launch: per-CTA fixed phases hide behind
 * other CTAs' folds); LATENCY plans for a call that runs alone (all CTAs start
 * together: more chunks per path, so more warps per SM).
 * AUTO = THROUGHPUT for device-buffer calls, LATENCY for synchronous host-buffer
 * calls. The plan (hence the rounding of the result) is a deterministic function
 * of the call's arguments and mode. */
#define SIGK_MODE_AUTO 0
#define SIGK_MODE_THROUGHPUT 1
#define SIGK_MODE_LATENCY 2

int sigk_sig_dim(int d, int N, size_t* D);
int sigk_level_offsets(int d, int N, size_t* offsets /* N+1 entries */);

int sigk_signature_f32(const float* X, size_t B, size_t L, int d, int N, float* out, unsigned flags,
                       void* stream, const sigk_tuning* tuning, sigk_stats* stats);
int sigk_signature_f64(const double* X, size_t B, size_t L, int d, int N, double* out, unsigned flags,
                       void* stream, const sigk_tuning* tuning, sigk_stats* stats);

/* Prefix signatures: out is (B, L-1, D), row (b, t) = signature of
 * X[b, 0..t+1] (the reference's PrefixSignatureBatch layout). L < 2 returns
 * SIGK_EDOMAIN like the reference. Flags and stream as for sigk_signature_*. */
int sigk_signature_stream_f32(const float* X, size_t B, size_t L, int d, int N, float* out, unsigned flags,
                              void* stream, const sigk_tuning* tuning, sigk_stats* stats);
int sigk_signature_stream_f64(const double* X, size_t B, size_t L, int d, int N, double* out, unsigned flags,
                              void* stream, const sigk_tuning* tuning, sigk_stats* stats);

/* The paper's parallel formulation (KernelKind::Parallel): N per-degree
 * passes, each a GPU cumulative-sum scan over the sequence of per-position
 * contributions, materialising every per-position level (B·(L-1)·D scalars of
 * device workspace, stream-ordered). SIGK_ERESOURCE with the reference's
 * message when B·L·d^N > memory_cap (sig_core.hpp:161-173; the reference
 * default is 2^31, kDefaultParallelMemoryCap) or depth > 64. Flags as for
 * sigk_signature_* plus SIGK_PREFIX_ROWS; SIGK_ASYNC_HOST is not supported. */
int sigk_signature_parallel_f32(const float* X, size_t B, size_t L, int d, int N, float* out, size_t memory_cap,
                                unsigned flags, void* stream, sigk_stats* stats);
int sigk_signature_parallel_f64(const double* X, size_t B, size_t L, int d, int N, double* out, size_t memory_cap,
                                unsigned flags, void* stream, sigk_stats* stats);

/* Reverse mode: grad (B, L, d) = d<cotangent, Sig(X)>/dX for cotangent (B, D).
 * flags: SIGK_X_ON_DEVICE means X, cotangent and grad are all device buffers
 * (asynchronous on `stream`); otherwise all three are host buffers. grad must
 * not overlap X or cotangent (it is written while X is still being read). */
int sigk_signature_vjp_f32(const float* X, size_t B, size_t L, int d, int N, const float* cotangent, float* grad,
                           unsigned flags, void* stream, const sigk_tuning* tuning, sigk_stats* stats);
int sigk_signature_vjp_f64(const double* X, size_t B, size_t L, int d, int N, const double* cotangent, double* grad,
                           unsigned flags, void* stream, const sigk_tuning* tuning, sigk_stats* stats);
/* Reverse mode of the parallel formulation (KernelKind::Parallel): the
 * adjoint of the per-degree scan passes, the reference's vjp_parallel
 * (src/autodiff.cpp:108-214), run as GPU suffix scans and per-position
 * contractions over (B, L-1, D) workspaces; memory_cap as for
 * sigk_signature_parallel_*. Same buffers and flags as sigk_signature_vjp_*. */
int sigk_signature_vjp_parallel_f32(const float* X, size_t B, size_t L, int d, int N, const float* cotangent, float* grad,
                                    size_t memory_cap, unsigned flags, void* stream, sigk_stats* stats);
int sigk_signature_vjp_parallel_f64(const double* X, size_t B, size_t L, int d, int N, const double* cotangent,
                                    double* grad, size_t memory_cap, unsigned flags, void* stream, sigk_stats* stats);

/* Host buffers in and out; rows [g*ceil(B/G), ...) run on device g, one host
 * thread per device, each shard copied in, folded and copied back into its
 * disjoint slice of `out`. num_gpus <= 0 means all visible devices. */
int sigk_signature_sharded_f32(const float* X, size_t B, size_t L, int d, int N, float* out, int num_gpus,
                               sigk_stats* stats);
int sigk_signature_sharded_f64(const double* X, size_t B, size_t L, int d, int N, double* out, int num_gpus,
                               sigk_stats* stats);

/* Synthetic benchmark input on the device: Brownian paths,
 * X[b,0,:] = 0, increments N(0, 1/(L-1)) from Philox4x32-10 keyed by
 * (seed, row0 + b, t, c) — identical rows for any sharding. */
int sigk_brownian_f32(float* X_dev, size_t B, size_t L, int d, uint64_t seed, size_t row0, void* stream);
int sigk_brownian_f64(double* X_dev, size_t B, size_t L, int d, uint64_t seed, size_t row0, void* stream);

/* The reference's benchmark inputs (bench.cpp:134-161): (B, L, d) float64
 * random walks from (seed, B, L, d), bit-identical to make_bench_paths. */
int sigk_make_bench_paths(uint64_t seed, size_t B, size_t L, int d, double* out);

/* Brute-force signature of ONE host path (len points, dim channels) by
 * direct enumeration of segment-index tuples (reference
 * signature_bruteforce, oracle.hpp:23-31, oracle.cpp:28-96; strict = 1 for
 * TupleClass::StrictlyIncreasing). One GPU thread per coefficient, the
 * reference's enumeration order and products: fp64 bit-identical. Limits as
 * the reference's OracleLimits: SIGK_ERESOURCE beyond them. Synchronous. */
int sigk_signature_bruteforce_f64(const double* path, size_t len, int dim, int depth, int max_segments,
                                  int max_depth, int max_dim, int strict, double* out);

/* Increments X[:, k+1] - X[:, k] into out (B, L-1, d) (reference
 * increments, kernels.cpp:71-87), and increments divided by m! for m =
 * 2..depth into out (depth-1, n) (reference scaled_increments,
 * kernels.cpp:89-104). Elementwise GPU kernels, fp64 bit-identical to the
 * reference. Flags and stream as for sigk_signature_*; host buffers make the
 * call synchronous. L = 1 / depth = 1 write nothing. */
int sigk_increments_f32(const float* X, size_t B, size_t L, int d, float* out, unsigned flags, void* stream);
int sigk_increments_f64(const double* X, size_t B, size_t L, int d, double* out, unsigned flags, void* stream);
int sigk_scaled_increments_f32(const float* inc, size_t n, int depth, float* out, unsigned flags, void* stream);
int sigk_scaled_increments_f64(const double* inc, size_t n, int depth, double* out, unsigned flags, void* stream);

/* The reference's training harness (model.cpp:222-263; paper §3.2) with the
 * signature forward and VJP on the GPU: writes `epochs` mean losses. kernel:
 * 0 sequential, 1 parallel, 2 auto; activation: 0 tanh, 1 identity. Returns
 * SIGK_EDOMAIN on bad config, SIGK_ETRAINING when the loss goes non-finite,
 * SIGK_EDEVICE on any other failure. */
int sigk_train(size_t n_samples, size_t seq_len, int sig_input_size, int depth, size_t batch_size, int epochs,
               double learning_rate, uint64_t seed, int kernel, int activation, double* epoch_losses);

/* 1 when a register-sliced fast variant exists for (d, N) in this precision
 * (0: the shape-generic kernel is used). *Q receives the prefix length. */
int sigk_has_fast_variant(int d, int N, int is_f64, int* Q);

/* The launch plan sigk_signature_* would use for this shape on the current
 * device (no kernel runs): family, Q, chunks, segments, fold_steps. */
int sigk_plan(size_t B, size_t L, int d, int N, int is_f64, const sigk_tuning* tuning, sigk_stats* plan);

/* FP32 FFMA-pipe peak microbenchmark (roofline denominator): launches
 * `blocks` x 256 threads, each running iters*128 independent-chain FFMAs;
 * *flops = 2 x FFMAs. Time it with events on `stream`. */
int sigk_bench_ffma(float* sink, int blocks, int iters, double* flops, void* stream);

/* Thread-local message of the last failing call on this thread ("" if none). */
const char* sigk_last_error(void);

/* ABI version: major*10000 + minor*100 + patch. */
int sigk_version(void);

#ifdef __cplusplus
}
#endif
#endif /* SIGK_H */
