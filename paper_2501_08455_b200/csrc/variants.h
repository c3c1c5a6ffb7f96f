// Host-side view of the variant table (no CUDA templates needed to include).
#pragma once

#include <cstddef>
#include <cstdint>
#include <cuda_runtime.h>

namespace sigk {

enum class KernelFamily : int { Path = 1, Flat = 2, Pair = 3, PFlat = 5 };  // = SIGK_FAMILY_*

// Pair family: in latency plans, segment counts 2..kMaxPairCluster run as
// thread-block clusters (one cluster per path, segment rows combined over
// distributed shared memory); otherwise (throughput plans, where clusters'
// gang scheduling measured 7% slower back to back at C3, or G >
// kMaxPairCluster) the rows combine through global scratch and arrival counters.
// Both combines run the same arithmetic in the same order.
constexpr int kMaxPairCluster = 8;

// One launch of the pair family (pair_kernel.cuh): B*G CTAs of one path
// segment each (SL steps as U chunks of CL). When G > 1 and `cluster`, the G
// CTAs of a path form a cluster and combine their rows over distributed shared
// memory; otherwise the segment rows go to `scratch` ((B*G, D) floats) and the
// last segment CTA of each path (per the zero-initialised `counters`, [B]
// ints) combines them into `out`.
struct PairLaunch {
    const void* X;
    int64_t B, L;
    int G;
    int64_t SL;
    int U, CL;
    void* out;
    void* scratch;
    void* counters;
    cudaStream_t s;
    bool overlap;
    void* ev_fold_start;  // optional events recorded around the fold kernel
    void* ev_fold_stop;
    bool capturing;
    void* phases;  // optional [B*G][8] int64 phase stamps
    bool cluster;  // G in [2, kMaxPairCluster]: cluster launch (no scratch, no counters)
    bool pos;      // position-table fold with a producer warp (ppair_kernel.cuh); U/2 * P <= 128
    // chunk paths (reverse mode): when sub_U > 0, path r of the launch (B = B0 * sub_U rows) is
    // chunk r % sub_U of path r / sub_U of X ((B0, sub_L, d)): points j*sub_CL .. min((j+1)*sub_CL,
    // sub_L - 1); L is then sub_CL + 1 (the gather kernel's layout, without the gather)
    int64_t sub_U = 0, sub_CL = 0, sub_L = 0;
};

struct Variant {
    int d, N;
    int Q;       // prefix length owned per thread
    int P;       // threads per (path, chunk) unit = d^Q
    int ops;     // FFMA-pipe ops per thread per step
    int loads;   // 16-byte shared-memory loads per thread per step
    int chen;    // FMAs of one Chen product (merge), Σ_{n>=2} (n-1) d^n
    KernelFamily family;
    int nt;      // path: max threads per CTA; flat: threads per CTA
    int T;       // steps per shared-memory tile
    // path: grid = B CTAs of U*P threads (U chunks per path); flat: U ignored
    cudaError_t (*launch)(const void* X, int64_t B, int64_t L, int U, void* out, cudaStream_t s, void* phases,
                          bool overlap_previous);
    // resident CTAs per SM for a given U (0 when it does not fit)
    cudaError_t (*occupancy)(int U, int* blocks_per_sm);
    // pair family only
    cudaError_t (*pair_launch)(const PairLaunch& a);
    cudaError_t (*pair_occupancy)(int U, int CL, int64_t SL, int G, bool cluster, int* blocks_per_sm);  // 0: does not fit
    int pair_units_max;  // max U/2 per CTA
    // pair family: prefix stream (B, L-1, D); G segments per path, CTA (b, g) starting from the row its
    // predecessor segment publishes in the same launch (pub/flags/epoch); cudaErrorInvalidValue when a
    // segment does not fit one CTA
    cudaError_t (*stream_launch)(const void* X, int64_t B, int64_t L, int U, void* out, cudaStream_t s, bool overlap,
                                 int G, void* pub, int* flags, int epoch);
    int pos_ops;          // pair family: FFMA-pipe ops per thread-step of the position-table fold (0: none)
    int pos_units_max;    // max U/2 of a position-table CTA
    cudaError_t (*pair_pos_occupancy)(int U, int CL, int64_t SL, int G, bool cluster, int* blocks_per_sm);
    // pair family: stage tile (steps) of the prefix-stream launch for (L, G, U); 0: does not fit
    int (*stream_tile_steps)(int64_t L, int G, int U);
    // pair family, reverse mode (vjp_prep.cuh): one CTA per path folds its U chunks (CL steps
    // each, R real) and runs both chunk passes in shared memory -> ends / cbars rows (B, R, D)
    // and zeros at the shared chunk points of grad; null where the shape has no slice walk
    cudaError_t (*vjp_prep_launch)(const void* X, int64_t B, int64_t L, int U, int CL, int R, const void* cot,
                                   void* ends, void* cbars, void* grad, cudaStream_t s);
    size_t (*vjp_prep_smem)(int U, int CL, int64_t L);  // bytes of one CTA
};

const Variant* find_variant(int d, int N, bool is_f64);  // first (smallest-Q) candidate
int find_variants(int d, int N, bool is_f64, const Variant** out, int max);
cudaError_t launch_generic_f32(const void* X, int64_t B, int64_t L, int d, int N, void* out, cudaStream_t s);
cudaError_t launch_generic_f64(const void* X, int64_t B, int64_t L, int d, int N, void* out, cudaStream_t s);
// chunk-parallel generic stream: U chunks of CL steps per path, chunk u > 0 starting from
// row b*U + u of `starts` (null when U == 1)
cudaError_t launch_generic_stream_f32(const void* X, int64_t B, int64_t L, int d, int N, void* out, cudaStream_t s,
                                      int U, int64_t CL, const void* starts);
cudaError_t launch_generic_stream_f64(const void* X, int64_t B, int64_t L, int d, int N, void* out, cudaStream_t s,
                                      int U, int64_t CL, const void* starts);
cudaError_t launch_brownian_f32(void* X, int64_t B, int64_t L, int d, uint64_t seed, int64_t row0, cudaStream_t s);
cudaError_t launch_brownian_f64(void* X, int64_t B, int64_t L, int d, uint64_t seed, int64_t row0, cudaStream_t s);

}  // namespace sigk
