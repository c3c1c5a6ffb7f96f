// Host-side view of the variant table (no CUDA templates needed to include).
#pragma once

#include <cstddef>
#include <cstdint>
#include <cuda_runtime.h>

namespace sigk {

enum class KernelFamily : int { Path = 0, Flat = 1 };

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
};

const Variant* find_variant(int d, int N, bool is_f64);  // first (smallest-Q) candidate
int find_variants(int d, int N, bool is_f64, const Variant** out, int max);
cudaError_t launch_generic_f32(const void* X, int64_t B, int64_t L, int d, int N, void* out, cudaStream_t s);
cudaError_t launch_generic_f64(const void* X, int64_t B, int64_t L, int d, int N, void* out, cudaStream_t s);
cudaError_t launch_brownian_f32(void* X, int64_t B, int64_t L, int d, uint64_t seed, int64_t row0, cudaStream_t s);
cudaError_t launch_brownian_f64(void* X, int64_t B, int64_t L, int d, uint64_t seed, int64_t row0, cudaStream_t s);

}  // namespace sigk
