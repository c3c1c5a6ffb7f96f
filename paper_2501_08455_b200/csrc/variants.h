// Host-side view of the variant table (no CUDA templates needed to include).
#pragma once

#include <cstddef>
#include <cstdint>
#include <cuda_runtime.h>

namespace sigk {

struct Variant {
    int d, N;
    int Q;      // prefix length owned per thread
    int NT;     // threads per CTA
    int T;      // steps per shared-memory tile
    int P;      // threads per (path, chunk) unit = d^Q
    int ops;    // FFMA-pipe ops per thread per step
    int chen;   // FMAs of one Chen product (merge), Σ_{n>=2} (n-1) d^n
    size_t smem;
    cudaError_t (*fold)(const void* X, int64_t B, int64_t L, int K, int CL, void* dst, cudaStream_t s);
    cudaError_t (*merge)(void* ws, int K, void* out, int64_t B, cudaStream_t s);
    cudaError_t (*occupancy)(int* blocks_per_sm);
};

const Variant* find_variant_f32(int d, int N);
const Variant* find_variant_f64(int d, int N);
cudaError_t launch_generic_f32(const void* X, int64_t B, int64_t L, int d, int N, void* out, cudaStream_t s);
cudaError_t launch_generic_f64(const void* X, int64_t B, int64_t L, int d, int N, void* out, cudaStream_t s);
cudaError_t launch_brownian_f32(void* X, int64_t B, int64_t L, int d, uint64_t seed, int64_t row0, cudaStream_t s);
cudaError_t launch_brownian_f64(void* X, int64_t B, int64_t L, int d, uint64_t seed, int64_t row0, cudaStream_t s);

}  // namespace sigk
