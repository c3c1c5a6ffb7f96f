// Compile-time variant table: one register-sliced fold (+ its Chen merge) per
// (precision, d, N), with the prefix length Q picked so the per-thread slice
// fits the register budget.
#pragma once

#include <cuda_runtime.h>

#include <atomic>
#include <cstdint>

#include "fold.cuh"
#include "generic.cuh"
#include "merge.cuh"
#include "variants.h"

namespace sigk {

// Smallest Q whose per-thread state (in 32-bit registers) fits the budget.
template <typename Real>
constexpr int pick_q(int d, int N) {
    constexpr int budget = 160;  // 32-bit registers of state per thread
    for (int q = 0; q < N; ++q) {
        int s = q > 1 ? q - 1 : 0;
        for (int n = (q > 1 ? q : 1); n <= N; ++n) s += ipow(d, n - q);
        if (s * (int)(sizeof(Real) / 4) <= budget) return q;
    }
    return N - 1;
}

template <typename Real, int DIM, int DEPTH>
struct VariantImpl {
    static constexpr int Q = pick_q<Real>(DIM, DEPTH);
    using SF = SliceFold<Real, DIM, DEPTH, Q>;
    static constexpr int NT = 128;
    static constexpr int T = fold_tile_steps(NT, SF::P, DIM);
    static constexpr size_t smem = fold_smem_bytes<Real, DIM, DEPTH, Q, NT, T>();

    // Opt in to >48 KB dynamic shared memory once per device (not stream-ordered,
    // so it must not be repeated inside a graph capture).
    static cudaError_t prepare() {
        static std::atomic<uint64_t> done{0};
        int dev = 0;
        cudaGetDevice(&dev);
        const uint64_t bit = 1ull << (dev & 63);
        if (smem <= 48 * 1024 || (done.load() & bit)) return cudaSuccess;
        cudaError_t e = cudaFuncSetAttribute(fold_kernel<Real, DIM, DEPTH, Q, NT, T>,
                                             cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
        if (e == cudaSuccess) done.fetch_or(bit);
        return e;
    }
    static cudaError_t fold(const void* X, int64_t B, int64_t L, int K, int CL, void* dst, cudaStream_t s) {
        cudaError_t e = prepare();
        if (e != cudaSuccess) return e;
        const int64_t lanes = B * (int64_t)K * SF::P;
        const int64_t grid = (lanes + NT - 1) / NT;
        fold_kernel<Real, DIM, DEPTH, Q, NT, T><<<(unsigned)grid, NT, smem, s>>>(
            static_cast<const Real*>(X), B, L, K, CL, static_cast<Real*>(dst));
        return cudaGetLastError();
    }
    static cudaError_t merge(void* ws, int K, void* out, int64_t B, cudaStream_t s) {
        merge_tree_kernel<Real, DIM, DEPTH><<<(unsigned)B, 512, 0, s>>>(static_cast<Real*>(ws), K, static_cast<Real*>(out));
        return cudaGetLastError();
    }
    static cudaError_t occupancy(int* blocks) {
        cudaError_t e = prepare();
        if (e != cudaSuccess) return e;
        return cudaOccupancyMaxActiveBlocksPerMultiprocessor(blocks, fold_kernel<Real, DIM, DEPTH, Q, NT, T>, NT, smem);
    }
    static constexpr Variant make() {
        int chen = 0;
        for (int n = 2; n <= DEPTH; ++n) chen += (n - 1) * ipow(DIM, n);
        return Variant{DIM, DEPTH, Q, NT, T, SF::P, SF::ops_per_step(), chen, smem, &fold, &merge, &occupancy};
    }
};

// Registry filled by the per-(precision, d) translation units at load time.
void register_variants(const Variant* table, int n, bool is_f64);

template <typename Real, int DIM, int... Ns>
struct DimTable {
    static constexpr Variant table[] = {VariantImpl<Real, DIM, Ns>::make()...};
    static constexpr int count = sizeof...(Ns);
};

}  // namespace sigk

// (d, N) pairs with a register-sliced instantiation (anything else runs the
// shape-generic kernel). Each (precision, d) row is compiled as its own
// translation unit (variants_inst.cu) so the build parallelises.
#define SIGK_DEPTHS_1 1, 2, 3, 4, 5, 6
#define SIGK_DEPTHS_2 1, 2, 3, 4, 5, 6
#define SIGK_DEPTHS_3 1, 2, 3, 4, 5
#define SIGK_DEPTHS_4 1, 2, 3, 4, 5
#define SIGK_DEPTHS_5 1, 2, 3, 4, 5
#define SIGK_DEPTHS_6 1, 2, 3, 4
#define SIGK_DEPTHS_7 1, 2, 3, 4
#define SIGK_DEPTHS_8 1, 2, 3, 4
#define SIGK_DEPTHS_10 1, 2, 3, 4, 5
#define SIGK_FAST_DIMS 1, 2, 3, 4, 5, 6, 7, 8, 10
