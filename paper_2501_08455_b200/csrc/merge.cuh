// Cross-chunk combine: Chen's identity as a fixed-order tree in shared memory.
//
// (A ⊠ B)_n = A_n + B_n + Σ_{i=1}^{n-1} A_i ⊗ B_{n-i}
// (reference chen_product, /root/reference/proj/src/tensor_algebra.cpp:80-102,
// same term order: c_n = a_n + b_n, then += a_i ⊗ b_{n-i} for i = 1..n-1).
//
// The U chunk signatures of one path sit in shared memory (sig[u][D]). They
// are combined pairwise in rounds h = 1, 2, 4, ...: slot j ← slot j ⊠ slot j+h
// for j ≡ 0 (mod 2h). The order is fixed, so the result is deterministic and
// independent of the launch shape. Each product overwrites its left operand
// one level at a time in DESCENDING order with a CTA barrier between levels:
// level n reads only levels < n of A, which are still intact. Inside a level
// the work is split into runs of d consecutive outputs I = R*d + c (last index
// varying): the whole run shares every prefix A_i[R / d^(n-i-1)] (one load
// each) and reads contiguous suffix runs B_{n-i}[(R mod d^(n-i-1))*d + c], so
// a run costs (n+1)d + n-1 loads for (n-1)d FMAs; all threads of the CTA share
// the runs of every pair of the round. Divisors are compile-time.
#pragma once

#include "sigk_common.cuh"

namespace sigk {

template <typename Real, int d, int n, int i>
__device__ __forceinline__ void chen_run_terms(const Real* __restrict__ A, const Real* __restrict__ Bm, int R,
                                               Real (&acc)[d]) {
    if constexpr (i < n) {
        constexpr int tail = ipow(d, n - i - 1);  // I / d^(n-i) = R / tail
        const Real a = A[level_off(d, i - 1) + R / tail];
        const Real* __restrict__ br = Bm + level_off(d, n - i - 1) + (R % tail) * d;
#pragma unroll
        for (int c = 0; c < d; ++c) acc[c] = fma(a, br[c], acc[c]);
        chen_run_terms<Real, d, n, i + 1>(A, Bm, R, acc);
    }
}

template <typename Real, int d, int N, int n>
__device__ __forceinline__ void merge_level_desc(Real* __restrict__ sig, int D, int h, int pairs) {
    if constexpr (n >= 1) {
        constexpr int runs = ipow(d, n - 1);
        constexpr int o = level_off(d, n - 1);
        const int work = pairs * runs;
        for (int w = threadIdx.x; w < work; w += blockDim.x) {
            const int pj = w / runs;
            const int R = w - pj * runs;
            Real* A = sig + (2 * h * pj) * D;
            const Real* Bm = A + h * D;
            Real acc[d];
#pragma unroll
            for (int c = 0; c < d; ++c) acc[c] = A[o + R * d + c] + Bm[o + R * d + c];
            chen_run_terms<Real, d, n, 1>(A, Bm, R, acc);
#pragma unroll
            for (int c = 0; c < d; ++c) A[o + R * d + c] = acc[c];
        }
        __syncthreads();
        merge_level_desc<Real, d, N, n - 1>(sig, D, h, pairs);
    }
}

// Tree-combine U signatures sig[0..U) (each D = level_off(d, N) values) into sig[0].
// Must be called by every thread of the CTA (contains barriers).
template <typename Real, int d, int N>
__device__ __forceinline__ void merge_tree_smem(Real* __restrict__ sig, int U) {
    constexpr int D = level_off(d, N);
    for (int h = 1; h < U; h <<= 1) {
        const int pairs = (U - h + 2 * h - 1) / (2 * h);  // j = 0, 2h, 4h, ... with j + h < U
        merge_level_desc<Real, d, N, N>(sig, D, h, pairs);
    }
}

}  // namespace sigk
