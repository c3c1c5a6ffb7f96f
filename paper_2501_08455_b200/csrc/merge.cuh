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
// every output element is independent, so all threads of the CTA share the
// work of every pair of the round (prefix index I / d^(n-i) into A_i, suffix
// index I mod d^(n-i) into B_{n-i}; divisors are compile-time).
#pragma once

#include "sigk_common.cuh"

namespace sigk {

template <typename Real, int d, int n, int i>
__device__ __forceinline__ void chen_terms(const Real* __restrict__ A, const Real* __restrict__ Bm, int I, Real& acc) {
    if constexpr (i < n) {
        constexpr int tail = ipow(d, n - i);
        acc = fma(A[level_off(d, i - 1) + I / tail], Bm[level_off(d, n - i - 1) + I % tail], acc);
        chen_terms<Real, d, n, i + 1>(A, Bm, I, acc);
    }
}

template <typename Real, int d, int N, int n>
__device__ __forceinline__ void merge_level_desc(Real* __restrict__ sig, int D, int h, int pairs) {
    if constexpr (n >= 1) {
        constexpr int lsz = ipow(d, n);
        constexpr int o = level_off(d, n - 1);
        const int work = pairs * lsz;
        for (int w = threadIdx.x; w < work; w += blockDim.x) {
            const int pj = w / lsz;
            const int I = w - pj * lsz;
            Real* A = sig + (2 * h * pj) * D;
            const Real* Bm = A + h * D;
            Real acc = A[o + I] + Bm[o + I];
            chen_terms<Real, d, n, 1>(A, Bm, I, acc);
            A[o + I] = acc;
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
