// Cross-chunk combine: Chen's identity as a fixed-order tree.
//
// (A ⊠ B)_n = A_n + B_n + Σ_{i=1}^{n-1} A_i ⊗ B_{n-i}
// (reference chen_product, /root/reference/proj/src/tensor_algebra.cpp:80-102,
// same term order: c_n = a_n + b_n, then += a_i ⊗ b_{n-i} for i = 1..n-1).
//
// Per path, the K chunk signatures (rows b*K .. b*K+K-1 of the scratch) are
// combined pairwise in rounds r = 1, 2, 4, ...: slot j ← slot j ⊠ slot j+r for
// j ≡ 0 (mod 2r). The order is fixed, so the result is deterministic and does
// not depend on the launch shape. Each product is written in place over its
// left operand, one level at a time in DESCENDING order with a CTA barrier
// between levels: level n only reads levels < n of A, which are still intact.
// Every output element is independent within a level: thread per element,
// prefix index I / d^(n-i) into A_i and suffix index I mod d^(n-i) into B_{n-i}.
#pragma once

#include "sigk_common.cuh"

namespace sigk {

template <typename Real, int DIM, int DEPTH>
__device__ __forceinline__ Real chen_elem(const Real* __restrict__ A, const Real* __restrict__ Bm, int n, int I) {
    Real acc = A[level_off(DIM, n - 1) + I] + Bm[level_off(DIM, n - 1) + I];
#pragma unroll
    for (int i = 1; i < DEPTH; ++i) {
        if (i < n) {
            int tail = 1;
#pragma unroll
            for (int q = 0; q < DEPTH; ++q)
                if (q < n - i) tail *= DIM;
            acc = fma(A[level_off(DIM, i - 1) + I / tail], Bm[level_off(DIM, n - i - 1) + I % tail], acc);
        }
    }
    return acc;
}

// One CTA per path. ws: (B*K, D) chunk signatures; the result goes to out (B, D).
template <typename Real, int DIM, int DEPTH>
__global__ void __launch_bounds__(512) merge_tree_kernel(Real* __restrict__ ws, int K, Real* __restrict__ out) {
    constexpr int D = level_off(DIM, DEPTH);
    const int64_t b = blockIdx.x;
    Real* base = ws + b * (int64_t)K * D;
    for (int r = 1; r < K; r <<= 1) {
        const int pairs = (K - r + 2 * r - 1) / (2 * r);  // j = 0, 2r, 4r, ... with j + r < K
        const bool last = (2 * r >= K);
#pragma unroll 1
        for (int n = DEPTH; n >= 1; --n) {
            int lsz = 1;
            for (int q = 0; q < n; ++q) lsz *= DIM;
            const int work = pairs * lsz;
            for (int w = threadIdx.x; w < work; w += blockDim.x) {
                const int pj = w / lsz;
                const int I = w - pj * lsz;
                Real* A = base + (int64_t)(2 * r * pj) * D;
                const Real* Bm = A + (int64_t)r * D;
                const Real v = chen_elem<Real, DIM, DEPTH>(A, Bm, n, I);
                if (last) {
                    out[b * D + level_off(DIM, n - 1) + I] = v;
                } else {
                    A[level_off(DIM, n - 1) + I] = v;
                }
            }
            __syncthreads();
        }
    }
}

}  // namespace sigk
