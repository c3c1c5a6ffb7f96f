// Increments and factorial-scaled increments (reference kernels.cpp:71-104):
// elementwise, HBM-bound utilities of the drop-in API (the signature kernels
// recompute δ inline and never read these). Same IEEE operations as the
// reference (one subtraction; division by the running double factorial), so
// fp64 results are bit-identical.
#pragma once
#include <cstdint>

namespace sigk {

// out (B, L-1, d): out[b, k, c] = X[b, k+1, c] - X[b, k, c]
template <typename Real>
__global__ void increments_kernel(const Real* __restrict__ X, int64_t B, int64_t L, int d, Real* __restrict__ out) {
    const int64_t row = (L - 1) * d;  // output elements per path
    const int64_t n = B * row;
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
        const int64_t b = i / row, r = i - b * row;
        const Real* src = X + b * L * d + r;
        out[i] = src[d] - src[0];
    }
}

// out (depth-1, n): out[m-2, i] = inc[i] / m!, m = 2..depth
template <typename Real>
__global__ void scaled_increments_kernel(const Real* __restrict__ inc, int64_t n, int depth, Real* __restrict__ out) {
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
        const Real v = inc[i];
        double f = 1.0;  // the reference accumulates the factorial in double
        for (int m = 2; m <= depth; ++m) {
            f *= m;
            out[(int64_t)(m - 2) * n + i] = v / (Real)f;
        }
    }
}

}  // namespace sigk
