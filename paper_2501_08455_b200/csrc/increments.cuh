// Increments and factorial-scaled increments (reference kernels.cpp:71-104):
// elementwise, HBM-bound utilities of the drop-in API (the signature kernels
// recompute δ inline and never read these). Same IEEE operations as the
// reference (one subtraction; division by the running double factorial), so
// fp64 results are bit-identical.
#pragma once
#include <cstdint>
#include <type_traits>

namespace sigk {

// out (B, L-1, d): out[b, k, c] = X[b, k+1, c] - X[b, k, c]. Path b's
// output is its input shifted by d elements, so each path is a contiguous
// run: vector loads of 16 bytes (float4 / double2) when the run and both
// pointers are 16-byte aligned, scalar otherwise (the two loads of an
// element hit the same or neighbouring sectors; L2 absorbs the overlap).
template <typename Real>
__global__ void increments_kernel(const Real* __restrict__ X, int64_t B, int64_t L, int d, Real* __restrict__ out) {
    const int64_t row = (L - 1) * d;  // output elements per path
    const int64_t n = B * row;
    constexpr int V = 16 / sizeof(Real);
    using Vec = typename std::conditional<sizeof(Real) == 4, float4, double2>::type;
    const bool vec = (row % V == 0) && (d % V == 0) && ((reinterpret_cast<uintptr_t>(X) | reinterpret_cast<uintptr_t>(out)) % 16 == 0);
    const int64_t stride = (int64_t)gridDim.x * blockDim.x;
    if (vec) {
        const int64_t nv = n / V, rowv = row / V, dv = d / V;
        const Vec* Xv = reinterpret_cast<const Vec*>(X);
        Vec* ov = reinterpret_cast<Vec*>(out);
        for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < nv; i += stride) {
            const int64_t b = i / rowv, r = i - b * rowv;
            const Vec* src = Xv + b * (rowv + dv) + r;  // path b starts at b*L*d = b*(row + d)
            const Vec lo = src[0], hi = src[dv];
            Vec o;
            if constexpr (sizeof(Real) == 4) o = make_float4(hi.x - lo.x, hi.y - lo.y, hi.z - lo.z, hi.w - lo.w);
            else o = make_double2(hi.x - lo.x, hi.y - lo.y);
            ov[i] = o;
        }
        return;
    }
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += stride) {
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
