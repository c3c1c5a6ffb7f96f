// The paper's parallel formulation (arXiv 2501.08455 §2.2) on the GPU: the
// reference's detail::parallel_forward<Real>
// (/root/reference/proj/include/sigkit/detail/sig_core.hpp:175-298), which
// KernelKind::Parallel selects (kernels.cpp:124-148, 150-154, 185-197).
//
// For each degree n = 1..N, one pass (one launch):
//   contribution  c_k[I] = (δ_k^{⊗n}/n!)[I] + Σ_{j=1}^{n-1} T_{n-j}[k-1][I / d^j] · (δ_k^{⊗j}/j!)[I % d^j]
//                 (the k = 0 term has no lower-degree prefix, sig_core.hpp:275-285)
//   level         T_n[k] = Σ_{k' <= k} c_{k'}   (inclusive cumulative sum along the sequence)
// Every per-position level is materialised in the (B, M, D) workspace W (the
// reference's ParallelState levels, in the row layout of the prefix-signature
// output, so W IS the signature_stream output when the caller asks for it).
// The cumulative sum is a two-phase parallel scan per CTA: 32 lanes = 32
// consecutive multi-indices I of one path, NW warps = NW contiguous ranges of
// k; phase 1 sums each warp's contributions, a fixed-order exclusive scan of
// the NW partial sums in shared memory gives each range its carry, phase 2
// recomputes the contributions and writes the running sums. Memory-bound by
// construction (the formulation materialises B·M·D scalars, which is why the
// reference caps it, sig_core.hpp:161-173); the fold kernels are the fast path.
#pragma once

#include <cstdint>

#include "sigk_common.cuh"

namespace sigk {

constexpr int kScanMaxDepth = 64;

template <typename Real>
struct ScanGeom {
    int64_t off[kScanMaxDepth + 1];    // level n starts at off[n-1] inside a D-row
    int64_t pw[kScanMaxDepth + 1];     // d^j
    Real inv_fact[kScanMaxDepth + 1];  // 1/j! (Real(1)/factorial, factorial accumulated in Real, :218-227)
};

// contribution c_k[I] of degree n at position k. rdig[j-1] = the j-th index
// of I counted from the last one, (I / d^(j-1)) % d; hi[j] = I / d^j. The diagonal terms are
// suffix products of δ over the trailing digits, scaled by 1/j!.
template <typename Real, int MAXN>
__device__ __forceinline__ Real scan_contrib(const Real* __restrict__ xk, const Real* __restrict__ prev, int d,
                                             int n, const ScanGeom<Real>& g, const int (&rdig)[MAXN + 1],
                                             const int64_t (&hi)[MAXN + 1]) {
    Real v = 0, sp = 1;
#pragma unroll
    for (int j = 1; j <= MAXN; ++j) {
        if (j <= n) {
            const int c = rdig[j - 1];
            sp *= xk[d + c] - xk[c];  // δ_k[c] (sig_core.hpp:208-216)
            if (j < n) {
                if (prev != nullptr) v = fma(prev[g.off[n - j - 1] + hi[j]], sp * g.inv_fact[j], v);
            } else {
                v += sp * g.inv_fact[n];
            }
        }
    }
    return v;
}

// One degree pass. grid.x = B * ceil(d^n / 32); block = 32 * NW. MAXN >= n.
template <typename Real, int NW, int MAXN>
__global__ void __launch_bounds__(32 * NW) degree_scan_kernel(const Real* __restrict__ X, int64_t L, int d, int n,
                                                              int64_t M, Real* __restrict__ W, int64_t D,
                                                              ScanGeom<Real> g) {
    __shared__ Real part[NW][32];
    const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
    const int64_t tiles = (g.pw[n] + 31) / 32;
    const int64_t b = blockIdx.x / tiles, tile = blockIdx.x - b * tiles;
    const int64_t I = tile * 32 + lane;
    const bool live = I < g.pw[n];
    const Real* xb = X + b * L * d;
    Real* wb = W + b * M * D;
    int rdig[MAXN + 1];
    int64_t hi[MAXN + 1];
#pragma unroll
    for (int r = 0; r <= MAXN; ++r) {
        rdig[r] = r < n ? (int)((I / g.pw[r]) % d) : 0;
        hi[r] = r < n ? I / g.pw[r] : 0;
    }
    const int64_t per = (M + NW - 1) / NW;
    const int64_t k0 = w * per < M ? w * per : M, k1 = k0 + per < M ? k0 + per : M;
    Real s = 0;
    if (live)
        for (int64_t k = k0; k < k1; ++k)
            s += scan_contrib<Real, MAXN>(xb + k * d, k > 0 ? wb + (k - 1) * D : nullptr, d, n, g, rdig, hi);
    part[w][lane] = s;
    __syncthreads();
    Real acc = 0;
    for (int v = 0; v < w; ++v) acc += part[v][lane];  // fixed-order carry into this range
    if (!live) return;
    Real* col = wb + g.off[n - 1] + I;
    for (int64_t k = k0; k < k1; ++k) {
        acc += scan_contrib<Real, MAXN>(xb + k * d, k > 0 ? wb + (k - 1) * D : nullptr, d, n, g, rdig, hi);
        col[k * D] = acc;
    }
}

}  // namespace sigk
