// Reverse mode of the paper's parallel formulation on the GPU: the
// reference's vjp_parallel (/root/reference/proj/src/autodiff.cpp:108-214),
// which signature_vjp selects for KernelKind::Parallel (:218-224). It is the
// adjoint of the per-degree scan passes of scan_kernel.cuh, not of the fold:
// a second, independent GPU route to the same gradient (the reference's two
// adjoints agree, test_autodiff.cpp:117-130).
//
// Workspaces, all in the (B, M, D) row layout of the prefix signatures:
//   W   forward levels T_n[k] (scan_kernel.cuh, the prefix rows),
//   Tb  level cotangents tbar_n[k], seeded with the output cotangent at k = M-1,
//   Db  cotangents of the diagonal terms diag_j[k] = δ_k^{⊗j}/j!.
// Degrees n = N..1, each:
//   degree_suffix_kernel      tbar_n <- inclusive suffix sum along k (the
//                             adjoint of the forward cumulative sum), and
//                             diagbar_n += tbar_n;
//   degree_distribute_kernel  every position k >= 1 hands tbar_n[k] to the
//                             factors of its cross terms (j = 1..n-1, m = n-j):
//                               tbar_m[k-1][I]  += Σ_J tbar_n[k][I·d^j + J] diag_j[k][J]
//                               diagbar_j[k][J] += Σ_I tbar_n[k][I·d^j + J] T_m[k-1][I]
//                             (contract_right / contract_left, sig_core.hpp:49-70).
// Then diag_chain_kernel runs diag_n = diag_{n-1} ⊗ δ / n backwards per
// position (n = N..2) into δ̄ rows, and vjp_grad_kernel turns them into
// ∂/∂X_t = δ̄_{t-1} - δ̄_t. Memory-bound and capped like the forward
// formulation (3 B·M·D scalars); the fold adjoint (vjp_slice.cuh) is the fast path.
#pragma once

#include <cstdint>

#include "scan_kernel.cuh"

namespace sigk {

// δ_k^{⊗j}/j! at multi-index J (digits of J, last one fastest), on the fly
// from the step's two points x0 = X[k], x1 = X[k+1] (32-bit digit arithmetic:
// every multi-index here is below the storage cap, 2^31).
template <typename Real>
__device__ __forceinline__ Real diag_entry(const Real* __restrict__ x0, const Real* __restrict__ x1, unsigned d, int j,
                                           unsigned J, Real inv_fact_j) {
    Real v = inv_fact_j;
    for (int r = 0; r < j; ++r) {
        const unsigned q = J / d, c = J - q * d;
        v *= x1[c] - x0[c];
        J = q;
    }
    return v;
}

// In-place inclusive suffix sum of level n of Tb along k, then Db level n += it.
// grid.x = B * ceil(d^n / 32); block = 32 * NW (NW contiguous ranges of k).
template <typename Real, int NW>
__global__ void __launch_bounds__(32 * NW) degree_suffix_kernel(int n, int64_t M, Real* __restrict__ Tb,
                                                                Real* __restrict__ Db, int64_t D, ScanGeom<Real> g) {
    __shared__ Real part[NW][32];
    const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
    const int64_t tiles = (g.pw[n] + 31) / 32;
    const int64_t b = blockIdx.x / tiles, tile = blockIdx.x - b * tiles;
    const int64_t I = tile * 32 + lane;
    const bool live = I < g.pw[n];
    const int64_t per = (M + NW - 1) / NW;
    const int64_t k0 = w * per < M ? w * per : M, k1 = k0 + per < M ? k0 + per : M;
    Real* col = Tb + b * M * D + g.off[n - 1] + I;
    Real* dcol = Db + b * M * D + g.off[n - 1] + I;
    Real s = 0;
    if (live)
        for (int64_t k = k0; k < k1; ++k) s += col[k * D];
    part[w][lane] = s;
    __syncthreads();
    Real acc = 0;
    for (int v = NW - 1; v > w; --v) acc += part[v][lane];  // fixed-order carry from the later ranges
    if (!live) return;
    for (int64_t k = k1 - 1; k >= k0; --k) {
        acc += col[k * D];
        col[k * D] = acc;
        dcol[k * D] += acc;
    }
}

// Cross-term distribution of degree n (n >= 2). One thread per (position
// k >= 1, output entry) of path blockIdx.y: entries [0, DLn) of a position are
// tbar_m[k-1] (levels m = 1..n-1 in row order), [DLn, 2 DLn) the diagbar_j[k]
// entries (levels j = 1..n-1).
template <typename Real>
__global__ void __launch_bounds__(256) degree_distribute_kernel(const Real* __restrict__ X, int64_t L, int d, int n,
                                                                int64_t M, const Real* __restrict__ W,
                                                                Real* __restrict__ Tb, Real* __restrict__ Db, int64_t D,
                                                                ScanGeom<Real> g) {
    const int64_t DLn = g.off[n - 1];  // entries of levels 1..n-1
    const int64_t per_pos = 2 * DLn;
    const int64_t total = (int64_t)(M - 1) * per_pos;  // positions k = 1..M-1 of one path
    const int64_t b = blockIdx.y;
    const Real* xb = X + b * L * d;
    Real* tb = Tb + b * M * D;
    Real* db = Db + b * M * D;
    const Real* wb = W + b * M * D;
    for (int64_t w = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; w < total; w += (int64_t)gridDim.x * blockDim.x) {
        const int64_t k = 1 + w / per_pos;
        int64_t e = w - (k - 1) * per_pos;
        const bool right = e < DLn;  // tbar_m[k-1] (else diagbar_j[k])
        if (!right) e -= DLn;
        int lev = 1;
        while (e >= g.off[lev]) ++lev;  // level of the output entry
        const unsigned idx = (unsigned)(e - g.off[lev - 1]);
        const Real* x0 = xb + k * d;
        const Real* x1 = x0 + d;
        const Real* u = tb + k * D + g.off[n - 1];  // tbar_n[k]
        Real acc = 0;
        if (right) {  // m = lev, j = n - m: Σ_J u[I·d^j + J] diag_j[J]
            const int j = n - lev;
            const unsigned pj = (unsigned)g.pw[j];
            const Real* row = u + (int64_t)idx * pj;
            for (unsigned J = 0; J < pj; ++J) acc += row[J] * diag_entry(x0, x1, (unsigned)d, j, J, g.inv_fact[j]);
            tb[(k - 1) * D + g.off[lev - 1] + idx] += acc;
        } else {  // j = lev, m = n - j: Σ_I u[I·d^j + J] T_m[k-1][I]
            const int j = lev, m = n - lev;
            const Real* tm = wb + (k - 1) * D + g.off[m - 1];
            const unsigned pm = (unsigned)g.pw[m], pj = (unsigned)g.pw[j];
            for (unsigned I = 0; I < pm; ++I) acc += u[(int64_t)I * pj + idx] * tm[I];
            db[k * D + g.off[j - 1] + idx] += acc;
        }
    }
}

// diag_n = diag_{n-1} ⊗ δ / n reversed per position, n = N..2 (in place on the
// Db row, autodiff.cpp:179-197), then δ̄ = diagbar_1 + the chain's δ terms ->
// dbar (B, M, d). One warp per position, lanes over the prefixes I:
//   dbp[I] += (1/n) Σ_c dbn[I·d + c] δ[c]
//   δ̄[c]  += (1/n) Σ_I dbn[I·d + c] diag_{n-1}[I]   (per-lane partials, 8 channels
//                                                    at a time, then a warp sum)
template <typename Real>
__global__ void __launch_bounds__(128) diag_chain_kernel(const Real* __restrict__ X, int64_t L, int d, int N, int64_t M,
                                                         int64_t B, Real* __restrict__ Db, int64_t D,
                                                         Real* __restrict__ dbar, ScanGeom<Real> g) {
    const int lane = threadIdx.x & 31;
    const int64_t gw = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    const int64_t nw = ((int64_t)gridDim.x * blockDim.x) >> 5;
    for (int64_t pos = gw; pos < B * M; pos += nw) {
        const int64_t b = pos / M, k = pos - (pos / M) * M;
        const Real* x0 = X + (b * L + k) * d;
        const Real* x1 = x0 + d;
        Real* row = Db + pos * D;
        Real* out = dbar + pos * d;
        for (int c = lane; c < d; c += 32) out[c] = 0;
        __syncwarp();
        for (int n = N; n >= 2; --n) {
            const Real inv = Real(1) / Real(n);
            const Real* dbn = row + g.off[n - 1];
            Real* dbp = row + g.off[n - 2];
            const unsigned pp = (unsigned)g.pw[n - 1];
            // δ̄ terms (read dbn only; dbp is level n-1, updated below)
            for (int c0 = 0; c0 < d; c0 += 8) {
                Real part[8];
#pragma unroll
                for (int q = 0; q < 8; ++q) part[q] = 0;
                for (unsigned I = lane; I < pp; I += 32) {
                    const Real dv = diag_entry(x0, x1, (unsigned)d, n - 1, I, g.inv_fact[n - 1]);
#pragma unroll
                    for (int q = 0; q < 8; ++q)
                        if (c0 + q < d) part[q] += dbn[(int64_t)I * d + c0 + q] * dv;
                }
#pragma unroll
                for (int q = 0; q < 8; ++q) {
                    Real v = part[q];
                    for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
                    if (lane == 0 && c0 + q < d) out[c0 + q] += inv * v;
                }
            }
            for (unsigned I = lane; I < pp; I += 32) {
                Real a = 0;
                for (int c = 0; c < d; ++c) a += dbn[(int64_t)I * d + c] * (x1[c] - x0[c]);
                dbp[I] += inv * a;
            }
            __syncwarp();
        }
        // + diagbar_1 after the chain (the n = 2 step updated it; level 1 = the increments)
        for (int c = lane; c < d; c += 32) out[c] += row[c];
        __syncwarp();
    }
}

}  // namespace sigk
