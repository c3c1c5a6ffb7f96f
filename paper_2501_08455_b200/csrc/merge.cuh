// Cross-chunk combine: the paper's per-degree cumulative-sum formulation
// (arXiv 2501.08455 §2.2; reference parallel_forward, sig_core.hpp:175-298)
// applied at CHUNK granularity, with Chen's identity (tensor_algebra.cpp:80-102)
// giving each chunk's contribution.
//
// Let C^(j) be the local signature of chunk j (folded from the identity) and
// P^(j) = C^(0) ⊠ ... ⊠ C^(j-1) the exclusive prefix (P^(0) = 1). Then
//     (P^(j) ⊠ C^(j))_n = P^(j)_n + c^(j)_n,
//     c^(j)_n = C^(j)_n + Σ_{a=1}^{n-1} P^(j)_a ⊗ C^(j)_{n-a},
// so P^(j)_n = Σ_{i<j} c^(i)_n is an exclusive prefix SUM over chunks of
// contributions that need only the prefixes of LOWER degrees. Degree by
// degree (n = 1..N-1): all chunks' contributions in parallel, then a plain
// exclusive scan over chunks; the path's degree-n value is the scan total.
// Degree N needs no scan, only the total Σ_j c^(j)_N — its cross terms are
// formed in registers by the threads that already hold C^(j)_N's slices, and
// the U contributions are summed in a fixed order (deterministic).
//
// Versus a log2(U)-round tree of full Chen products this has N phases, no
// full products, and the dominant degree-N work runs FFMA-dense from
// registers.
#pragma once

#include "fold.cuh"

namespace sigk {

// Degree n (< N), fused: one thread per element I walks the chunks in order,
// forming each chunk's contribution c_n[I] (from the already-scanned lower
// prefixes) and writing the running exclusive sum into pf; the total (the
// path's degree-n coefficient) goes to out. The walk is batched 8 chunks at a
// time so the shared-memory loads of a batch are in flight together.
template <typename Real, int d, int N, int n>
__device__ __forceinline__ void scan_lower_levels(const Real* __restrict__ cl, Real* __restrict__ pf, int U,
                                                  Real* __restrict__ out) {
    if constexpr (n < N) {
        constexpr int DL = level_off(d, N - 1);
        constexpr int lsz = ipow(d, n);
        constexpr int o = level_off(d, n - 1);
        for (int I = threadIdx.x; I < lsz; I += blockDim.x) {
            // per-element offsets of the cross terms P_a[I / d^(n-a)] * C_{n-a}[I mod d^(n-a)]
            int po[n > 1 ? n - 1 : 1], co[n > 1 ? n - 1 : 1];
#pragma unroll
            for (int a = 1; a < n; ++a) {
                const int tail = ipow(d, n - a);
                po[a - 1] = level_off(d, a - 1) + I / tail;
                co[a - 1] = level_off(d, n - a - 1) + I % tail;
            }
            Real acc = Real(0);
            const Real* cu = cl;
            Real* pu = pf;
            auto contrib = [&](const Real* c, const Real* p) {
                Real x = c[o + I];
#pragma unroll
                for (int a = 1; a < n; ++a) x = fma(p[po[a - 1]], c[co[a - 1]], x);
                return x;
            };
            int u = 0;
            for (; u + 8 <= U; u += 8, cu += 8 * DL, pu += 8 * DL) {  // 8 chunks of loads in flight
                Real c[8];
#pragma unroll
                for (int k = 0; k < 8; ++k) c[k] = contrib(cu + k * DL, pu + k * DL);
#pragma unroll
                for (int k = 0; k < 8; ++k) {
                    pu[k * DL + o + I] = acc;
                    acc += c[k];
                }
            }
            for (; u < U; ++u, cu += DL, pu += DL) {
                const Real x = contrib(cu, pu);
                pu[o + I] = acc;
                acc += x;
            }
            out[o + I] = acc;
        }
        __syncthreads();
        scan_lower_levels<Real, d, N, n + 1>(cl, pf, U, out);
    }
}

// Degree-N contribution of this thread's slice: st's top block plus
// Σ_a P_a[(pre,J)[:a]] · C_{N-a}[(pre,J)[a:]] with P from pf and C's lower
// degrees from cl (this chunk's rows). Accumulated into red (d^{N-Q} values).
template <typename SF, int a, typename Real>
__device__ __forceinline__ void top_cross_terms(const Real* __restrict__ p, const Real* __restrict__ c, int pre,
                                                Real (&acc)[ipow(SF::d, SF::N - SF::QQ)]) {
    constexpr int d = SF::d, N = SF::N, Q = SF::QQ;
    if constexpr (a < N) {
        constexpr int FJ = ipow(d, N - Q);  // outputs per thread
        constexpr int tail = ipow(d, N - a);
        const Real* pa = p + level_off(d, a - 1);
        const Real* cb = c + level_off(d, N - a - 1);
        if constexpr (a <= Q) {  // prefix scalar P_a[p_1..p_a]; suffix row C_{N-a}[(p_{a+1}..p_Q), J]
            const Real pv = pa[pre / ipow(d, Q - a)];
            const Real* cr = cb + (pre % ipow(d, Q - a)) * FJ;
#pragma unroll
            for (int J = 0; J < FJ; ++J) acc[J] = fma(pv, cr[J], acc[J]);
        } else {  // prefix P_a[pre, J[:a-Q]] (slice of P), suffix C_{N-a}[J[a-Q:]]
            const Real* pr = pa + pre * ipow(d, a - Q);
#pragma unroll
            for (int J = 0; J < FJ; ++J) acc[J] = fma(pr[J / tail], cb[J % tail], acc[J]);
        }
        top_cross_terms<SF, a + 1>(p, c, pre, acc);
    }
}

// Per-thread stride of the degree-N contribution rows, padded when it is a
// multiple of the 32 banks so the row stores do not conflict.
template <typename SF>
__host__ __device__ constexpr int red_stride() {
    constexpr int FJ = ipow(SF::d, SF::N - SF::QQ);
    return FJ % 32 == 0 ? FJ + 1 : FJ;
}

template <typename SF>
__host__ __device__ constexpr size_t combine_smem_elems(int U) {
    return (size_t)U * (2 * level_off(SF::d, SF::N - 1) + SF::P * red_stride<SF>());
}

// Combine the U chunk signatures held in registers by the CTA (thread (u, pre)
// holds st = slice pre of chunk u) into the path's signature row `out`.
// smem: at least U*(2*level_off(d,N-1) + d^N) Reals. Call from all threads.
template <typename SF, typename Real, typename Phase>
__device__ __forceinline__ void combine_chunks(Real (&st)[SF::S], int u, int pre, int U, Real* __restrict__ smem,
                                               Real* __restrict__ out, Phase&& phase) {
    constexpr int d = SF::d, N = SF::N, Q = SF::QQ;
    constexpr int DL = level_off(d, N - 1);
    constexpr int FJ = ipow(d, N - Q);
    constexpr int FP = red_stride<SF>();  // padded per-thread stride: no bank conflicts
    constexpr int o = level_off(d, N - 1);
    Real* cl = smem;               // [U][DL] chunk signatures, degrees < N
    Real* pf = cl + U * DL;        // [U][DL] exclusive prefixes
    Real* red = pf + U * DL;       // [U][P][FP] degree-N contributions
    if (U == 1) {  // a single chunk: its signature is the path's
        store_levels_below<SF, 1>(st, pre, cl);
        Real* r = red + pre * FP;
#pragma unroll
        for (int J = 0; J < FJ; ++J) r[J] = st[SF::top_off(N) + J];
        __syncthreads();
        for (int i = threadIdx.x; i < DL; i += blockDim.x) out[i] = cl[i];
        for (int F = threadIdx.x; F < ipow(d, N); F += blockDim.x) out[o + F] = red[(F / FJ) * FP + F % FJ];
        return;
    }
    store_levels_below<SF, 1>(st, pre, cl + u * DL);
    __syncthreads();
    phase(4);
    scan_lower_levels<Real, d, N, 1>(cl, pf, U, out);
    phase(5);
    Real acc[FJ];
#pragma unroll
    for (int J = 0; J < FJ; ++J) acc[J] = st[SF::top_off(N) + J];
    top_cross_terms<SF, 1>(pf + u * DL, cl + u * DL, pre, acc);
    Real* r = red + (u * SF::P + pre) * FP;
#pragma unroll
    for (int J = 0; J < FJ; ++J) r[J] = acc[J];
    __syncthreads();
    phase(6);
    constexpr int LN = ipow(d, N);
    // fixed summation order over chunks; 2 elements x 8 chunks of loads in flight
    for (int F0 = threadIdx.x; F0 < LN; F0 += 2 * blockDim.x) {
        const int F1 = F0 + blockDim.x < LN ? F0 + blockDim.x : F0;
        const Real* q0 = red + (F0 / FJ) * FP + F0 % FJ;
        const Real* q1 = red + (F1 / FJ) * FP + F1 % FJ;
        constexpr int RS = SF::P * FP;  // stride between chunks
        Real s0 = Real(0), s1 = Real(0);
        int v = 0;
        for (; v + 8 <= U; v += 8, q0 += 8 * RS, q1 += 8 * RS) {
            Real t0[8], t1[8];
#pragma unroll
            for (int k = 0; k < 8; ++k) {
                t0[k] = q0[k * RS];
                t1[k] = q1[k * RS];
            }
#pragma unroll
            for (int k = 0; k < 8; ++k) {
                s0 += t0[k];
                s1 += t1[k];
            }
        }
        for (; v < U; ++v, q0 += RS, q1 += RS) {
            s0 += *q0;
            s1 += *q1;
        }
        out[o + F0] = s0;
        if (F0 + blockDim.x < LN) out[o + F1] = s1;
    }
}

}  // namespace sigk
