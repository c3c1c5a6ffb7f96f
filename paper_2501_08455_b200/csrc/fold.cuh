// Prefix-sliced, chunked Horner fold of Chen's recurrence on sm_100a.
//
// What it computes (reference: detail::sequential_forward<Real>,
// /root/reference/proj/include/sigkit/detail/sig_core.hpp:116-147, with
// exp_into :72-90 and fold_step :92-114): for every path b,
//     S(b) = exp(dX_0) ⊠ exp(dX_1) ⊠ ... ⊠ exp(dX_{M-1}),  M = L-1,
// truncated at depth N, flattened to levels 1..N (layout sig_core.hpp:7-10).
//
// How:
//  * One step S ← S ⊠ exp(δ) is evaluated in Horner form, level by level in
//    DESCENDING order so lower levels are still the previous state:
//        u_1 = δ/n + T_1,  u_k = u_{k-1} ⊗ δ/(n-k+1) + T_k,  T_n += u_{n-1} ⊗ δ.
//    Every element of every stage is exactly one FFMA, W(d,N) per step.
//  * Leading-index closure: after a step, T_n[p_1..p_Q, ...] depends only on
//    entries with the same prefix (and on δ). A thread therefore owns one
//    prefix P = (p_1..p_Q) — the whole slice T_n[P, *] for n >= Q plus the Q-1
//    redundant scalars T_m[p_1..p_m], m < Q — entirely in registers, and
//    never talks to another thread during the fold.
//  * A "unit" is (path b, chunk k): the chunk's local signature over steps
//    [k*CL, (k+1)*CL). Chunks past the end are padded with δ = 0, which is
//    an exact identity step (fma(u, 0, T) == T). Chunk signatures are
//    combined afterwards with Chen's identity (merge.cuh).
//  * Increments are produced cooperatively per tile of T steps: each thread
//    loads X[t], X[t+1] for a few (unit, step, channel) entries (coalesced,
//    prefetched into registers one tile ahead), forms δ and its scaled
//    copies δ/m, and stores them to a double-buffered shared-memory table;
//    consumers read them back with 16-byte broadcast loads.
#pragma once

#include "sigk_common.cuh"

namespace sigk {

// Units (path, chunk) that one CTA of NT threads can touch: NT/P whole units
// plus one straddling each CTA boundary.
__host__ __device__ constexpr int fold_units_per_cta(int NT, int P) {
    return P >= NT ? 2 : (NT % P == 0 ? NT / P + 1 : NT / P + 2);
}

// Steps per shared-memory tile: up to 8, fewer when a CTA holds many units so
// the per-thread register prefetch (2 values per entry) stays <= 16 registers.
__host__ __device__ constexpr int fold_tile_steps(int NT, int P, int d) {
    int t = 8;
    while (t > 1 && fold_units_per_cta(NT, P) * t * d > 8 * NT) --t;
    return t;
}

template <typename Real, int DIM, int DEPTH, int Q>
struct SliceFold {
    static constexpr int d = DIM;
    static constexpr int N = DEPTH;
    static constexpr int P = ipow(d, Q);             // slices (threads) per unit
    static constexpr int NLOW = Q > 1 ? Q - 1 : 0;   // redundant scalars T_1..T_{Q-1}
    static constexpr int NMIN = Q > 1 ? Q : 1;       // first level stored as a slice
    __host__ __device__ static constexpr int top_off(int n) {  // register offset of slice level n
        int o = NLOW;
        for (int m = NMIN; m < n; ++m) o += ipow(d, m - Q);
        return o;
    }
    static constexpr int S = top_off(N + 1);         // registers of state per thread
    static constexpr int NV = N - Q;                 // vector rows δ/m, m = 1..NV
    static constexpr int VW = Vec16<Real>::n;
    static constexpr int VEC = round_up(NV * d, VW); // table: vector part
    static constexpr int SCW = Q > 0 ? round_up(N, VW) : 0;
    static constexpr int TAB = VEC + (Q > 0 ? d * SCW : 0);  // table row per (unit, step)
    static constexpr int QS = Q > 0 ? Q : 1;
    static constexpr int QQ = Q;
    // FFMA-pipe ops per thread per step (the Horner count restricted to a slice,
    // including the redundant prefix chains).
    __host__ __device__ static constexpr int ops_per_step() {
        int ops = 0;
        for (int n = 1; n <= N; ++n) {
            if (n > Q) {
                ops += Q;  // scalar chain stages (stage 1 is an add)
                for (int k = Q + 1; k <= n; ++k) ops += ipow(d, k - Q);
            } else {
                ops += n;
            }
        }
        return ops;
    }

    __device__ __forceinline__ static Real& scal(Real (&st)[S], int k) {
        // T_k[p_1..p_k] for k <= Q
        return k < Q ? st[k - 1] : st[top_off(Q)];
    }

    // Level n of one Horner step. vs[(m-1)*d + c] = δ[c]/m ; sc[k-1][m-1] = δ[p_k]/m.
    template <int n>
    __device__ __forceinline__ static void level(Real (&st)[S], const Real (&vs)[VEC],
                                                 const Real (&sc)[QS][SCW > 0 ? SCW : 1]) {
        if constexpr (n > Q) {
            constexpr int F = n - Q;  // free (per-thread) indices of level n
            Real u0 = Real(0);
            if constexpr (Q >= 1) {
                u0 = sc[0][n - 1] + scal(st, 1);
#pragma unroll
                for (int k = 2; k <= Q; ++k) u0 = fma(u0, sc[k - 1][n - k], scal(st, k));
            }
            if constexpr (F == 1) {
                constexpr int o = top_off(n);
                if constexpr (Q == 0) {  // n == 1: T_1 += δ
#pragma unroll
                    for (int c = 0; c < d; ++c) st[o + c] += vs[c];
                } else {
#pragma unroll
                    for (int c = 0; c < d; ++c) st[o + c] = fma(u0, vs[c], st[o + c]);
                }
            } else {
                Real ua[ipow(d, F - 1)];
                {   // stage k = Q+1 uses δ/(n-Q)
                    constexpr int o = top_off(Q + 1);
                    constexpr int r = (n - Q - 1) * d;
                    if constexpr (Q == 0) {
#pragma unroll
                        for (int c = 0; c < d; ++c) ua[c] = vs[r + c] + st[o + c];
                    } else {
#pragma unroll
                        for (int c = 0; c < d; ++c) ua[c] = fma(u0, vs[r + c], st[o + c]);
                    }
                }
                stages<n, Q + 2>(st, vs, ua);
                constexpr int o = top_off(n);
#pragma unroll
                for (int J = 0; J < ipow(d, F); ++J) st[o + J] = fma(ua[J / d], vs[J % d], st[o + J]);
            }
        } else {  // scalar level n <= Q
            if constexpr (n == 1) {
                scal(st, 1) += sc[0][0];
            } else {
                Real u = sc[0][n - 1] + scal(st, 1);
#pragma unroll
                for (int k = 2; k <= n - 1; ++k) u = fma(u, sc[k - 1][n - k], scal(st, k));
                scal(st, n) = fma(u, sc[n - 1][0], scal(st, n));
            }
        }
    }

    // Vector stages k = K0 .. n-1 (in place, expanding ua by a factor d each).
    template <int n, int k, int UA>
    __device__ __forceinline__ static void stages(Real (&st)[S], const Real (&vs)[VEC], Real (&ua)[UA]) {
        if constexpr (k <= n - 1) {
            constexpr int sz = ipow(d, k - Q);
            constexpr int o = top_off(k);
            constexpr int r = (n - k) * d;  // row m = n-k+1
#pragma unroll
            for (int J = sz - 1; J >= 0; --J) ua[J] = fma(ua[J / d], vs[r + J % d], st[o + J]);
            stages<n, k + 1>(st, vs, ua);
        }
    }

    template <int n>
    __device__ __forceinline__ static void levels_desc(Real (&st)[S], const Real (&vs)[VEC],
                                                       const Real (&sc)[QS][SCW > 0 ? SCW : 1]) {
        if constexpr (n >= 1) {
            level<n>(st, vs, sc);
            levels_desc<n - 1>(st, vs, sc);
        }
    }

    __device__ __forceinline__ static void step(Real (&st)[S], const Real (&vs)[VEC],
                                                const Real (&sc)[QS][SCW > 0 ? SCW : 1]) {
        levels_desc<N>(st, vs, sc);
    }
};

// Register state of one thread -> its slice of a flat (D) signature row.
template <typename SF, int n, typename Real>
__device__ __forceinline__ void store_levels(Real (&st)[SF::S], int pre, Real* __restrict__ row) {
    constexpr int d = SF::d, Q = SF::QQ;
    if constexpr (n <= SF::N) {
        if constexpr (n >= SF::NMIN) {
            constexpr int sz = ipow(d, n - Q);
            constexpr int o = SF::top_off(n);
            Real* dst = row + level_off(d, n - 1) + (int64_t)pre * sz;
#pragma unroll
            for (int J = 0; J < sz; ++J) dst[J] = st[o + J];
        } else {  // redundant prefix scalar T_n[p_1..p_n], n < Q: one writer each
            constexpr int tail = ipow(d, Q - n);
            if (pre % tail == 0) row[level_off(d, n - 1) + pre / tail] = st[n - 1];
        }
        store_levels<SF, n + 1>(st, pre, row);
    }
}

template <typename SF, typename Real>
__device__ __forceinline__ void store_slice(Real (&st)[SF::S], int pre, Real* __restrict__ row) {
    store_levels<SF, 1>(st, pre, row);
}

// X: (B, L, d) row-major. dst: (B*K, D) rows, row = b*K + k.
template <typename Real, int DIM, int DEPTH, int Q, int NT, int T>
__global__ void __launch_bounds__(NT) fold_kernel(const Real* __restrict__ X, int64_t B, int64_t L, int K,
                                                  int CL, Real* __restrict__ dst) {
    using SF = SliceFold<Real, DIM, DEPTH, Q>;
    constexpr int d = DIM;
    constexpr int P = SF::P;
    constexpr int TAB = SF::TAB;
    constexpr int VEC = SF::VEC;
    constexpr int SCW = SF::SCW;
    constexpr int VW = SF::VW;
    constexpr int NU = fold_units_per_cta(NT, P);  // max units one CTA touches
    constexpr int ENT = NU * T * d;                // producer entries per tile
    constexpr int EPT = (ENT + NT - 1) / NT;
    constexpr int D = level_off(d, DEPTH);
    using V = typename Vec16<Real>::type;

    extern __shared__ __align__(16) unsigned char smem_raw[];
    Real* tab = reinterpret_cast<Real*>(smem_raw);  // [2][T][NU][TAB]

    const int64_t M = L - 1;
    const int64_t units = B * (int64_t)K;
    const int64_t g0 = (int64_t)blockIdx.x * NT;
    const int64_t u0 = g0 / P;
    const int64_t g = g0 + threadIdx.x;
    const int64_t unit = g / P;
    const int pre = (int)(g % P);
    const bool active = unit < units;
    const int uu = (int)(unit - u0);

    int dig[SF::QS];
#pragma unroll
    for (int k = 0; k < SF::QS; ++k) dig[k] = (Q > 0) ? (pre / ipow(d, Q - 1 - k)) % d : 0;

    Real st[SF::S];
#pragma unroll
    for (int i = 0; i < SF::S; ++i) st[i] = Real(0);

    Real xa[EPT], xb[EPT];
    auto load = [&](int tile) {
#pragma unroll
        for (int i = 0; i < EPT; ++i) {
            const int e = threadIdx.x + i * NT;
            xa[i] = Real(0);
            xb[i] = Real(0);
            if (e < ENT) {
                const int c = e % d;
                const int s = (e / d) % T;
                const int ue = e / (d * T);
                const int64_t un = u0 + ue;
                const int j = tile * T + s;
                if (un < units && j < CL) {
                    const int64_t b = un / K;
                    const int64_t t = (un % K) * (int64_t)CL + j;
                    if (t < M) {
                        const Real* p = X + (b * L + t) * d + c;
                        xa[i] = __ldg(p);
                        xb[i] = __ldg(p + d);
                    }
                }
            }
        }
    };
    auto store = [&](int buf) {
#pragma unroll
        for (int i = 0; i < EPT; ++i) {
            const int e = threadIdx.x + i * NT;
            if (e < ENT) {
                const int c = e % d;
                const int s = (e / d) % T;
                const int ue = e / (d * T);
                Real* row = tab + (((size_t)buf * T + s) * NU + ue) * TAB;
                const Real dl = xb[i] - xa[i];
#pragma unroll
                for (int m = 1; m <= SF::NV; ++m) row[(m - 1) * d + c] = dl * (Real(1) / Real(m));
                if constexpr (Q > 0) {
#pragma unroll
                    for (int m = 1; m <= DEPTH; ++m) row[VEC + c * SCW + (m - 1)] = dl * (Real(1) / Real(m));
                }
            }
        }
    };

    const int ntiles = (CL + T - 1) / T;
    load(0);
    for (int tile = 0; tile < ntiles; ++tile) {
        const int buf = tile & 1;
        store(buf);
        __syncthreads();
        if (tile + 1 < ntiles) load(tile + 1);
        if (active) {
#pragma unroll 1
            for (int s = 0; s < T; ++s) {
                const Real* row = tab + (((size_t)buf * T + s) * NU + uu) * TAB;
                Real vs[VEC];
#pragma unroll
                for (int i = 0; i < VEC / VW; ++i) {
                    const V v = reinterpret_cast<const V*>(row)[i];
                    if constexpr (VW == 4) {
                        vs[4 * i] = v.x; vs[4 * i + 1] = v.y; vs[4 * i + 2] = v.z; vs[4 * i + 3] = v.w;
                    } else {
                        vs[2 * i] = v.x; vs[2 * i + 1] = v.y;
                    }
                }
                Real sc[SF::QS][SCW > 0 ? SCW : 1];
                if constexpr (Q > 0) {
#pragma unroll
                    for (int k = 0; k < Q; ++k) {
                        const Real* sr = row + VEC + dig[k] * SCW;
#pragma unroll
                        for (int i = 0; i < SCW / VW; ++i) {
                            const V v = reinterpret_cast<const V*>(sr)[i];
                            if constexpr (VW == 4) {
                                sc[k][4 * i] = v.x; sc[k][4 * i + 1] = v.y; sc[k][4 * i + 2] = v.z; sc[k][4 * i + 3] = v.w;
                            } else {
                                sc[k][2 * i] = v.x; sc[k][2 * i + 1] = v.y;
                            }
                        }
                    }
                } else {
                    sc[0][0] = Real(0);
                }
                SF::step(st, vs, sc);
            }
        }
    }
    if (active) store_slice<SF>(st, pre, dst + unit * (int64_t)D);
}

template <typename Real, int DIM, int DEPTH, int Q, int NT, int T>
constexpr size_t fold_smem_bytes() {
    using SF = SliceFold<Real, DIM, DEPTH, Q>;
    constexpr int NU = fold_units_per_cta(NT, SF::P);
    return sizeof(Real) * 2ull * T * NU * SF::TAB;
}

}  // namespace sigk
