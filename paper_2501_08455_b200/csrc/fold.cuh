// Prefix-sliced Horner fold of Chen's recurrence: the per-thread math shared
// by the sm_100a fold kernels (path_kernel.cuh, flat_kernel.cuh).
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
//    [k*CL, (k+1)*CL). Steps past the end are padded with δ = 0, which is an
//    exact identity step (fma(u, 0, T) == T). Chunk signatures are combined
//    with Chen's identity (merge.cuh).
//  * Increments are produced cooperatively per tile of steps into a
//    shared-memory table (produce_entry): the vector δ/m rows every thread of
//    the unit reads with 16-byte broadcast loads, plus per-channel scalar
//    rows δ[c]/m for the prefix digits (consume_step).
#pragma once

#include "sigk_common.cuh"

namespace sigk {

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
    // Operand modes. Table mode (Q <= 1): the table row holds every scaled
    // vector δ/m (m = 1..N-Q) plus per-channel scalar rows δ[c]/m, so a step
    // is pure FFMA. Lean mode (Q >= 2, where a thread's step is short and the
    // shared-memory wavefronts per FFMA would bind): the row holds δ only; the
    // thread reads δ[p_k] for its prefix digits and folds the 1/m factors into
    // its (short) running products with a few FMULs.
    static constexpr bool LEAN = Q >= 2;
    static constexpr int NV = LEAN ? 1 : N - Q;      // vector rows δ/m, m = 1..NV
    static constexpr int VW = Vec16<Real>::n;
    static constexpr int VEC = round_up(NV * d, VW); // table: vector part
    static constexpr int SCW = (Q > 0 && !LEAN) ? round_up(N, VW) : 0;
    static constexpr int TAB = VEC + d * SCW;        // table row per (unit, step)
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

    // Level n of one Horner step. Table mode: vs[(m-1)*d + c] = δ[c]/m,
    // sc[k-1][m-1] = δ[p_k]/m. Lean mode: vs[c] = δ[c], sc[k-1][0] = δ[p_k].
    template <int n>
    __device__ __forceinline__ static void level(Real (&st)[S], const Real (&vs)[VEC],
                                                 const Real (&sc)[QS][SCW > 0 ? SCW : 1]) {
        if constexpr (LEAN) {
            level_lean<n>(st, vs, sc);
        } else if constexpr (n > Q) {
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

    // Lean-mode level n (Q >= 2): identical Horner chain, with δ/m formed as
    // (running product * 1/m) * δ so only δ itself is read from the table.
    template <int n>
    __device__ __forceinline__ static void level_lean(Real (&st)[S], const Real (&dv)[VEC],
                                                      const Real (&dp)[QS][SCW > 0 ? SCW : 1]) {
        constexpr Real inv_n = Real(1) / Real(n);
        if constexpr (n > Q) {
            constexpr int F = n - Q;
            Real u0 = fma(dp[0][0], inv_n, scal(st, 1));  // δ[p1]/n + T_1[p1]
#pragma unroll
            for (int k = 2; k <= Q; ++k) u0 = fma(u0 * (Real(1) / Real(n - k + 1)), dp[k - 1][0], scal(st, k));
            if constexpr (F == 1) {
                constexpr int o = top_off(n);
#pragma unroll
                for (int c = 0; c < d; ++c) st[o + c] = fma(u0, dv[c], st[o + c]);
            } else {
                Real ua[ipow(d, F - 1)];
                {   // stage k = Q+1, factor 1/(n-Q)
                    constexpr int o = top_off(Q + 1);
                    const Real us = u0 * (Real(1) / Real(n - Q));
#pragma unroll
                    for (int c = 0; c < d; ++c) ua[c] = fma(us, dv[c], st[o + c]);
                }
                stages_lean<n, Q + 2>(st, dv, ua);
                constexpr int o = top_off(n);
#pragma unroll
                for (int J = 0; J < ipow(d, F); ++J) st[o + J] = fma(ua[J / d], dv[J % d], st[o + J]);
            }
        } else {  // scalar level n <= Q
            if constexpr (n == 1) {
                scal(st, 1) += dp[0][0];
            } else {
                Real u = fma(dp[0][0], inv_n, scal(st, 1));
#pragma unroll
                for (int k = 2; k <= n - 1; ++k) u = fma(u * (Real(1) / Real(n - k + 1)), dp[k - 1][0], scal(st, k));
                scal(st, n) = fma(u, dp[n - 1][0], scal(st, n));
            }
        }
    }

    template <int n, int k, int UA>
    __device__ __forceinline__ static void stages_lean(Real (&st)[S], const Real (&dv)[VEC], Real (&ua)[UA]) {
        if constexpr (k <= n - 1) {
            constexpr int sz = ipow(d, k - Q);
            constexpr int o = top_off(k);
            constexpr Real inv = Real(1) / Real(n - k + 1);
#pragma unroll
            for (int J = 0; J < sz / d; ++J) ua[J] *= inv;  // prescale the previous stage
#pragma unroll
            for (int J = sz - 1; J >= 0; --J) ua[J] = fma(ua[J / d], dv[J % d], st[o + J]);
            stages_lean<n, k + 1>(st, dv, ua);
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

// Register state of one thread -> its slice of degrees n..NMAX of a flat
// signature row (degree m at offset level_off(d, m-1)).
template <typename SF, int n, int NMAX, typename Real>
__device__ __forceinline__ void store_levels(Real (&st)[SF::S], int pre, Real* __restrict__ row) {
    constexpr int d = SF::d, Q = SF::QQ;
    if constexpr (n <= NMAX) {
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
        store_levels<SF, n + 1, NMAX>(st, pre, row);
    }
}

template <typename SF, typename Real>
__device__ __forceinline__ void store_slice(Real (&st)[SF::S], int pre, Real* __restrict__ row) {
    store_levels<SF, 1, SF::N>(st, pre, row);
}

// Degrees 1..N-1 only (the inputs of the chunk combine, merge.cuh).
template <typename SF, int n, typename Real>
__device__ __forceinline__ void store_levels_below(Real (&st)[SF::S], int pre, Real* __restrict__ row) {
    store_levels<SF, n, SF::N - 1>(st, pre, row);
}

// The operands of one Horner step, in registers: the δ/m vectors and the
// thread's prefix scalars δ[p_k]/m.
template <typename SF, typename Real>
struct StepRegs {
    Real vs[SF::VEC];
    Real sc[SF::QS][SF::SCW > 0 ? SF::SCW : 1];
};

// Load a step's table row from shared memory with 16-byte broadcast loads.
template <typename SF, typename Real>
__device__ __forceinline__ void load_row(StepRegs<SF, Real>& r, const Real* __restrict__ row, const int (&dig)[SF::QS]) {
    using V = typename Vec16<Real>::type;
    constexpr int VW = SF::VW, VEC = SF::VEC, SCW = SF::SCW;
#pragma unroll
    for (int i = 0; i < VEC / VW; ++i) {
        const V v = reinterpret_cast<const V*>(row)[i];
        if constexpr (VW == 4) {
            r.vs[4 * i] = v.x; r.vs[4 * i + 1] = v.y; r.vs[4 * i + 2] = v.z; r.vs[4 * i + 3] = v.w;
        } else {
            r.vs[2 * i] = v.x; r.vs[2 * i + 1] = v.y;
        }
    }
    if constexpr (SF::LEAN) {  // δ[p_k]: one scalar load per prefix digit
#pragma unroll
        for (int k = 0; k < SF::QQ; ++k) r.sc[k][0] = row[dig[k]];
    } else if constexpr (SF::QQ > 0) {
#pragma unroll
        for (int k = 0; k < SF::QQ; ++k) {
            const Real* sr = row + VEC + dig[k] * SCW;
#pragma unroll
            for (int i = 0; i < SCW / VW; ++i) {
                const V v = reinterpret_cast<const V*>(sr)[i];
                if constexpr (VW == 4) {
                    r.sc[k][4 * i] = v.x; r.sc[k][4 * i + 1] = v.y; r.sc[k][4 * i + 2] = v.z; r.sc[k][4 * i + 3] = v.w;
                } else {
                    r.sc[k][2 * i] = v.x; r.sc[k][2 * i + 1] = v.y;
                }
            }
        }
    } else {
        r.sc[0][0] = Real(0);
    }
}

// The T steps of one tile (rows base, base + stride, ...), software-pipelined:
// the row of step s+1 is in flight while the FFMAs of step s issue, so the
// shared-memory latency never sits on the Horner chain.
// (PIPE = false: plain loop, for register-tight variants that hide the
// latency with more resident warps instead.)
template <typename SF, int T, bool PIPE = true, typename Real>
__device__ __forceinline__ void consume_tile(Real (&st)[SF::S], const Real* __restrict__ base, size_t stride,
                                             const int (&dig)[SF::QS]) {
    if constexpr (!PIPE) {
#pragma unroll 1
        for (int s = 0; s < T; ++s) {
            StepRegs<SF, Real> r;
            load_row<SF>(r, base + (size_t)s * stride, dig);
            SF::step(st, r.vs, r.sc);
        }
        return;
    }
    StepRegs<SF, Real> ra, rb;
    load_row<SF>(ra, base, dig);
#pragma unroll 1
    for (int s = 0; s < T; s += 2) {
        if (s + 1 < T) load_row<SF>(rb, base + (size_t)(s + 1) * stride, dig);
        SF::step(st, ra.vs, ra.sc);
        if (s + 2 < T) load_row<SF>(ra, base + (size_t)(s + 2) * stride, dig);
        if (s + 1 < T) SF::step(st, rb.vs, rb.sc);
    }
}

// Write one increment δ (component c of step s) into a table row: the vector
// part δ/m (m = 1..N-Q) and, for sliced variants, the scalar row of c
// (δ/m, m = 1..N) that threads whose prefix digit is c load in one go.
template <typename SF, typename Real>
__device__ __forceinline__ void produce_entry(Real* __restrict__ row, int c, Real dl) {
#pragma unroll
    for (int m = 1; m <= SF::NV; ++m) row[(m - 1) * SF::d + c] = dl * (Real(1) / Real(m));
    if constexpr (SF::SCW > 0) {
#pragma unroll
        for (int m = 1; m <= SF::N; ++m) row[SF::VEC + c * SF::SCW + (m - 1)] = dl * (Real(1) / Real(m));
    }
}

template <typename SF>
__device__ __forceinline__ void prefix_digits(int pre, int (&dig)[SF::QS]) {
#pragma unroll
    for (int k = 0; k < SF::QS; ++k) dig[k] = (SF::QQ > 0) ? (pre / ipow(SF::d, SF::QQ - 1 - k)) % SF::d : 0;
}

}  // namespace sigk
