// Reverse mode, slice-parallel (the layout of the forward fold): one warp
// walks `SLOTS` (path, chunk) items backwards, lane (slot, p) owning the
// prefix slice p = (p_1..p_Q) of the cotangent C̄ and of the state A:
// levels n >= Q as the d^(n-Q) entries with that prefix, levels n < Q as the
// scalars at p_1..p_n. Per step (C = A ⊠ exp(δ)):
//   δ̄ by reverse-mode through the lane's own Horner chains (each output
//       element of C is owned by exactly one lane: slices by their lane,
//       low-level scalars by the lane whose trailing digits are zero), then
//       one segmented sum of d values over the slot's lanes;
//   Ā_m = Σ_j C̄_{m+j} · E_j by Horner over the trailing index inside the
//       slice (m >= Q), continued across lanes by segmented sums for m < Q.
// Exactly the mathematics of the element-parallel kernel (vjp_kernel.cuh)
// and of the reference's fold adjoint (autodiff.cpp:31-107), with every
// contraction along the trailing index in registers: d FMAs per output, no
// block barriers (only __syncwarp around the per-warp reduction scratch).
#pragma once

#include "vjp_kernel.cuh"

namespace sigk {

// Prefix length for the slice adjoint: the largest q < N with d^q <= 32 and
// at most 48 state values per lane; 0 when none (the element-parallel kernel).
__host__ __device__ constexpr int vjp_slice_q(int d, int N) {
    int best = 0;
    for (int q = 1; q < N; ++q) {
        if (ipow(d, q) > 32) break;
        int s = q - 1;
        for (int n = q; n <= N; ++n) s += ipow(d, n - q);
        if (s <= 48) best = q;
    }
    return best;
}

template <int d, int N, int Q>
struct SliceLayout {
    static constexpr int P = ipow(d, Q);
    static constexpr int SLOTS = 32 / P;
    static constexpr int NLOW = Q - 1;  // levels 1..Q-1 as scalars
    __host__ __device__ static constexpr int top_off(int n) {  // slice of level n >= Q
        int o = NLOW;
        for (int m = Q; m < n; ++m) o += ipow(d, m - Q);
        return o;
    }
    static constexpr int S = top_off(N + 1);
    // vector Horner stages k = Q+1..N-1 (sizes d^(k-Q)), flat
    __host__ __device__ static constexpr int vo(int k) {
        int o = 0;
        for (int m = Q + 1; m < k; ++m) o += ipow(d, m - Q);
        return o;
    }
    static constexpr int VS = vo(N) > 0 ? vo(N) : 1;
    static constexpr int GMAX = ipow(d, N - Q);
};

template <typename Real, int d, int N, int Q>
struct SliceRev {
    using LY = SliceLayout<d, N, Q>;
    static constexpr int S = LY::S, NLOW = LY::NLOW, VS = LY::VS;
    __device__ __forceinline__ static Real& sc(Real (&v)[S], int k) { return k < Q ? v[k - 1] : v[NLOW]; }
    // level n (compile time): forward Horner chain of level n, then its reverse for δ̄
    template <int n>
    __device__ __forceinline__ static void levels(Real (&a)[S], Real (&cb)[S], const Real (&dl)[d],
                                                  const Real (&dp)[Q + 1], Real (&gd)[d], Real (&gk)[Q + 1], int p) {
        if constexpr (n <= N) {

            Real us[Q + 1], usb[Q + 1];
            const int kq = n - 1 < Q ? n - 1 : Q;  // scalar chain length for level n
            if (kq >= 1) {
                us[1] = dp[1] * (Real(1) / Real(n)) + sc(a, 1);
#pragma unroll
                for (int k = 2; k <= Q; ++k)
                    if (k <= kq) us[k] = us[k - 1] * dp[k] * (Real(1) / Real(n - k + 1)) + sc(a, k);
            }
            if (n > Q) {
                Real uv[VS], ub[VS];
                // forward vector stages k = Q+1..n-1
#pragma unroll
                for (int k = Q + 1; k <= N - 1; ++k) {
                    if (k <= n - 1) {
                        const Real inv = Real(1) / Real(n - k + 1);
#pragma unroll
                        for (int J = 0; J < ipow(d, k - Q); ++J) {
                            const Real prev = k == Q + 1 ? us[Q] : uv[LY::vo(k - 1) + J / d];
                            uv[LY::vo(k) + J] = prev * dl[J % d] * inv + a[LY::top_off(k) + J];
                        }
                    }
                }
                // output level n: T_n'[J] = A_n[J] + u_{n-1}[J/d] δ[J%d]
                if (n - 1 > Q) {
#pragma unroll
                    for (int J = 0; J < ipow(d, n - 1 - Q); ++J) {
                        Real acc = Real(0);
#pragma unroll
                        for (int c = 0; c < d; ++c) {
                            const Real cv = cb[LY::top_off(n) + J * d + c];
                            acc += cv * dl[c];
                            gd[c] += cv * uv[LY::vo(n - 1) + J];
                        }
                        ub[LY::vo(n - 1) + J] = acc;
                    }
                    // vector stages backwards k = n-1 .. Q+2
#pragma unroll
                    for (int k = N - 1; k >= Q + 2; --k) {
                        if (k <= n - 1) {
                            const Real inv = Real(1) / Real(n - k + 1);
#pragma unroll
                            for (int J = 0; J < ipow(d, k - 1 - Q); ++J) {
                                Real acc = Real(0);
#pragma unroll
                                for (int c = 0; c < d; ++c) {
                                    const Real ubv = ub[LY::vo(k) + J * d + c];
                                    acc += ubv * dl[c];
                                    gd[c] += inv * ubv * uv[LY::vo(k - 1) + J];
                                }
                                ub[LY::vo(k - 1) + J] = inv * acc;
                            }
                        }
                    }
                    // stage Q+1: u_{Q+1}[c] = u_Q δ[c] / (n-Q) + A_{Q+1}[c]
                    {
                        const Real inv = Real(1) / Real(n - Q);
                        Real acc = Real(0);
#pragma unroll
                        for (int c = 0; c < d; ++c) {
                            acc += ub[LY::vo(Q + 1) + c] * dl[c];
                            gd[c] += inv * ub[LY::vo(Q + 1) + c] * us[Q];
                        }
                        usb[Q] = inv * acc;
                    }
                } else {  // n == Q+1: T'[c] = A[c] + u_Q δ[c]
                    Real acc = Real(0);
#pragma unroll
                    for (int c = 0; c < d; ++c) {
                        const Real cv = cb[LY::top_off(n) + c];
                        acc += cv * dl[c];
                        gd[c] += cv * us[Q];
                    }
                    usb[Q] = acc;
                }
                // scalar chain backwards k = Q..2, then k = 1
#pragma unroll
                for (int k = Q; k >= 2; --k) {
                    const Real inv = Real(1) / Real(n - k + 1);
                    gk[k] += usb[k] * us[k - 1] * inv;
                    usb[k - 1] = usb[k] * dp[k] * inv;
                }
                gk[1] += usb[1] * (Real(1) / Real(n));
            } else if (p % ipow(d, Q - n) == 0) {  // scalar output owned by this lane
                const Real cn = sc(cb, n);
                if (n == 1) {
                    gk[1] += cn;
                } else {
                    gk[n] += cn * us[n - 1];
                    usb[n - 1] = cn * dp[n];
#pragma unroll
                    for (int k = Q; k >= 2; --k) {
                        if (k <= n - 1) {
                            const Real inv = Real(1) / Real(n - k + 1);
                            gk[k] += usb[k] * us[k - 1] * inv;
                            usb[k - 1] = usb[k] * dp[k] * inv;
                        }
                    }
                    gk[1] += usb[1] * (Real(1) / Real(n));
                }
            }

            levels<n + 1>(a, cb, dl, dp, gd, gk, p);
        }
    }
};

// One Horner step S <- S ⊠ exp(δ) on a lane's slice (levels descending, so
// lower levels are still the old state): the slice-local fold of the forward
// kernels in scalar form. With -δ it undoes a step (exp(-δ) is the inverse of
// exp(δ)), which is how the backward walk recovers the states it needs.
template <typename Real, int d, int N, int Q>
struct VjpSliceFold {
    using LY = SliceLayout<d, N, Q>;
    static constexpr int S = LY::S, NLOW = LY::NLOW, VS = LY::VS;
    __device__ __forceinline__ static Real& sc(Real (&v)[S], int k) { return k < Q ? v[k - 1] : v[NLOW]; }
    template <int n>
    __device__ __forceinline__ static void levels(Real (&st)[S], const Real (&dl)[d], const Real (&dp)[Q + 1]) {
        if constexpr (n >= 1) {
            if constexpr (n == 1) {
                sc(st, 1) += dp[1];
            } else {
                Real u = dp[1] * (Real(1) / Real(n)) + sc(st, 1);
                constexpr int kq = n - 1 < Q ? n - 1 : Q;
#pragma unroll
                for (int k = 2; k <= kq; ++k) u = u * dp[k] * (Real(1) / Real(n - k + 1)) + sc(st, k);
                if constexpr (n <= Q) {
                    sc(st, n) += u * dp[n];
                } else {
                    Real uv[VS];
#pragma unroll
                    for (int k = Q + 1; k <= n - 1; ++k) {
                        const Real inv = Real(1) / Real(n - k + 1);
#pragma unroll
                        for (int J = ipow(d, k - Q) - 1; J >= 0; --J) {
                            const Real prev = k == Q + 1 ? u : uv[LY::vo(k - 1) + J / d];
                            uv[LY::vo(k) + J] = prev * dl[J % d] * inv + st[LY::top_off(k) + J];
                        }
                    }
#pragma unroll
                    for (int J = 0; J < ipow(d, n - Q); ++J) {
                        const Real prev = n - 1 == Q ? u : uv[LY::vo(n - 1) + J / d];
                        st[LY::top_off(n) + J] += prev * dl[J % d];
                    }
                }
            }
            levels<n - 1>(st, dl, dp);
        }
    }
};

template <typename Real, int d, int N, int Q>
struct SliceGather {
    using LY = SliceLayout<d, N, Q>;
    template <int n>
    __device__ __forceinline__ static void level(const Real* __restrict__ row, bool ok, const int (&lvl)[N - Q + 1],
                                                 Real (&dst)[LY::S]) {
        if constexpr (n <= N) {
#pragma unroll
            for (int r = 0; r < ipow(d, n - Q); ++r) dst[LY::top_off(n) + r] = ok ? __ldcg(row + lvl[n - Q] + r) : Real(0);
            level<n + 1>(row, ok, lvl, dst);
        }
    }
};

template <typename Real, int d, int N, int Q>
__global__ void __launch_bounds__(128) vjp_slice_kernel(const Real* __restrict__ X, int64_t L, int64_t items,
                                                        int U, int64_t CL, const Real* __restrict__ ends,
                                                        const Real* __restrict__ cbars, Real* __restrict__ grad) {
    using LY = SliceLayout<d, N, Q>;
    constexpr int P = LY::P, SLOTS = LY::SLOTS, S = LY::S, NLOW = LY::NLOW, VS = LY::VS, GMAX = LY::GMAX;
    constexpr int D = level_off(d, N);
    __shared__ Real red[4][32][d + 1];
    const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
    const int slot = lane / P, p = lane - (lane / P) * P;
    const bool lane_on = slot < SLOTS;
    const int64_t item = ((int64_t)blockIdx.x * 4 + warp) * SLOTS + (lane_on ? slot : 0);
    const bool valid = lane_on && item < items;
    const int64_t it = valid ? item : 0;
    const int64_t b = it / U, j = it - (it / U) * U;
    const int64_t M = L - 1;
    const int64_t s_lo = j * CL < M ? j * CL : M, s_hi = (j + 1) * CL < M ? (j + 1) * CL : M;
    int dg[Q + 1];  // digits p_1..p_Q
#pragma unroll
    for (int k = 1; k <= Q; ++k) dg[k] = (p / ipow(d, Q - k)) % d;
    // 1 where digit p_k is channel c: folds the lane's δ[p_k] partials into δ̄ by FMA
    Real dmask[Q + 1][d];
#pragma unroll
    for (int k = 1; k <= Q; ++k)
#pragma unroll
        for (int c = 0; c < d; ++c) dmask[k][c] = dg[k] == c ? Real(1) : Real(0);
    Real (&rd)[32][d + 1] = red[warp];

    // the lane's slice inside a signature row: low scalars at level k (k < Q),
    // then level n >= Q at lvl[n - Q] .. + d^(n-Q) (per-lane bases, compile-time layout)
    int low[Q], lvl[N - Q + 1];
#pragma unroll
    for (int k = 1; k < Q; ++k) low[k - 1] = level_off(d, k - 1) + p / ipow(d, Q - k);
#pragma unroll
    for (int n = Q; n <= N; ++n) lvl[n - Q] = level_off(d, n - 1) + p * ipow(d, n - Q);
    Real cb[S], an[S];
    const Real* crow = cbars + it * D;
    auto gather = [&](const Real* __restrict__ row, bool ok, Real(&dst)[S]) {
#pragma unroll
        for (int k = 1; k < Q; ++k) dst[k - 1] = ok ? __ldcg(row + low[k - 1]) : Real(0);
        SliceGather<Real, d, N, Q>::template level<Q>(row, ok, lvl, dst);
    };
    const Real* xb = X + b * L * d;
    pdl_trigger();
    pdl_wait();  // cbars and ends come from the previous launches: read them through L2
                 // (ld.global.cg), never through an L1 line filled while those launches ran
    gather(crow, valid, cb);
    // the state at the chunk's end (the forward prefix, ends row), walked back
    // one step at a time: S_s = S_{s+1} ⊠ exp(-δ_s)
    gather(ends + it * D, valid, an);
    // scal(k): A_k / C̄_k at prefix p_1..p_k for k <= Q
    auto sc = [&](Real (&v)[S], int k) -> Real& { return k < Q ? v[k - 1] : v[NLOW]; };
    // points X[s+1] (hi) and X[s] (lo) of the current step in registers (all d
    // channels, and the lane's digit channels p_k separately: a register array
    // indexed by p_k would go to local memory); X[s-1] is loaded one step ahead
    Real xhi[d], xlo[d], phi[Q + 1], plo[Q + 1];
    const bool any = valid && s_hi > s_lo;
#pragma unroll
    for (int c = 0; c < d; ++c) {
        xhi[c] = any ? xb[s_hi * d + c] : Real(0);
        xlo[c] = any ? xb[(s_hi - 1) * d + c] : Real(0);
    }
#pragma unroll
    for (int k = 1; k <= Q; ++k) {
        phi[k] = any ? xb[s_hi * d + dg[k]] : Real(0);
        plo[k] = any ? xb[(s_hi - 1) * d + dg[k]] : Real(0);
    }
    // ∂/∂X_t = δ̄_{t-1} - δ̄_t, written as the walk goes: interior points of the
    // chunk and the path's end points directly, a point shared with a
    // neighbouring chunk by an atomic add onto the zero the chunk pass left
    // there (two terms from two chunks: the sum is order independent)
    const bool first_chunk = j == 0, last_chunk = j == U - 1;
    Real* gb = grad + b * L * d;
    Real prev = Real(0);  // δ̄_{s+1} of this lane's component
    // past the chunk's start the point repeats (δ = 0, the identity step): the
    // next point is loaded through a running pointer, or kept
    const Real* xp = xb + (s_hi - 2) * d;  // X[s - 1] for the first step s = s_hi - 1
    for (int64_t st = 0; st < CL; ++st, xp -= d) {
        const int64_t s = s_hi - 1 - st;
        const bool pre_on = valid && s - 1 >= s_lo;
        Real xnx[d], pnx[Q + 1];
#pragma unroll
        for (int c = 0; c < d; ++c) xnx[c] = pre_on ? xp[c] : xlo[c];
#pragma unroll
        for (int k = 1; k <= Q; ++k) pnx[k] = pre_on ? xp[dg[k]] : plo[k];
        Real dl[d], dp[Q + 1];
#pragma unroll
        for (int c = 0; c < d; ++c) dl[c] = xhi[c] - xlo[c];
#pragma unroll
        for (int k = 1; k <= Q; ++k) dp[k] = phi[k] - plo[k];
#pragma unroll
        for (int c = 0; c < d; ++c) {
            xhi[c] = xlo[c];
            xlo[c] = xnx[c];
        }
#pragma unroll
        for (int k = 1; k <= Q; ++k) {
            phi[k] = plo[k];
            plo[k] = pnx[k];
        }
        {
            Real ndl[d], ndp[Q + 1];
#pragma unroll
            for (int c = 0; c < d; ++c) ndl[c] = -dl[c];
#pragma unroll
            for (int k = 1; k <= Q; ++k) ndp[k] = -dp[k];
            VjpSliceFold<Real, d, N, Q>::template levels<N>(an, ndl, ndp);
            if (s == 0) {  // S_0: the identity, exactly (a branch, not S selects per step)
#pragma unroll
                for (int i = 0; i < S; ++i) an[i] = Real(0);
            }
        }
        Real gd[d], gk[Q + 1];
#pragma unroll
        for (int c = 0; c < d; ++c) gd[c] = Real(0);
#pragma unroll
        for (int k = 0; k <= Q; ++k) gk[k] = Real(0);
        // ---- δ̄: reverse through each level's Horner chain (owned outputs only)
        SliceRev<Real, d, N, Q>::template levels<1>(an, cb, dl, dp, gd, gk, p);
        // ---- Ā = C̄ pulled back through ⊠ exp(δ)
        Real ab[S];
#pragma unroll
        for (int J = 0; J < GMAX; ++J) ab[LY::top_off(N) + J] = cb[LY::top_off(N) + J];
        Real gq[Q + 1];  // G_Q of the targets m < Q (scalar per lane)
        // the first Horner stage (level N-1) contracts C̄_N with δ for every target m;
        // only its 1/(N-m) factor depends on m, so the contraction is shared
        constexpr int H = ipow(d, N - 1 - Q);
        Real h[H];
#pragma unroll
        for (int J = 0; J < H; ++J) {
            Real acc = Real(0);
#pragma unroll
            for (int c = 0; c < d; ++c) acc += cb[LY::top_off(N) + J * d + c] * dl[c];
            h[J] = acc;
        }
#pragma unroll
        for (int m = N - 1; m >= 1; --m) {
            // Horner down to level max(m, Q) inside the slice
            const int stop = m > Q ? m : Q;
            Real g0[GMAX], g1[GMAX];
#pragma unroll
            for (int J = 0; J < GMAX; ++J) g0[J] = cb[LY::top_off(N) + J];
#pragma unroll
            for (int l = N - 1; l >= Q; --l) {
                if (l >= stop) {
                    const Real inv = Real(1) / Real(l - m + 1);
#pragma unroll
                    for (int J = 0; J < ipow(d, l - Q); ++J) {
                        Real acc = Real(0);
                        if (l == N - 1) {
                            acc = h[J];
                        } else {
#pragma unroll
                            for (int c = 0; c < d; ++c) acc += ((N - 1 - l) % 2 == 0 ? g0[J * d + c] : g1[J * d + c]) * dl[c];
                        }
                        const Real v = cb[LY::top_off(l) + J] + inv * acc;
                        if ((N - 1 - l) % 2 == 0) g1[J] = v;
                        else g0[J] = v;
                    }
                }
            }
            const bool in1 = (N - 1 - stop) % 2 == 0;  // the last stage wrote g1
            if (m >= Q) {
#pragma unroll
                for (int J = 0; J < ipow(d, m - Q > 0 ? m - Q : 0); ++J) ab[LY::top_off(m) + J] = in1 ? g1[J] : g0[J];
            } else {
                gq[m] = in1 ? g1[0] : g0[0];
            }
        }
        // targets m < Q: continue across lanes, level l = Q-1 .. m (segmented sums over digit l+1)
#pragma unroll
        for (int m = Q - 1; m >= 1; --m) {
            Real gcur = gq[m];
#pragma unroll
            for (int l = Q - 1; l >= 1; --l) {
                if (l >= m) {
                    __syncwarp();
                    rd[lane][0] = gcur * dp[l + 1];
                    __syncwarp();
                    // idle lanes (lane >= SLOTS*P) read their own slot's range clamped to slot 0
                    const int stride = ipow(d, Q - l - 1);
                    const int base = (lane_on ? slot : 0) * P + (p / ipow(d, Q - l)) * ipow(d, Q - l);
                    Real sum = Real(0);
#pragma unroll
                    for (int c = 0; c < d; ++c) sum += rd[base + c * stride][0];
                    gcur = sc(cb, l) + (Real(1) / Real(l - m + 1)) * sum;
                }
            }
            ab[m - 1] = lane_on ? gcur : Real(0);  // idle lanes read slot 0's sums: keep them at zero
        }
        // ---- δ̄_s = segmented sum of the lanes' partials
        if constexpr (SLOTS == 1 && d <= 5) {
            // one item per warp: transposed butterfly over 32 lanes (idle lanes hold
            // zeros). After the xor-16/8/4 rounds lane l keeps component (l >> 2) & 7
            // of its half-sums; xor-2/1 finish it.
            Real v8[8];
#pragma unroll
            for (int c = 0; c < 8; ++c) {
                Real v = Real(0);
                if (c < d) {
                    v = gd[c];
#pragma unroll
                    for (int k = 1; k <= Q; ++k) v = fma(dmask[k][c], gk[k], v);
                }
                v8[c] = v;
            }
            const bool b4 = lane & 16, b3 = lane & 8, b2 = lane & 4;
            Real w4[4], w2[2];
#pragma unroll
            for (int i = 0; i < 4; ++i) {
                const Real mine = b4 ? v8[4 + i] : v8[i], other = b4 ? v8[i] : v8[4 + i];
                w4[i] = mine + __shfl_xor_sync(0xffffffffu, other, 16);
            }
#pragma unroll
            for (int i = 0; i < 2; ++i) {
                const Real mine = b3 ? w4[2 + i] : w4[i], other = b3 ? w4[i] : w4[2 + i];
                w2[i] = mine + __shfl_xor_sync(0xffffffffu, other, 8);
            }
            Real w = (b2 ? w2[1] : w2[0]) + __shfl_xor_sync(0xffffffffu, b2 ? w2[0] : w2[1], 4);
            w += __shfl_xor_sync(0xffffffffu, w, 2);
            w += __shfl_xor_sync(0xffffffffu, w, 1);
            const int c = (lane >> 2) & 7;
            if ((lane & 3) == 0 && c < d && item < items && s >= s_lo) {
                if (st > 0) gb[(s + 1) * d + c] = w - prev;
                else if (last_chunk) gb[(s + 1) * d + c] = w;
                else atomicAdd(gb + (s + 1) * d + c, w);
                if (s == s_lo) {
                    if (first_chunk) gb[s * d + c] = -w;
                    else atomicAdd(gb + s * d + c, -w);
                }
                prev = w;
            }
        } else {
            __syncwarp();
#pragma unroll
            for (int c = 0; c < d; ++c) {
                Real v = gd[c];
#pragma unroll
                for (int k = 1; k <= Q; ++k) v = fma(dmask[k][c], gk[k], v);
                rd[lane][c] = v;
            }
            __syncwarp();
            if (valid && s >= s_lo && p < d) {
                Real sum = Real(0);
                for (int q = 0; q < P; ++q) sum += rd[slot * P + q][p];
                if (st > 0) gb[(s + 1) * d + p] = sum - prev;
                else if (last_chunk) gb[(s + 1) * d + p] = sum;
                else atomicAdd(gb + (s + 1) * d + p, sum);
                if (s == s_lo) {
                    if (first_chunk) gb[s * d + p] = -sum;
                    else atomicAdd(gb + s * d + p, -sum);
                }
                prev = sum;
            }
        }
        // steps past a short chunk's start run with δ = 0, where the pull-back is
        // the identity (Ā == C̄ exactly), so no per-step select is needed (idle
        // lanes stay at zero: their only nonzero inputs, the low-level sums, are masked)
#pragma unroll
        for (int i = 0; i < S; ++i) cb[i] = ab[i];
    }
}

// Compile-time (d, N) forms of the per-path chunk passes (vjp_kernel.cuh:
// vjp_boundary_kernel is the runtime form): constant level offsets and
// divisors so the index math folds away.
template <typename Real, int d, int N>
struct ChunkPasses {
    static constexpr int D = level_off(d, N);
    __device__ __forceinline__ static int off(int n) { return level_off(d, n); }
    // terms in the adjoint sum of a level-n entry: Σ_{k=1}^{N-n} d^k
    __host__ __device__ static constexpr int terms(int n) { return n >= N ? 0 : level_off(d, N - n); }
    __host__ __device__ static constexpr bool wide(int n) { return terms(n) >= 64; }
    // Entry loops have compile-time trip counts (NT threads per CTA), so each
    // thread's index math is loop-invariant across the chunk steps.
    static constexpr int NT = 256, NW = NT / 32;
    // nxt = cur pulled back through right multiplication by sig (the adjoint of
    // cur ↦ cur ⊠ sig): entry I of level n sums Σ_k Σ_J cur[n+k][I·d^k + J]·sig[k][J].
    // Wide levels: one warp per entry, lanes split J, butterfly sum (fixed order).
    template <int n>
    __device__ __forceinline__ static void adjoint_wide(const Real* __restrict__ cur, const Real* __restrict__ sig,
                                                        Real* __restrict__ nxt) {
        if constexpr (n <= N) {
            if constexpr (wide(n)) {
                const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
#pragma unroll
                for (int it = 0; it < (ipow(d, n) + NW - 1) / NW; ++it) {
                    const int I = w + it * NW;
                    if (I < ipow(d, n)) {
                        Real acc = Real(0);
#pragma unroll
                        for (int k = 1; n + k <= N; ++k) {
                            const Real* cr = cur + off(n + k - 1) + I * ipow(d, k);
                            const Real* er = sig + off(k - 1);
#pragma unroll
                            for (int jt = 0; jt < (ipow(d, k) + 31) / 32; ++jt) {
                                const int J = lane + 32 * jt;
                                if (J < ipow(d, k)) acc = fma(cr[J], er[J], acc);
                            }
                        }
#pragma unroll
                        for (int o = 16; o > 0; o >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, o);
                        if (lane == 0) nxt[off(n - 1) + I] = acc + cur[off(n - 1) + I];
                    }
                }
            }
            adjoint_wide<n + 1>(cur, sig, nxt);
        }
    }
    // narrow levels: one thread per entry
    template <int n>
    __device__ __forceinline__ static void adjoint_narrow(const Real* __restrict__ cur, const Real* __restrict__ sig,
                                                          Real* __restrict__ nxt) {
        if constexpr (n <= N) {
            if constexpr (!wide(n)) {
#pragma unroll
                for (int it = 0; it < (ipow(d, n) + NT - 1) / NT; ++it) {
                    // reversed thread order: the first warps carry the wide entries
                    const int I = NT - 1 - (int)threadIdx.x + it * NT;
                    if (I < ipow(d, n)) {
                        Real acc = cur[off(n - 1) + I];
#pragma unroll
                        for (int k = 1; n + k <= N; ++k) {
                            const Real* cr = cur + off(n + k - 1) + I * ipow(d, k);
                            const Real* er = sig + off(k - 1);
#pragma unroll
                            for (int J = 0; J < ipow(d, k); ++J) acc = fma(cr[J], er[J], acc);
                        }
                        nxt[off(n - 1) + I] = acc;
                    }
                }
            }
            adjoint_narrow<n + 1>(cur, sig, nxt);
        }
    }
    // nxt = cur ⊠ sig (Chen product)
    template <int n>
    __device__ __forceinline__ static void product(const Real* __restrict__ cur, const Real* __restrict__ sig,
                                                   Real* __restrict__ nxt) {
        if constexpr (n <= N) {
#pragma unroll
            for (int it = 0; it < (ipow(d, n) + NT - 1) / NT; ++it) {
                const int I = (int)threadIdx.x + it * NT;
                if (I < ipow(d, n)) {
                    Real v = cur[off(n - 1) + I] + sig[off(n - 1) + I];
#pragma unroll
                    for (int a = 1; a < n; ++a) {
                        const int tail = ipow(d, n - a);
                        v = fma(cur[off(a - 1) + I / tail], sig[off(n - a - 1) + I % tail], v);
                    }
                    nxt[off(n - 1) + I] = v;
                }
            }
            product<n + 1>(cur, sig, nxt);
        }
    }
};

// Boundary + ends in one pass per path: cbars rows (cotangent at every chunk
// end, backwards from the output cotangent) and ends rows (forward prefix at
// every chunk end). The forward scan and the backward pull-back are
// independent chains, so step t does forward product t and backward
// pull-back U-1-t together (one barrier per step). resident != 0: all U chunk
// signatures are staged in shared memory up front ((U + 4) D values);
// otherwise each step stages its two rows ((4 + 2) D values).
template <typename Real, int d, int N>
__global__ void __launch_bounds__(ChunkPasses<Real, d, N>::NT) vjp_chunk_passes_kernel(const Real* __restrict__ C, const Real* __restrict__ cot,
                                                               int U, int resident, Real* __restrict__ cbars,
                                                               Real* __restrict__ ends, int64_t L, int64_t CL,
                                                               Real* __restrict__ grad) {
    using CP = ChunkPasses<Real, d, N>;
    constexpr int D = CP::D;
    extern __shared__ __align__(16) unsigned char smem_raw[];
    Real* curF = reinterpret_cast<Real*>(smem_raw);
    Real* nxtF = curF + D;
    Real* curB = nxtF + D;
    Real* nxtB = curB + D;
    Real* sigs = nxtB + D;  // resident: [U][D]; else [2][D]
    const int64_t b = blockIdx.x;
    const int tid = threadIdx.x, nth = blockDim.x;
    const Real* Cb = C + b * U * D;
    pdl_trigger();
    pdl_wait();
    // the slice walk adds the two chunks' terms of every shared chunk point onto zeros
    for (int i = tid; i < (U - 1) * d; i += nth) grad[(b * L + (int64_t)(i / d + 1) * CL) * d + i % d] = Real(0);
    if (resident) {  // the predecessor's rows: L2, not L1; 16-byte loads when aligned
        const size_t bytes = (size_t)U * D * sizeof(Real);
        if (bytes % 16 == 0 && (reinterpret_cast<uintptr_t>(Cb) & 15) == 0) {
            const int4* src = reinterpret_cast<const int4*>(Cb);
            int4* dst = reinterpret_cast<int4*>(sigs);
            const int n16 = (int)(bytes / 16);
#pragma unroll 8
            for (int i = tid; i < n16; i += nth) dst[i] = __ldcg(src + i);
        } else {
            for (int i = tid; i < U * D; i += nth) sigs[i] = __ldcg(Cb + i);
        }
    }
    for (int i = tid; i < D; i += nth) {
        const Real v = __ldcg(cot + b * D + i);
        curF[i] = Real(0);
        curB[i] = v;
        cbars[(b * U + U - 1) * D + i] = v;
    }
    for (int t = 0; t < U; ++t) {
        const int jb = U - 1 - t;  // backward: cbars[jb-1] = cbars[jb] pulled back through C_jb
        const Real *sF = sigs + (size_t)t * D, *sB = sigs + (size_t)jb * D;
        if (!resident) {
            for (int i = tid; i < D; i += nth) {
                sigs[i] = __ldcg(Cb + (size_t)t * D + i);
                if (jb >= 1) sigs[D + i] = __ldcg(Cb + (size_t)jb * D + i);
            }
            sF = sigs;
            sB = sigs + D;
        }
        __syncthreads();
        if (jb >= 1) CP::template adjoint_wide<1>(curB, sB, nxtB);
        CP::template product<1>(curF, sF, nxtF);
        if (jb >= 1) CP::template adjoint_narrow<1>(curB, sB, nxtB);
        __syncthreads();
        Real* x = curF;
        curF = nxtF;
        nxtF = x;
        x = curB;
        curB = nxtB;
        nxtB = x;
        // rows out (coalesced; the next step writes the other buffers)
        Real* ef = ends + (b * U + t) * D;
        Real* cf = cbars + (b * U + (jb >= 1 ? jb - 1 : 0)) * D;
        for (int i = tid; i < D; i += nth) {
            ef[i] = curF[i];
            if (jb >= 1) cf[i] = curB[i];
        }
    }
}

// The same two passes by degree, every chunk at once (round 2; the pass above
// is U dependent Chen steps per path, ~1.9 us each on B200). With E^(j) =
// C^(0) ⊠ ... ⊠ C^(j) (the ends rows) and T^(j) = C^(j+1) ⊠ ... ⊠ C^(U-1)
// (T^(U-1) = 1), level n of either needs only levels < n of the other rows:
//   E_n^(j) = E_n^(j-1) + C_n^(j) + Σ_{a=1}^{n-1} E_a^(j-1) ⊗ C_{n-a}^(j)
//   T_n^(j) = T_n^(j+1) + C_n^(j+1) + Σ_{a=1}^{n-1} C_a^(j+1) ⊗ T_{n-a}^(j+1)
// (tensor_algebra.cpp:80-102). Per level two barrier-separated phases: the
// increments (every (chunk, entry) independent), then the running sums over
// the chunks (one thread per entry; its loads are independent of the sum).
// Then the cotangent at every chunk end is the output cotangent pulled back
// through right multiplication by T^(j) (the composition of the per-chunk
// pull-backs the pass above applies one at a time):
//   cbar^(j)_m[I] = cot_m[I] + Σ_{k=1}^{N-m} Σ_J cot_{m+k}[I·J] T_k^(j)[J].
// Two CTAs per path (the forward and the backward scan run concurrently).
// Shared memory (ScanPasses::smem): the C rows, levels < N of the E and T
// rows and the cotangent; the level-N increments of E replace C_N in place and
// their sums go straight to the ends rows (T_N is never needed).
template <typename Real, int d, int N>
struct ScanPasses {
    static constexpr int D = level_off(d, N), DL = level_off(d, N - 1);
    static constexpr int NT = 512;
    __host__ __device__ static constexpr size_t smem(int U) { return ((size_t)U * D + (size_t)2 * U * DL + D) * sizeof(Real); }
};

// The two passes on shared-memory rows (any block size): Cs [U][D] the chunk
// signatures, Es / Ts
// [U][DL], cs [D] the output cotangent. FWD: E, written to the ends rows eb;
// BWD: T, then the cbar rows cb. Barriers inside: every thread of the block calls it.
template <typename Real, int d, int N, bool FWD, bool BWD>
__device__ __forceinline__ void scan_passes_smem(Real* __restrict__ Cs, Real* __restrict__ Es, Real* __restrict__ Ts,
                                                 const Real* __restrict__ cs, int U, Real* __restrict__ eb,
                                                 Real* __restrict__ cb, int tid, int nth) {
    constexpr int D = level_off(d, N), DL = level_off(d, N - 1);
    // one barrier per level: the thread owning entry I of level n (of E, or of T) walks the
    // chunks with the running sum in a register; the increment's loads (lower levels, done
    // at earlier levels) do not depend on the sum, so consecutive chunks overlap
#pragma unroll
    for (int n = 1; n <= N; ++n) {
        const int sz = ipow(d, n), on = level_off(d, n - 1);
        const int nE = FWD ? sz : 0, nT = (BWD && n < N) ? sz : 0;  // T_N is never needed
        for (int w = tid; w < nE + nT; w += nth) {
            if (w < nE) {  // E_n^(j) = E_n^(j-1) + C_n^(j) + Σ_a E_a^(j-1) ⊗ C_{n-a}^(j)
                const int I = w;
                Real run = Real(0);
                const Real* c = Cs + on + I;
                Real* e = Es + on + I;
                Real* g = eb + on + I;
#pragma unroll 4
                for (int j = 0; j < U; ++j) {
                    Real x = c[(size_t)j * D];
                    if (j > 0) {
#pragma unroll
                        for (int a = 1; a < n; ++a) {
                            const int tail = ipow(d, n - a);
                            x = fma(Es[(size_t)(j - 1) * DL + level_off(d, a - 1) + I / tail],
                                    Cs[(size_t)j * D + level_off(d, n - a - 1) + I % tail], x);
                        }
                    }
                    run += x;
                    if (n < N) e[(size_t)j * DL] = run;
                    g[(size_t)j * D] = run;
                }
            } else {  // T_n^(j) = T_n^(j+1) + C_n^(j+1) + Σ_a C_a^(j+1) ⊗ T_{n-a}^(j+1)
                const int I = w - nE;
                Real run = Real(0);
                Real* t = Ts + on + I;
                t[(size_t)(U - 1) * DL] = Real(0);
#pragma unroll 4
                for (int j = U - 2; j >= 0; --j) {
                    Real y = Cs[(size_t)(j + 1) * D + on + I];
#pragma unroll
                    for (int a = 1; a < n; ++a) {
                        const int tail = ipow(d, n - a);
                        y = fma(Cs[(size_t)(j + 1) * D + level_off(d, a - 1) + I / tail],
                                Ts[(size_t)(j + 1) * DL + level_off(d, n - a - 1) + I % tail], y);
                    }
                    run += y;
                    t[(size_t)j * DL] = run;
                }
            }
        }
        __syncthreads();
    }
    if constexpr (BWD) {
        // cbar rows, level by level (compile-time index structure; four partial sums:
        // the level-1 entries carry ~D terms)
#pragma unroll
        for (int m = 1; m <= N; ++m) {
            const int sz = ipow(d, m), om = level_off(d, m - 1);
            for (int w = tid; w < U * sz; w += nth) {
                const int j = w / sz, I = w - (w / sz) * sz;
                Real acc[4] = {cs[om + I], Real(0), Real(0), Real(0)};
                if (j < U - 1) {
                    const Real* tj = Ts + (size_t)j * DL;
#pragma unroll
                    for (int k = 1; k <= N - m; ++k) {
                        const Real* cr = cs + level_off(d, m + k - 1) + I * ipow(d, k);
                        const Real* tr = tj + level_off(d, k - 1);
#pragma unroll 16
                        for (int J = 0; J < ipow(d, k); ++J) acc[J & 3] = fma(cr[J], tr[J], acc[J & 3]);
                    }
                }
                cb[(size_t)j * D + om + I] = (acc[0] + acc[1]) + (acc[2] + acc[3]);
            }
        }
    }
}

template <typename Real, int d, int N>
__global__ void __launch_bounds__(ScanPasses<Real, d, N>::NT) vjp_scan_passes_kernel(
    const Real* __restrict__ C, const Real* __restrict__ cot, int U, int, Real* __restrict__ cbars,
    Real* __restrict__ ends, int64_t L, int64_t CL, Real* __restrict__ grad) {
    using SP = ScanPasses<Real, d, N>;
    constexpr int D = SP::D, DL = SP::DL;
    extern __shared__ __align__(16) unsigned char smem_raw[];
    Real* Cs = reinterpret_cast<Real*>(smem_raw);  // [U][D]  C^(j)
    Real* Es = Cs + (size_t)U * D;                   // [U][DL] E^(j), levels < N
    Real* Ts = Es + (size_t)U * DL;                  // [U][DL] T^(j), levels < N
    Real* cs = Ts + (size_t)U * DL;                  // [D] output cotangent
    // two CTAs per path: even blocks run the forward scan (E, the ends rows; they also zero
    // the gradient's shared chunk points), odd blocks the backward scan (T, then the cbar rows)
    const bool fwd = (blockIdx.x & 1) == 0;
    const int64_t b = blockIdx.x >> 1;
    const int tid = threadIdx.x;
    const Real* Cb = C + b * U * D;
    pdl_trigger();
    pdl_wait();
    if (fwd) {
        Real* gb = grad + b * L * d;
        for (int i = tid; i < (U - 1) * d; i += SP::NT) {
            const int j = i / d;
            gb[(int64_t)(j + 1) * CL * d + (i - j * d)] = Real(0);
        }
    }
    // the predecessor's rows through L2 (ld.global.cg), 16-byte loads when aligned
    if ((((size_t)U * D * sizeof(Real)) & 15) == 0 && (reinterpret_cast<uintptr_t>(Cb) & 15) == 0) {
        const int4* src = reinterpret_cast<const int4*>(Cb);
        int4* dst = reinterpret_cast<int4*>(Cs);
        const int n16 = (int)((size_t)U * D * sizeof(Real) / 16);
#pragma unroll 4
        for (int i = tid; i < n16; i += SP::NT) dst[i] = __ldcg(src + i);
    } else {
#pragma unroll 4
        for (int i = tid; i < U * D; i += SP::NT) Cs[i] = __ldcg(Cb + i);
    }
    if (!fwd)
        for (int i = tid; i < D; i += SP::NT) cs[i] = __ldcg(cot + b * D + i);
    __syncthreads();
    if (fwd) scan_passes_smem<Real, d, N, true, false>(Cs, Es, Ts, cs, U, ends + b * U * D, nullptr, tid, SP::NT);
    else scan_passes_smem<Real, d, N, false, true>(Cs, Es, Ts, cs, U, nullptr, cbars + b * U * D, tid, SP::NT);
}

}  // namespace sigk
