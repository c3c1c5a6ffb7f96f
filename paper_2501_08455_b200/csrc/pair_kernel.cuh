// Pair-fold kernel: the sm_100a fp32 fold in packed FP32x2 arithmetic.
//
// Same math as fold.cuh (reference detail::sequential_forward<Real>,
// /root/reference/proj/include/sigkit/detail/sig_core.hpp:116-147; Horner form
// of exp_into :72-90 + fold_step :92-114), organised
// around the Blackwell packed FMA (PTX fma.rn.f32x2 -> SASS FFMA2):
//
//  * Pairs. A thread owns the prefix slice `pre` of TWO chunks of one path
//    (chunks 2k and 2k+1) and advances both in lockstep: every state value,
//    every table operand and every Horner temporary is a (chunk 2k, chunk 2k+1)
//    pair in one 64-bit register pair, so every FMA of the step is one FFMA2.
//    Measured on B200 (tools/ffma_pattern_probe.cu): FFMA2 with one reused
//    operand issues at the FFMA peak while using half the issue slots, where
//    scalar FFMA with two fresh register operands loses 10-20% to register
//    bank conflicts. The freed issue slots absorb the shared-memory operand
//    loads and loop overhead.
//  * Table. Step operands come from a shared-memory table of (pair-unit,
//    step) rows holding δ/m for m = 1..N-1 for the CTA's whole segment, built
//    once by all threads (coalesced loads of X, δ = X[t+1] - X[t]) before a
//    single barrier; the fold itself then runs barrier-free from registers
//    and 16-byte broadcast loads of the table.
//  * Segments. Long paths are split into G segments of one CTA each; a CTA
//    writes R = A_seg ⊠ C_seg to scratch and the last segment CTA of the path
//    to finish (fence + per-path counter) applies the same combine across
//    the G segment rows.
//  * Chunk starts. Chunk j folds from A = (1, X[s_j] - X[0], 0, ..., 0)
//    instead of the identity: the fold is S <- S ⊠ exp(δ) so it yields
//    Y = A ⊠ C (Chen, tensor_algebra.cpp:80-102) at no extra cost, and the
//    combine (pair_combine) no longer needs any P_1 ⊗ C cross term.
#pragma once

#include <cooperative_groups.h>

#include "fold.cuh"

namespace sigk {

using f2 = unsigned long long;  // packed (lo = chunk 2k, hi = chunk 2k+1) float pair

__device__ __forceinline__ f2 f2_pack(float lo, float hi) {
    f2 r;
    asm("mov.b64 %0, {%1, %2};" : "=l"(r) : "f"(lo), "f"(hi));
    return r;
}
__device__ __forceinline__ void f2_unpack(f2 v, float& lo, float& hi) {
    asm("mov.b64 {%0, %1}, %2;" : "=f"(lo), "=f"(hi) : "l"(v));
}
__device__ __forceinline__ f2 ffma2(f2 a, f2 b, f2 c) {
    f2 r;
    asm("fma.rn.f32x2 %0, %1, %2, %3;" : "=l"(r) : "l"(a), "l"(b), "l"(c));
    return r;
}
__device__ __forceinline__ f2 fadd2(f2 a, f2 b) {
    f2 r;
    asm("add.rn.f32x2 %0, %1, %2;" : "=l"(r) : "l"(a), "l"(b));
    return r;
}
__device__ __forceinline__ f2 f2_bcast(float s) { return f2_pack(s, s); }

__device__ __forceinline__ f2 fmul2(f2 a, f2 b) {
    f2 r;
    asm("mul.rn.f32x2 %0, %1, %2;" : "=l"(r) : "l"(a), "l"(b));
    return r;
}

// Per-thread Horner step on pairs. Table rows hold δ/m for m = 1..NR. Table
// mode (LEAN = false, NR = N-1): every scaled operand comes from the table and
// a step is exactly ops_per_step() FFMA2/FADD2. Lean mode (LEAN = true, NR = 1,
// used for Q >= 2 where a thread's scalar chains are short): the table holds
// δ only (a third of the shared memory, so more CTAs fit per SM) and the 1/m
// factors are folded into the running products with a few FMUL2.
template <int DIM, int DEPTH, int Q, bool LEAN_ = (Q >= 2)>
struct PairFold {
    static constexpr int d = DIM, N = DEPTH, QQ = Q;
    static constexpr bool LEAN = LEAN_;
    static constexpr int P = ipow(d, Q);             // slices (threads) per pair-unit
    static constexpr int NLOW = Q > 1 ? Q - 1 : 0;   // redundant scalars T_1..T_{Q-1}
    static constexpr int NMIN = Q > 1 ? Q : 1;       // first level stored as a slice
    __host__ __device__ static constexpr int top_off(int n) {
        int o = NLOW;
        for (int m = NMIN; m < n; ++m) o += ipow(d, m - Q);
        return o;
    }
    static constexpr int S = top_off(N + 1);          // state pairs per thread
    static constexpr int FJ = ipow(d, N - Q);         // level-N values per thread
    static constexpr int NR = (LEAN || N == 1) ? 1 : N - 1;  // table rows δ/m, m = 1..NR
    static constexpr int RP = (d % 2) ? d + 1 : d;    // pairs per row (16-byte aligned rows)
    static constexpr int RS = NR * RP;                // pairs per (step, pair-unit)
    static constexpr int NV = LEAN ? 1 : (Q == 0 ? NR : N - Q);  // vector rows a step reads
    static constexpr int QS = Q > 0 ? Q : 1;
    static constexpr int GM = LEAN ? 1 : NR;          // digit k >= 2 reads rows 1..GM

    // FMA-pipe ops per thread per step (each one FFMA2/FADD2/FMUL2 = 2 FMA-pipe cycles).
    __host__ __device__ static constexpr int ops_per_step() {
        int ops = 0;
        for (int n = 1; n <= N; ++n) {
            if (n > Q) {
                ops += Q;
                for (int k = Q + 1; k <= n; ++k) ops += ipow(d, k - Q);
                if (LEAN) {
                    for (int k = 2; k <= Q; ++k) ops += (n - k + 1 > 1);            // digit chain scalings
                    for (int k = Q + 1; k <= n - 1; ++k)                              // vector stage prescales
                        ops += (n - k + 1 > 1) ? (k == Q + 1 ? 1 : ipow(d, k - Q - 1)) : 0;
                }
            } else {
                ops += n;
                if (LEAN)
                    for (int k = 2; k <= n - 1; ++k) ops += (n - k + 1 > 1);
            }
        }
        return ops;
    }
    // shared-memory load instructions per thread per step
    __host__ __device__ static constexpr int loads_per_step() {
        int l = NV * ((d + 1) / 2) + (Q > 0 ? 1 : 0);
        for (int k = 2; k <= Q; ++k) l += LEAN ? 1 : N - k + 1;
        return l;
    }

    // 32-bit registers of one step's operands; the fold prefetches the next
    // step's operands when state + two operand sets stay within ~96 registers
    static constexpr int OPREGS = 2 * (NV * d + (Q > 0 ? 1 : 0) + (Q > 1 ? (Q - 1) * GM : 0));
    static constexpr bool PREFETCH = 2 * S + 2 * OPREGS <= 96;

    struct Ops {
        f2 v[NV][d];    // v[m-1][c] = δ[c] / m
        f2 g1;          // δ[p_1]
        f2 g[QS][GM];   // g[k-1][m-1] = δ[p_k] / m, k >= 2
    };

    __device__ __forceinline__ static f2& scal(f2 (&st)[S], int k) { return k < Q ? st[k - 1] : st[top_off(Q)]; }

    __device__ __forceinline__ static void load(Ops& o, const f2* __restrict__ row, const int (&dig)[QS]) {
#pragma unroll
        for (int m = 0; m < NV; ++m) {
            const f2* r = row + m * RP;
#pragma unroll
            for (int c = 0; c + 1 < d; c += 2) {
                const ulonglong2 v = *reinterpret_cast<const ulonglong2*>(r + c);
                o.v[m][c] = v.x;
                o.v[m][c + 1] = v.y;
            }
            if constexpr (d % 2) o.v[m][d - 1] = r[d - 1];
        }
        if constexpr (Q > 0) o.g1 = row[dig[0]];
#pragma unroll
        for (int k = 2; k <= Q; ++k)
#pragma unroll
            for (int m = 1; m <= (LEAN ? 1 : N - k + 1); ++m) o.g[k - 1][m - 1] = row[(m - 1) * RP + dig[k - 1]];
    }

    // u * δ[p_k]/m + T: table mode reads δ[p_k]/m, lean mode scales u first
    __device__ __forceinline__ static f2 chain(f2 u, const Ops& o, int k, int m, f2 T) {
        if constexpr (LEAN) {
            if (m > 1) u = fmul2(u, f2_bcast(1.0f / float(m)));
            return ffma2(u, o.g[k - 1][0], T);
        } else {
            return ffma2(u, o.g[k - 1][m - 1], T);
        }
    }
    // row m of δ as the multiplier for stage operands (lean: row 1, caller prescaled)
    __device__ __forceinline__ static f2 vrow(const Ops& o, int m, int c) { return LEAN ? o.v[0][c] : o.v[m - 1][c]; }

    template <int n>
    __device__ __forceinline__ static void level(f2 (&st)[S], const Ops& o) {
        constexpr float inv_n = 1.0f / float(n);
        if constexpr (n > Q) {
            constexpr int F = n - Q;
            f2 u0 = 0;
            if constexpr (Q >= 1) {
                u0 = ffma2(o.g1, f2_bcast(inv_n), scal(st, 1));  // δ[p1]/n + T_1[p1]
#pragma unroll
                for (int k = 2; k <= Q; ++k) u0 = chain(u0, o, k, n - k + 1, scal(st, k));
            }
            if constexpr (F == 1) {
                constexpr int ot = top_off(n);
#pragma unroll
                for (int c = 0; c < d; ++c) {
                    if constexpr (Q == 0) st[ot + c] = fadd2(st[ot + c], o.v[0][c]);  // n == 1
                    else st[ot + c] = ffma2(u0, o.v[0][c], st[ot + c]);
                }
            } else {
                f2 ua[ipow(d, F - 1)];
                {
                    constexpr int o1 = top_off(Q + 1);
                    constexpr int m = n - Q;  // stage Q+1 multiplies by δ/(n-Q)
                    if constexpr (Q == 0) {
#pragma unroll
                        for (int c = 0; c < d; ++c) ua[c] = ffma2(o.v[0][c], f2_bcast(inv_n), st[o1 + c]);
                    } else {
                        const f2 us = (LEAN && m > 1) ? fmul2(u0, f2_bcast(1.0f / float(m))) : u0;
#pragma unroll
                        for (int c = 0; c < d; ++c) ua[c] = ffma2(us, vrow(o, m, c), st[o1 + c]);
                    }
                }
                stages<n, Q + 2>(st, o, ua);
                constexpr int ot = top_off(n);
#pragma unroll
                for (int J = 0; J < ipow(d, F); ++J) st[ot + J] = ffma2(ua[J / d], o.v[0][J % d], st[ot + J]);
            }
        } else {  // scalar level n <= Q
            if constexpr (n == 1) {
                scal(st, 1) = fadd2(scal(st, 1), o.g1);
            } else {
                f2 u = ffma2(o.g1, f2_bcast(inv_n), scal(st, 1));
#pragma unroll
                for (int k = 2; k <= n - 1; ++k) u = chain(u, o, k, n - k + 1, scal(st, k));
                scal(st, n) = ffma2(u, o.g[n - 1][0], scal(st, n));
            }
        }
    }

    template <int n, int k, int UA>
    __device__ __forceinline__ static void stages(f2 (&st)[S], const Ops& o, f2 (&ua)[UA]) {
        if constexpr (k <= n - 1) {
            constexpr int sz = ipow(d, k - Q);
            constexpr int ok = top_off(k);
            constexpr int m = n - k + 1;
            if constexpr (LEAN && m > 1) {
#pragma unroll
                for (int J = 0; J < sz / d; ++J) ua[J] = fmul2(ua[J], f2_bcast(1.0f / float(m)));
            }
#pragma unroll
            for (int J = sz - 1; J >= 0; --J) ua[J] = ffma2(ua[J / d], vrow(o, m, J % d), st[ok + J]);
            stages<n, k + 1>(st, o, ua);
        }
    }

    template <int n>
    __device__ __forceinline__ static void levels_desc(f2 (&st)[S], const Ops& o) {
        if constexpr (n >= 1) {
            level<n>(st, o);
            levels_desc<n - 1>(st, o);
        }
    }
    __device__ __forceinline__ static void step(f2 (&st)[S], const Ops& o) { levels_desc<N>(st, o); }
};

__device__ __forceinline__ void cp_async4(void* dst, const void* src) {
    asm volatile("cp.async.ca.shared.global [%0], [%1], 4;" ::"r"(static_cast<uint32_t>(__cvta_generic_to_shared(dst))),
                 "l"(src)
                 : "memory");
}
__device__ __forceinline__ void cp_async_wait_all() { asm volatile("cp.async.wait_all;" ::: "memory"); }
__device__ __forceinline__ uint32_t smem_addr(const void* p) {
    return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_addr(bar)), "r"(count) : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity) {
    asm volatile(
        "{\n\t.reg .pred p;\n"
        "LAB_WAIT:\n\t"
        "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n\t"
        "@!p bra LAB_WAIT;\n}" ::"r"(smem_addr(bar)),
        "r"(parity)
        : "memory");
}

// ---------------------------------------------------------------------------
// Chen combine of U consecutive pieces (chunks of a segment, or segments of a
// path). Piece j carries Y^(j) = A^(j) ⊠ C^(j), A^(j) = (1, P^(j)_1, 0, ..., 0),
// with P^(j) = P^(0) ⊠ C^(0) ⊠ ... ⊠ C^(j-1) and P^(0) = (1, p1_0, 0, ...):
//   P^(j+1)_1 = Y^(j)_1
//   P^(j+1)_n = P^(j)_n + Y^(j)_n + Σ_{a=2}^{n-1} P^(j)_a ⊗ C^(j)_{n-a}      (2 <= n < N)
//   out_N     = Σ_j [ Y^(j)_N + Σ_{a=2}^{N-1} P^(j)_a ⊗ C^(j)_{N-a} ]
//   C^(j)_1 = Y^(j)_1 - P^(j)_1,  C^(j)_m = Y^(j)_m - P^(j)_1 ⊗ C^(j)_{m-1}
// (the a = 1 cross terms are inside Y already; reference ⊠:
// tensor_algebra.cpp:80-102). Fixed summation order: deterministic for a given U.
template <int d, int N>
struct CombineLayout {
    static constexpr int DL = level_off(d, N - 1);               // levels 1..N-1
    static constexpr int DC = level_off(d, N > 2 ? N - 2 : 0);   // C levels 1..N-2
    static constexpr int LN = ipow(d, N);
    static constexpr int LNP = round_up(LN, 4);                  // padded row of level-N partial sums
    // ylow[U][DL], p10[d] (+pad), cm[U][DC], pf[U+1][DL], then red_rows x LNP (16-byte aligned)
    __host__ __device__ static constexpr size_t red_off(int U) {
        return (size_t)round_up((int)((size_t)U * DL + round_up(d, 4) + (size_t)U * DC + (size_t)(U + 1) * DL), 4);
    }
    __host__ __device__ static constexpr size_t floats(int U, int red_rows) {
        return red_off(U) + (size_t)red_rows * LNP;
    }
};

// P1S = true: pieces were folded from A^(j) = (1, P^(j)_1, 0, ...) as above.
// P1S = false (d = 1, where the recovery C_m = Y_m - P_1 ⊗ C_{m-1} would
// cancel catastrophically): pieces were folded from the identity, Y^(j) =
// C^(j), and the cross terms run from a = 1 (the plain Chen product).
template <int d, int N, bool P1S>
struct CombineSmem {
    using CL_ = CombineLayout<d, N>;
    static constexpr int AMIN = P1S ? 2 : 1;  // first cross-term degree
    float* ylow;  // [U][DL]  levels < N of Y^(j)
    float* p10;   // [d]      P^(0)_1
    float* cm;    // [U][DC]  C^(j)_m, m = 1..N-2 (P1S only)
    float* pf;    // [U+1][DL] P^(j), levels < N
    float* red;   // [rows][LNP]
    const float* p0 = nullptr;  // levels 2..N-1 of P^(0) (row layout, DL floats); null: zero
    __device__ CombineSmem(float* base, int U) {
        ylow = base;
        p10 = ylow + (size_t)U * CL_::DL;
        cm = p10 + round_up(d, 4);
        pf = cm + (size_t)U * CL_::DC;
        red = base + CL_::red_off(U);
    }
    // P^(j)_1[i] (P1S: the previous piece's Y_1; otherwise from the scan)
    __device__ __forceinline__ float p1(int j, int i) const {
        if constexpr (P1S) return j == 0 ? p10[i] : ylow[(size_t)(j - 1) * CL_::DL + i];
        else return pf[(size_t)j * CL_::DL + i];
    }
    __device__ __forceinline__ float y(int j, int n, int I) const {
        return ylow[(size_t)j * CL_::DL + level_off(d, n - 1) + I];
    }
    // level m (1 <= m <= N-2 for P1S, <= N-1 otherwise) of C^(j), as a row pointer
    __device__ __forceinline__ const float* crow(int j, int m) const {
        if constexpr (P1S) return cm + (size_t)j * CL_::DC + level_off(d, m - 1);
        else return ylow + (size_t)j * CL_::DL + level_off(d, m - 1);
    }
};

// C^(j)_{a-b}[I[b:a]] (digits of I in dg). P1S: the chain C_1 = Y_1 - P_1,
// C_m[i, rest] = Y_m[i, rest] - P_1[i] C_{m-1}[rest]; otherwise Y itself.
template <int d, int N, bool P1S>
__device__ __forceinline__ float c_chain(const CombineSmem<d, N, P1S>& S, int j, const int* dg, int a, int b) {
    if constexpr (!P1S) {
        int idx = 0;
        for (int r = b; r < a; ++r) idx = idx * d + dg[r];
        return S.y(j, a - b, idx);
    } else {
        float c = S.y(j, 1, dg[a - 1]) - S.p1(j, dg[a - 1]);
        int tail = dg[a - 1], w = d;
        for (int r = a - 2; r >= b; --r) {
            tail += dg[r] * w;
            w *= d;
            c = fmaf(-S.p1(j, dg[r]), c, S.y(j, a - r, tail));
        }
        return c;
    }
}

// Phase B (P1S only; all threads, no barriers inside): cm[j] = C^(j)_m for
// m = 1..N-2, and pf[j] level 1 = P^(j)_1 for j = 0..U.
template <int d, int N, bool P1S>
__device__ __forceinline__ void build_c(const CombineSmem<d, N, P1S>& S, int U, int tid, int nth) {
    if constexpr (P1S) {
        constexpr int DL = CombineLayout<d, N>::DL, DC = CombineLayout<d, N>::DC;
        // threads that take part in fused_scan (tid < d^(N-1)) get the last shares
        const int t0 = (tid + nth - (ipow(d, N - 1) % nth)) % nth;
        if constexpr (N >= 2) {
            for (int i = t0; i < (U + 1) * d; i += nth) S.pf[(size_t)(i / d) * DL + i % d] = S.p1(i / d, i % d);
        }
#pragma unroll
        for (int m = 1; m <= N - 2; ++m) {
            const int sz = ipow(d, m);
            for (int i = t0; i < U * sz; i += nth) {
                const int j = i / sz, I = i - (i / sz) * sz;
                int dg[N > 2 ? N - 2 : 1];
#pragma unroll
                for (int r = 0; r < m; ++r) dg[r] = (I / ipow(d, m - 1 - r)) % d;
                S.cm[(size_t)j * DC + level_off(d, m - 1) + I] = c_chain<d, N, P1S>(S, j, dg, m, 0);
            }
        }
    }
}

// Fused scan (one thread per level-(N-1) element I, sequential over pieces):
// the thread carries P^(j)_a[I[:a]] for every scanned degree a in registers,
// so all levels advance in one pass; pf[j][level a] is written by the thread
// whose trailing digits are zero.
template <int d, int N, bool P1S>
__device__ __forceinline__ void fused_scan(const CombineSmem<d, N, P1S>& S, int U, int tid, int nth) {
    constexpr int DL = CombineLayout<d, N>::DL;
    constexpr int E = N - 1;                 // top scanned level
    constexpr int A0 = P1S ? 2 : 1;          // first scanned level
    if constexpr (E >= A0) {
        for (int I = tid; I < ipow(d, E); I += nth) {
            int dg[E];
#pragma unroll
            for (int r = 0; r < E; ++r) dg[r] = (I / ipow(d, E - 1 - r)) % d;
            float P[E + 1];
            int idx[E + 1];
            bool wr[E + 1];
#pragma unroll
            for (int a = A0; a <= E; ++a) {
                idx[a] = I / ipow(d, E - a);
                wr[a] = I % ipow(d, E - a) == 0;
                P[a] = (a == 1) ? S.p10[idx[1]] : (S.p0 ? __ldcg(S.p0 + level_off(d, a - 1) + idx[a]) : 0.f);  // p0: a previous launch's output, via L2
                if (wr[a]) S.pf[level_off(d, a - 1) + idx[a]] = P[a];
            }
            // long scans (U >= 16, the latency plans): blocks of V pieces whose inputs
            // (Y entries, chain factors: independent of P) are all loaded before the
            // block's pf stores, so only the FMA recurrence through P is serial;
            // short scans keep the plain walk (measured: the blocked form costs the
            // back-to-back U = 10 plan 1%, saves ~1 K cycles at U = 20)
            constexpr int V = 4;
            const int jb = U >= 16 ? U - U % V : 0;
            for (int j0 = 0; j0 < jb; j0 += V) {
                float yv[V][E + 1], cv[V][E + 1][E + 1];
#pragma unroll
                for (int u = 0; u < V; ++u) {
#pragma unroll
                    for (int a = A0; a <= E; ++a) {
                        yv[u][a] = S.y(j0 + u, a, idx[a]);
#pragma unroll
                        for (int b = A0; b < a; ++b) cv[u][a][b] = c_chain<d, N, P1S>(S, j0 + u, dg, a, b);
                    }
                }
#pragma unroll
                for (int u = 0; u < V; ++u) {
                    float nP[E + 1];
#pragma unroll
                    for (int a = A0; a <= E; ++a) {
                        float x = P[a] + yv[u][a];
#pragma unroll
                        for (int b = A0; b < a; ++b) x = fmaf(P[b], cv[u][a][b], x);
                        nP[a] = x;
                    }
#pragma unroll
                    for (int a = A0; a <= E; ++a) {
                        P[a] = nP[a];
                        if (wr[a]) S.pf[(size_t)(j0 + u + 1) * DL + level_off(d, a - 1) + idx[a]] = P[a];
                    }
                }
            }
#pragma unroll 4
            for (int j = jb; j < U; ++j) {
                float nP[E + 1];
#pragma unroll
                for (int a = A0; a <= E; ++a) {
                    float x = P[a] + S.y(j, a, idx[a]);
#pragma unroll
                    for (int b = A0; b < a; ++b) x = fmaf(P[b], c_chain<d, N, P1S>(S, j, dg, a, b), x);
                    nP[a] = x;
                }
#pragma unroll
                for (int a = A0; a <= E; ++a) {
                    P[a] = nP[a];
                    if (wr[a]) S.pf[(size_t)(j + 1) * DL + level_off(d, a - 1) + idx[a]] = P[a];
                }
            }
        }
    }
}

// Level-N cross terms Σ_{a=AMIN}^{N-1} P^(j)_a ⊗ C^(j)_{N-a} for the FJ =
// d^(N-Q) outputs (pre, J) of a prefix slice, accumulated into acc
// (compile-time index structure: the prefix part is a scalar for a <= Q, a
// short row otherwise).
template <int d, int N, int Q, bool P1S, int a>
__device__ __forceinline__ void top_cross_slice(const CombineSmem<d, N, P1S>& S, int j, int pre,
                                                float (&acc)[ipow(d, N - Q)]) {
    constexpr int DL = CombineLayout<d, N>::DL;
    if constexpr (a < N) {
        constexpr int FJ = ipow(d, N - Q);
        constexpr int tail = ipow(d, N - a);
        const float* pa = S.pf + (size_t)j * DL + level_off(d, a - 1);
        const float* cb = S.crow(j, N - a);
        if constexpr (a <= Q) {
            const float pv = pa[pre / ipow(d, Q - a)];
            const float* cr = cb + (pre % ipow(d, Q - a)) * FJ;
#pragma unroll
            for (int J = 0; J < FJ; ++J) acc[J] = fmaf(pv, cr[J], acc[J]);
        } else {
            constexpr int PW = ipow(d, a - Q);
            const float* pr = pa + pre * PW;
            float pv[PW], cv[tail];
#pragma unroll
            for (int i = 0; i < PW; ++i) pv[i] = pr[i];
#pragma unroll
            for (int i = 0; i < tail; ++i) cv[i] = cb[i];
#pragma unroll
            for (int J = 0; J < FJ; ++J) acc[J] = fmaf(pv[J / tail], cv[J % tail], acc[J]);
        }
        top_cross_slice<d, N, Q, P1S, a + 1>(S, j, pre, acc);
    }
}

// Sum of `rows` rows of LN values (row stride LNP, 16-byte aligned) in a fixed
// order -> dst (scalar stores; dst has no alignment guarantee).
template <int LN, int LNP>
__device__ __forceinline__ void sum_rows(const float* __restrict__ red, int rows, float* __restrict__ dst) {
    for (int q = threadIdx.x; q < LNP / 4; q += blockDim.x) {
        const float4* p = reinterpret_cast<const float4*>(red) + q;
        float4 s = make_float4(0.f, 0.f, 0.f, 0.f);
        int v = 0;
        for (; v + 4 <= rows; v += 4) {
            float4 t[4];
#pragma unroll
            for (int u = 0; u < 4; ++u) t[u] = p[(size_t)(v + u) * (LNP / 4)];
#pragma unroll
            for (int u = 0; u < 4; ++u) {
                s.x += t[u].x;
                s.y += t[u].y;
                s.z += t[u].z;
                s.w += t[u].w;
            }
        }
        for (; v < rows; ++v) {
            const float4 t = p[(size_t)v * (LNP / 4)];
            s.x += t.x;
            s.y += t.y;
            s.z += t.z;
            s.w += t.w;
        }
        const int F = 4 * q;
        if (F < LN) dst[F] = s.x;
        if (F + 1 < LN) dst[F + 1] = s.y;
        if (F + 2 < LN) dst[F + 2] = s.z;
        if (F + 3 < LN) dst[F + 3] = s.w;
    }
}

// Levels 1..N-1 of both chunks of a thread's slice -> ylow rows 2k, 2k+1
// (redundant prefix scalars are written by one thread each).
template <typename PF, int n>
__device__ __forceinline__ void store_low_levels(const f2 (&st)[PF::S], int k, int pre, float* __restrict__ ylow) {
    constexpr int d = PF::d, Q = PF::QQ;
    constexpr int DL = level_off(d, PF::N - 1);
    if constexpr (n < PF::N) {
        float* y0 = ylow + (size_t)(2 * k) * DL + level_off(d, n - 1);
        float* y1 = y0 + DL;
        if constexpr (n >= PF::NMIN) {
            constexpr int sz = ipow(d, n - Q);
            constexpr int o = PF::top_off(n);
#pragma unroll
            for (int J = 0; J < sz; ++J) {
                float lo, hi;
                f2_unpack(st[o + J], lo, hi);
                y0[pre * sz + J] = lo;
                y1[pre * sz + J] = hi;
            }
        } else {
            constexpr int tail = ipow(d, Q - n);
            if (pre % tail == 0) {
                float lo, hi;
                f2_unpack(st[n - 1], lo, hi);
                y0[pre / tail] = lo;
                y1[pre / tail] = hi;
            }
        }
        store_low_levels<PF, n + 1>(st, k, pre, ylow);
    }
}

// Segment combine of one path, run by the last of its G segment CTAs to
// finish: rows Rb[g] (g = 0..G-1, written by the path's segment CTAs) are the
// pieces of the combine above with P^(0)_1 = 0; the result goes to orow.
// Loads bypass L1 (ld.global.cg): the rows were written by other SMs.
template <int d, int N, bool P1S>
__device__ __forceinline__ void segment_combine_path(const float* __restrict__ Rb, int G, float* __restrict__ smem,
                                                     float* __restrict__ orow) {
    using CLY = CombineLayout<d, N>;
    constexpr int D = level_off(d, N), DL = CLY::DL, LN = CLY::LN;
    CombineSmem<d, N, P1S> S(smem, G);
    float* top = smem + CLY::floats(G, 0);  // [G][LN] level-N parts of the rows
    const int tid = threadIdx.x, nth = blockDim.x;
    // stage all G rows (L2 reads, 8 loads in flight per thread before the stores)
    constexpr int V = 8;
    for (int i0 = tid; i0 < G * D; i0 += V * nth) {
        float v[V];
#pragma unroll
        for (int u = 0; u < V; ++u) v[u] = i0 + u * nth < G * D ? __ldcg(Rb + i0 + u * nth) : 0.f;
#pragma unroll
        for (int u = 0; u < V; ++u) {
            const int i = i0 + u * nth;
            if (i < G * D) {
                const int j = i / D, r = i - j * D;
                if (r < DL) S.ylow[(size_t)j * DL + r] = v[u];
                else top[(size_t)j * LN + r - DL] = v[u];
            }
        }
    }
    if (tid < d) S.p10[tid] = 0.f;
    __syncthreads();
    fused_scan<d, N, P1S>(S, G, tid, nth);
    build_c<d, N, P1S>(S, G, tid, nth);
    __syncthreads();
    const float* pG = S.pf + (size_t)G * DL;
    for (int i = tid; i < DL; i += nth) orow[i] = pG[i];
    for (int F = tid; F < LN; F += nth) {
        float acc = 0.f;
        for (int j = 0; j < G; ++j) {
            float x = top[(size_t)j * LN + F];
            if constexpr (N == 1 && P1S) {
                if (j != G - 1) x = 0.f;
            }
#pragma unroll
            for (int a = (P1S ? 2 : 1); a < N; ++a) {
                const int tail = ipow(d, N - a);
                x = fmaf(S.pf[(size_t)j * DL + level_off(d, a - 1) + F / tail], S.crow(j, N - a)[F % tail], x);
            }
            acc += x;
        }
        orow[DL + F] = acc;
    }
}

// Segment combine inside a thread-block cluster: the G segment CTAs of one
// path form one cluster, each holds its segment row (A_seg ⊠ C_seg, the same
// pieces as segment_combine_path) in its own shared memory at `segrow`. Every
// CTA gathers the G rows over distributed shared memory (no global round
// trip, no arrival counters), runs the (tiny) scan over the G pieces, and
// writes its own 1/G share of the output row. Two cluster barriers: rows
// complete before the gather; gathers complete before any CTA reuses or
// releases its shared memory.
template <int d, int N, bool P1S>
__device__ __forceinline__ void cluster_segment_combine(const float* segrow, int G, float* __restrict__ smem,
                                                        float* __restrict__ orow) {
    namespace cg = cooperative_groups;
    cg::cluster_group cl = cg::this_cluster();
    using CLY = CombineLayout<d, N>;
    constexpr int D = level_off(d, N), DL = CLY::DL, LN = CLY::LN;
    CombineSmem<d, N, P1S> S(smem, G);
    float* top = smem + CLY::floats(G, 0);  // [G][LN] level-N parts of the rows
    const int tid = threadIdx.x, nth = blockDim.x;
    cl.sync();  // every segment row is in its CTA's shared memory
    constexpr int V = 8;  // remote loads in flight per thread
    for (int i0 = tid; i0 < G * D; i0 += V * nth) {
        float v[V];
#pragma unroll
        for (int u = 0; u < V; ++u) {
            const int i = i0 + u * nth;
            v[u] = 0.f;
            if (i < G * D) {
                const int j = i / D;
                v[u] = cl.map_shared_rank(segrow, j)[i - j * D];
            }
        }
#pragma unroll
        for (int u = 0; u < V; ++u) {
            const int i = i0 + u * nth;
            if (i < G * D) {
                const int j = i / D, r = i - j * D;
                if (r < DL) S.ylow[(size_t)j * DL + r] = v[u];
                else top[(size_t)j * LN + r - DL] = v[u];
            }
        }
    }
    if (tid < d) S.p10[tid] = 0.f;
    cl.sync();  // all gathers done (remote rows may now be released); local staging visible
    fused_scan<d, N, P1S>(S, G, tid, nth);
    build_c<d, N, P1S>(S, G, tid, nth);
    __syncthreads();
    pdl_wait();  // output writes are ordered after the previous launch
    const int rank = (int)cl.block_rank();
    const int per = (D + G - 1) / G, lo = rank * per, hi = min(D, lo + per);
    const float* pG = S.pf + (size_t)G * DL;
    for (int i = lo + tid; i < hi; i += nth) {
        if (i < DL) {
            orow[i] = pG[i];
            continue;
        }
        const int F = i - DL;
        float acc = 0.f;
        for (int j = 0; j < G; ++j) {
            float x = top[(size_t)j * LN + F];
            if constexpr (N == 1 && P1S) {
                if (j != G - 1) x = 0.f;
            }
#pragma unroll
            for (int a = (P1S ? 2 : 1); a < N; ++a) {
                const int tail = ipow(d, N - a);
                x = fmaf(S.pf[(size_t)j * DL + level_off(d, a - 1) + F / tail], S.crow(j, N - a)[F % tail], x);
            }
            acc += x;
        }
        orow[i] = acc;
    }
}

// Steps 1-2 of a pair-family CTA (also used by the prefix-stream kernel):
// stage the segment's points X[seg0 .. seg0+slen] into `raw` and build the
// δ table `tab` ([CL][UP][RS] pairs). Returns the (shifted) raw pointer. The
// table is complete after the caller's next __syncthreads().
template <typename PF>
__device__ __forceinline__ float* pair_stage_and_table(const float* __restrict__ xb, int64_t seg0, int64_t slen,
                                                       int CL, int UP, f2* __restrict__ tab, float* raw,
                                                       uint64_t* bar, long long* staged_stamp = nullptr) {
    constexpr int d = PF::d, RS = PF::RS, RP = PF::RP, NR = PF::NR;
    const int tid = threadIdx.x, nth = blockDim.x;
    // 1. stage the segment's points X[seg0 .. seg0+slen]: one TMA bulk copy of
    //    the 16-byte-aligned body (completion on an mbarrier), plain loads for
    //    the <= 3 ragged floats at each end. raw is shifted so body addresses
    //    stay 16-byte aligned in shared memory.
    const float* src = xb + seg0 * d;
    const int nraw = (int)((slen + 1) * d);
    const uintptr_t sa = reinterpret_cast<uintptr_t>(src);
    raw += (sa & 15) / 4;
    {
        const uintptr_t a = (sa + 15) & ~uintptr_t(15), e = (sa + 4ull * nraw) & ~uintptr_t(15);
        const int h = (int)((a - sa) / 4);                                  // head floats
        const int nb = e > a ? (int)((e - a) / 4) : 0;                      // body floats
        const int t0 = nb > 0 ? h + nb : 0;                                 // first tail float
        if (tid == 0) {
            mbar_init(bar, 1);
            asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
        }
        __syncthreads();
        if (tid == 0 && nb > 0) {
            asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_addr(bar)),
                         "r"((uint32_t)(4 * nb))
                         : "memory");
            asm volatile(
                "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                    smem_addr(raw + h)),
                "l"(src + h), "r"((uint32_t)(4 * nb)), "r"(smem_addr(bar))
                : "memory");
        }
        if (nb == 0) {
            for (int i = tid; i < nraw; i += nth) raw[i] = src[i];
        } else {
            if (tid < h) raw[tid] = src[tid];
            const int tt = nth - 1 - tid;
            if (tt < nraw - t0) raw[t0 + tt] = src[t0 + tt];
            mbar_wait(bar, 0);
        }
    }
    __syncthreads();
    if (staged_stamp != nullptr && threadIdx.x == 0) *staged_stamp = clock64();  // probes: staging done
    // 2. the operand table: row (s, kk) = (δ_{2kk}[c]/m, δ_{2kk+1}[c]/m), m = 1..NR.
    //    Column (kk, c) is split into `parts` contiguous step ranges, one per thread;
    //    steps where both chunks are real run predicate-free, padding steps (δ = 0,
    //    only in the last chunks of a segment) after them.
    {
        const int cols = UP * d;
        const int parts = nth / cols > 0 ? nth / cols : 1;
        const int len = (CL + parts - 1) / parts;
        const int sl = (int)slen;
        for (int t = tid; t < cols * parts; t += nth) {
            const int col = t % cols, part = t / cols;
            const int kk = col / d, c = col - (col / d) * d;
            const int s0 = part * len, s1 = min(CL, s0 + len);
            const int cs0 = min(2 * kk * CL, sl), cs1 = min((2 * kk + 1) * CL, sl);
            const int lim0 = min(cs0 + CL, sl) - cs0, lim1 = min(cs1 + CL, sl) - cs1;  // real steps
            int o0 = (cs0 + s0) * d + c, o1 = (cs1 + s0) * d + c;
            int ro = (s0 * UP + kk) * RS + c;
            float x0 = s0 <= lim0 ? raw[o0] : 0.f, x1 = s0 <= lim1 ? raw[o1] : 0.f;
            const int sf = min(s1, min(lim0, lim1));
            int sidx = s0;
#pragma unroll 4
            for (; sidx < sf; ++sidx) {
                const float y0 = raw[o0 + d], y1 = raw[o1 + d];
                const float dl0 = y0 - x0, dl1 = y1 - x1;
                x0 = y0;
                x1 = y1;
#pragma unroll
                for (int m = 1; m <= NR; ++m) tab[ro + (m - 1) * RP] = f2_pack(dl0 * (1.0f / m), dl1 * (1.0f / m));
                o0 += d;
                o1 += d;
                ro += UP * RS;
            }
            for (; sidx < s1; ++sidx) {
                const float y0 = sidx < lim0 ? raw[o0 + d] : x0, y1 = sidx < lim1 ? raw[o1 + d] : x1;
                const float dl0 = y0 - x0, dl1 = y1 - x1;
                x0 = y0;
                x1 = y1;
#pragma unroll
                for (int m = 1; m <= NR; ++m) tab[ro + (m - 1) * RP] = f2_pack(dl0 * (1.0f / m), dl1 * (1.0f / m));
                o0 += d;
                o1 += d;
                ro += UP * RS;
            }
        }
    }
    return raw;
}

// Geometry of one pair-kernel launch (host and device agree on it).
struct PairGeom {
    int G;          // segments per path (grid = B * G)
    int64_t SL;     // steps per segment
    int U, UP, CL;  // chunks per segment (even), pair-units, steps per chunk
    int threads;    // block size (multiple of 32, >= UP * P)
    int raw_floats; // (SL + 1) * d rounded up to 4
    long long* phases;  // optional [grid][12] SM-clock stamps of thread 0 (10) + globaltimer at entry/exit (tools/pair_probe.py)
    int* counters;      // G > 1: [B] arrival counters (zero between launches)
    int smem_bytes;     // dynamic shared memory of the launch (the last 16 bytes hold a flag)
    float* final_out;   // G > 1: (B, D) signatures (the kernel's `out` then holds the (B*G, D) segment rows)
    // prefix-stream kernel, G > 1, in-kernel look-back: CTA (b, g) publishes the
    // signature of X[0 .. end of its segment] in pub row b*G + g and sets
    // flags[b*G + g] = epoch (a per-call value, so flags never need resetting)
    float* pub = nullptr;
    int* flags = nullptr;
    int epoch = 0;
    int segrow_off = 0;  // cluster launches: byte offset of the segment row in shared memory
    int64_t sub_U = 0, sub_CL = 0, sub_L = 0;  // chunk paths (PairLaunch::sub_U)
};

// Path `b` of a pair-family launch: its points and step count (chunk paths:
// a run of sub_CL + 1 points inside a path of X, shorter at the path's end).
__device__ __forceinline__ const float* pair_path(const float* X, int64_t L, int d, const PairGeom& g, int64_t b,
                                                  int64_t* M) {
    if (g.sub_U > 0) {
        const int64_t p = b / g.sub_U, j = b - (b / g.sub_U) * g.sub_U;
        const int64_t s0 = j * g.sub_CL, left = g.sub_L - 1 - s0;
        *M = left < g.sub_CL ? (left > 0 ? left : 0) : g.sub_CL;
        return X + (p * g.sub_L + (s0 < g.sub_L ? s0 : g.sub_L - 1)) * d;
    }
    *M = L - 1;
    return X + b * L * d;
}

// Offset of the cluster path's segment row (past every other use of the buffer).
template <int d, int N, int Q>
__host__ __device__ constexpr size_t pair_segrow_off(int U, int CL, int raw_floats, int G) {
    using PF = PairFold<d, N, Q>;
    const size_t seg = G > 1 ? (CombineLayout<d, N>::floats(G, 0) + (size_t)G * ipow(d, N)) * 4 : 0;
    const size_t fold = (size_t)CL * (U / 2) * PF::RS * 8 + (size_t)raw_floats * 4 + 16 + 16;
    const size_t comb = CombineLayout<d, N>::floats(U, U / 2) * 4;
    const size_t m = fold > comb ? fold : comb;
    return ((m > seg ? m : seg) + 15) / 16 * 16;
}

template <int d, int N, int Q>
__host__ __device__ constexpr size_t pair_smem_bytes(int U, int CL, int raw_floats, int G = 1, bool cluster = false) {
    return pair_segrow_off<d, N, Q>(U, CL, raw_floats, G) + (cluster ? (size_t)level_off(d, N) * 4 : 0) +
           16;  // + the segment-combine flag
}

// Steps 5-6 of a pair-family CTA after its fold (shared by pair_kernel and
// ppair_kernel): combine the U chunks of the segment (Chen, tensor_algebra.cpp:
// 80-102) and write the row, or hand it to the segment combine when G > 1.
// Every thread of the CTA calls it (fold threads with `active`).
template <typename PF, bool CLUSTER, bool P1S, typename Phase>
__device__ __forceinline__ void pair_combine_store(const f2 (&st)[PF::S], bool active, int k, int pre, float p10v,
                                                   const PairGeom& g, int64_t rowid, int64_t b,
                                                   float* __restrict__ out, unsigned char* smem_raw, Phase phase) {
    constexpr int d = PF::d, N = PF::N, Q = PF::QQ, FJ = PF::FJ;
    using CLY = CombineLayout<d, N>;
    constexpr int D = level_off(d, N), DL = CLY::DL, LN = CLY::LN;
    const int U = g.U, UP = g.UP;
    const int tid = threadIdx.x, nth = blockDim.x;
    CombineSmem<d, N, P1S> S(reinterpret_cast<float*>(smem_raw), U);
    if (active) store_low_levels<PF, 1>(st, k, pre, S.ylow);
    if constexpr (N >= 2) {
        if (tid < d) S.p10[tid] = p10v;  // P^(0)_1
    }
    __syncthreads();
    fused_scan<d, N, P1S>(S, U, tid, nth);
    build_c<d, N, P1S>(S, U, tid, nth);
    __syncthreads();
    phase(5);
    float* orow = out + rowid * D;
    if (active) {
        constexpr int ot = PF::top_off(N);
        float r[FJ];
#pragma unroll
        for (int h = 0; h < 2; ++h) {
            const int j = 2 * k + h;
            float acc[FJ];
#pragma unroll
            for (int J = 0; J < FJ; ++J) {
                float lo, hi;
                f2_unpack(st[ot + J], lo, hi);
                acc[J] = h ? hi : lo;
                if constexpr (N == 1 && P1S) {
                    if (j != U - 1) acc[J] = 0.f;  // level 1 of the segment = the last chunk's Y_1
                }
            }
            top_cross_slice<d, N, Q, P1S, P1S ? 2 : 1>(S, j, pre, acc);
#pragma unroll
            for (int J = 0; J < FJ; ++J) r[J] = h ? r[J] + acc[J] : acc[J];
        }
        float* rr = S.red + (size_t)k * CLY::LNP + (size_t)pre * FJ;
#pragma unroll
        for (int J = 0; J < FJ; ++J) rr[J] = r[J];
    }
    __syncthreads();
    phase(6);
    if constexpr (CLUSTER) {
        // the segment row stays in shared memory for the cluster combine
        float* segrow = reinterpret_cast<float*>(smem_raw + g.segrow_off);
        const float* pU = S.pf + (size_t)U * DL;
        for (int i = tid; i < DL; i += nth) segrow[i] = pU[i];
        sum_rows<LN, CLY::LNP>(S.red, UP, segrow + DL);
        phase(7);
        phase(8);
        cluster_segment_combine<d, N, P1S>(segrow, g.G, reinterpret_cast<float*>(smem_raw), out + b * D);
        phase(9);
        return;
    }
    pdl_wait();  // the previous launch has completed: output writes are ordered after its
    const float* pU = S.pf + (size_t)U * DL;
    for (int i = tid; i < DL; i += nth) orow[i] = pU[i];
    sum_rows<LN, CLY::LNP>(S.red, UP, orow + DL);
    phase(7);
    if (g.G > 1) {
        // segment row written to scratch; the last of the path's G CTAs combines them
        // (classic fence + counter: no second kernel, no grid-wide serialisation)
        int* s_last = reinterpret_cast<int*>(smem_raw + g.smem_bytes - 16);
        __threadfence();
        __syncthreads();
        if (tid == 0) *s_last = atomicAdd(g.counters + b, 1) == g.G - 1;
        __syncthreads();
        phase(8);
        if (*s_last) {
            __threadfence();
            if (tid == 0) g.counters[b] = 0;  // ready for the next launch
            segment_combine_path<d, N, P1S>(out + b * g.G * D, g.G, reinterpret_cast<float*>(smem_raw),
                                            g.final_out + b * D);
        }
    }
    phase(9);
}

// X: (B, L, d) fp32. grid = B * G CTAs; CTA (b, g) folds steps
// [g*SL, min((g+1)*SL, M)) of path b as U chunks and writes row b*G + g of
// `out` ((B*G, D)): A_seg ⊠ C_seg with A_seg = (1, X[seg start] - X[0], 0, ...),
// i.e. the path's signature when G == 1.
// CLUSTER: launched with a cluster of G CTAs per path (G <= 8); the segment
// rows are combined over distributed shared memory (cluster_segment_combine)
// and `out` is the (B, D) output itself.
template <int DIM, int DEPTH, int Q, int NT, int MINB, bool CLUSTER = false, bool P1S = (DIM > 1 && DEPTH > 1)>
__global__ void __launch_bounds__(NT, MINB) pair_kernel(const float* __restrict__ X, int64_t L, PairGeom g,
                                                        float* __restrict__ out) {
    using PF = PairFold<DIM, DEPTH, Q>;
    using CLY = CombineLayout<DIM, DEPTH>;
    constexpr int d = DIM, N = DEPTH, P = PF::P, RS = PF::RS, RP = PF::RP, NR = PF::NR;
    constexpr int D = level_off(DIM, DEPTH);
    constexpr int DL = CLY::DL, DC = CLY::DC, LN = CLY::LN, FJ = PF::FJ;
    extern __shared__ __align__(16) unsigned char smem_raw[];

    const int64_t rowid = blockIdx.x;
    const int64_t b = rowid / g.G, sg = rowid - b * g.G;
    int64_t M;
    const float* __restrict__ xb = pair_path(X, L, d, g, b, &M);
    const int64_t seg0 = sg * g.SL < M ? sg * g.SL : M;
    const int64_t slen = (seg0 + g.SL < M ? seg0 + g.SL : M) - seg0;
    const int U = g.U, UP = g.UP, CL = g.CL;
    const int tid = threadIdx.x, nth = blockDim.x;

    f2* tab = reinterpret_cast<f2*>(smem_raw);                                   // [CL][UP][RS]
    float* raw = reinterpret_cast<float*>(smem_raw + (size_t)CL * UP * RS * 8);  // [(slen+1)*d + 4]
    uint64_t* bar = reinterpret_cast<uint64_t*>(raw + g.raw_floats + 4);         // staging mbarrier

    auto phase = [&](int i) {
        if (g.phases != nullptr && tid == 0) {
            g.phases[rowid * 12 + i] = clock64();
            if (i == 0 || i == 9) {  // wall time (ns) at entry and exit: SM clock and launch spread
                unsigned long long t;
                asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
                g.phases[rowid * 12 + 10 + (i == 9)] = (long long)t;
            }
        }
    };
    phase(0);
    pdl_trigger();  // the next launch may start on free SMs now
    // X[b, 0, c] for the chunk starts (P_1 = X[s_j] - X[0]) and P^(0)_1, issued early
    const bool active = tid < UP * P;
    const int k = active ? tid / P : 0;
    const int pre = active ? tid - (tid / P) * P : 0;
    int dig[PF::QS];
#pragma unroll
    for (int q = 0; q < PF::QS; ++q) dig[q] = (Q > 0) ? (pre / ipow(d, Q > 0 ? Q - 1 - q : 0)) % d : 0;
    float x0[Q == 0 ? d : 1];
#pragma unroll
    for (int c = 0; c < (Q == 0 ? d : 1); ++c) x0[c] = __ldg(xb + (Q == 0 ? c : dig[0]));
    float p10v = 0.f;
    if (P1S && tid < d) p10v = __ldg(xb + seg0 * d + tid) - __ldg(xb + tid);
    raw = pair_stage_and_table<PF>(xb, seg0, slen, CL, UP, tab, raw, bar,
                                   (g.phases != nullptr && g.G == 1) ? g.phases + rowid * 12 + 8 : nullptr);
    phase(1);
    // 3. per-thread state: slice `pre` of chunks 2k and 2k+1, started from (1, X[s_j] - X[0], 0, ...)
    f2 st[PF::S];
#pragma unroll
    for (int i = 0; i < PF::S; ++i) st[i] = 0;
    if (P1S && active) {
        const int64_t c0 = (2 * k) * (int64_t)CL < slen ? (2 * k) * (int64_t)CL : slen;
        const int64_t c1 = (2 * k + 1) * (int64_t)CL < slen ? (2 * k + 1) * (int64_t)CL : slen;
        if constexpr (Q == 0) {
#pragma unroll
            for (int c = 0; c < d; ++c) st[PF::top_off(1) + c] = f2_pack(raw[c0 * d + c] - x0[c], raw[c1 * d + c] - x0[c]);
        } else {
            const int c = dig[0];
            PF::scal(st, 1) = f2_pack(raw[c0 * d + c] - x0[0], raw[c1 * d + c] - x0[0]);
        }
    }
    __syncthreads();
    if (tid == 0) asm volatile("mbarrier.inval.shared::cta.b64 [%0];" ::"r"(smem_addr(bar)) : "memory");
    phase(2);
    // 4. the fold: CL Horner steps, barrier-free
    if (active) {
        const f2* base = tab + (size_t)k * RS;
        const size_t stride = (size_t)UP * RS;
        if constexpr (PF::PREFETCH) {
            typename PF::Ops oa, ob;
            PF::load(oa, base, dig);
            int i = 0;
            for (; i + 2 <= CL; i += 2) {  // operands of the next step are in flight during this one
                PF::load(ob, base + (size_t)(i + 1) * stride, dig);
                PF::step(st, oa);
                if (i + 2 < CL) PF::load(oa, base + (size_t)(i + 2) * stride, dig);
                PF::step(st, ob);
            }
            if (i < CL) PF::step(st, oa);
        } else {
#pragma unroll 2
            for (int i = 0; i < CL; ++i) {
                typename PF::Ops o;
                PF::load(o, base + (size_t)i * stride, dig);
                PF::step(st, o);
            }
        }
    }
    phase(3);
    __syncthreads();  // table and staging are dead: reuse them for the combine
    phase(4);
    // 5. combine the U chunks
    pair_combine_store<PF, CLUSTER, P1S>(st, active, k, pre, p10v, g, rowid, b, out, smem_raw, phase);
}

}  // namespace sigk
