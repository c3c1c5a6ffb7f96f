// Position-table fold (pair family, FP32x2): the Horner step of PairFold
// (pair_kernel.cuh; reference sig_core.hpp:72-114) with
// the level-1 state and the first stage of every level's chain read from a
// table instead of computed per thread. Used by ppair_kernel.cuh, measured
// in isolation by tools/pair_step_probe.cu.
#pragma once

#include "pair_kernel.cuh"

namespace sigk {
// Position-table variant of PairFold (P1S chunk starts, Q >= 1). Since a
// chunk folds from A = (1, X[s_j] - X[0], 0, ...), T_1 at any step is just the
// current point relative to X[0]. The table therefore carries, per (step,
// pair-unit, channel c), besides δ[c] the chain starts of every level n >= 2
//     a_n[c] = (X[t][c] - X[0][c] + δ[c]/n) / (n-1)
// (the 1/(n-1) is the scaling the next Horner stage would apply), so a thread
// neither keeps T_1 nor forms the level starts or their first scaling:
// d=5, N=4, Q=2 drops from 45 to 39 FFMA2-class ops per step (credited work:
// 38.8) for N-1 more shared-memory pair loads. T_1 is restored from the
// points after the fold (restore_t1).
template <int DIM, int DEPTH, int Q>
struct PosFold {
    static_assert(Q >= 1 && Q < DEPTH, "position mode needs a prefix digit");
    static constexpr int d = DIM, N = DEPTH, QQ = Q;
    static constexpr bool LEAN = true;
    static constexpr int P = ipow(d, Q);
    static constexpr int NLOW = Q > 1 ? Q - 1 : 0;
    static constexpr int NMIN = Q > 1 ? Q : 1;
    __host__ __device__ static constexpr int top_off(int n) {
        int o = NLOW;
        for (int m = NMIN; m < n; ++m) o += ipow(d, m - Q);
        return o;
    }
    static constexpr int S = top_off(N + 1);
    static constexpr int FJ = ipow(d, N - Q);
    static constexpr int RP = (d % 2) ? d + 1 : d;
    static constexpr int NR = N;          // row 0: δ; rows n-1 (n = 2..N): a_n
    static constexpr int RS = NR * RP;
    static constexpr int QS = Q;
    static constexpr bool POS = true;

    __host__ __device__ static constexpr int ops_per_step() {
        int ops = 0;
        for (int n = 2; n <= N; ++n) {
            if (n > Q) {
                ops += Q - 1;                                        // digit chain k = 2..Q
                for (int k = 3; k <= Q; ++k) ops += (n - k + 1 > 1);  // their scalings
                ops += (Q >= 2 && n - Q > 1) ? 1 : 0;                // stage Q+1 prescale
                for (int k = Q + 1; k <= n; ++k) ops += ipow(d, k - Q);
                for (int k = Q + 2; k <= n - 1; ++k) ops += (n - k + 1 > 1) ? ipow(d, k - Q - 1) : 0;
            } else {
                ops += n - 1;
                for (int k = 3; k <= n - 1; ++k) ops += (n - k + 1 > 1);
            }
        }
        return ops;
    }
    __host__ __device__ static constexpr int loads_per_step() { return (d + 1) / 2 + (Q - 1) + (N - 1); }

    struct Ops {
        f2 v[d];         // δ[c]
        f2 a[N + 1];     // a[n] = a_n[p1], n = 2..N
        f2 g[QS + 1];    // g[k] = δ[p_k], k = 2..Q
    };

    __device__ __forceinline__ static f2& scal(f2 (&st)[S], int k) { return k < Q ? st[k - 1] : st[top_off(Q)]; }

    __device__ __forceinline__ static void load(Ops& o, const f2* __restrict__ row, const int (&dig)[QS]) {
#pragma unroll
        for (int c = 0; c + 1 < d; c += 2) {
            const ulonglong2 v = *reinterpret_cast<const ulonglong2*>(row + c);
            o.v[c] = v.x;
            o.v[c + 1] = v.y;
        }
        if constexpr (d % 2) o.v[d - 1] = row[d - 1];
#pragma unroll
        for (int n = 2; n <= N; ++n) o.a[n] = row[(n - 1) * RP + dig[0]];
#pragma unroll
        for (int k = 2; k <= Q; ++k) o.g[k] = row[dig[k - 1]];
    }

    template <int n>
    __device__ __forceinline__ static void level(f2 (&st)[S], const Ops& o) {
        if constexpr (n == 1) {
            // T_1 is not tracked (restore_t1)
        } else if constexpr (n > Q) {
            constexpr int F = n - Q;
            f2 u = o.a[n];  // (T_1 + δ[p1]/n) / (n-1)
#pragma unroll
            for (int k = 2; k <= Q; ++k) {
                if (k >= 3 && n - k + 1 > 1) u = fmul2(u, f2_bcast(1.0f / float(n - k + 1)));
                u = ffma2(u, o.g[k], scal(st, k));
            }
            if constexpr (F == 1) {
                constexpr int ot = top_off(n);
#pragma unroll
                for (int c = 0; c < d; ++c) st[ot + c] = ffma2(u, o.v[c], st[ot + c]);
            } else {
                constexpr int m = n - Q;
                const f2 us = (Q >= 2 && m > 1) ? fmul2(u, f2_bcast(1.0f / float(m))) : u;
                f2 ua[ipow(d, F - 1)];
                {
                    constexpr int o1 = top_off(Q + 1);
#pragma unroll
                    for (int c = 0; c < d; ++c) ua[c] = ffma2(us, o.v[c], st[o1 + c]);
                }
                stages<n, Q + 2>(st, o, ua);
                constexpr int ot = top_off(n);
#pragma unroll
                for (int J = 0; J < ipow(d, F); ++J) st[ot + J] = ffma2(ua[J / d], o.v[J % d], st[ot + J]);
            }
        } else {  // scalar level 2 <= n <= Q
            f2 u = o.a[n];
#pragma unroll
            for (int k = 2; k <= n - 1; ++k) {
                if (k >= 3 && n - k + 1 > 1) u = fmul2(u, f2_bcast(1.0f / float(n - k + 1)));
                u = ffma2(u, o.g[k], scal(st, k));
            }
            scal(st, n) = ffma2(u, o.g[n], scal(st, n));
        }
    }

    template <int n, int k, int UA>
    __device__ __forceinline__ static void stages(f2 (&st)[S], const Ops& o, f2 (&ua)[UA]) {
        if constexpr (k <= n - 1) {
            constexpr int sz = ipow(d, k - Q);
            constexpr int ok = top_off(k);
            constexpr int m = n - k + 1;
            if constexpr (m > 1) {
#pragma unroll
                for (int J = 0; J < sz / d; ++J) ua[J] = fmul2(ua[J], f2_bcast(1.0f / float(m)));
            }
#pragma unroll
            for (int J = sz - 1; J >= 0; --J) ua[J] = ffma2(ua[J / d], o.v[J % d], st[ok + J]);
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

}  // namespace sigk
