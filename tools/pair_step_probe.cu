// Microbenchmark: issue rate of the pair-fold Horner step (pair_kernel.cuh,
// PairFold::step) with operands streamed from a shared-memory table exactly as
// the kernel's fold loop does (software-pipelined loads), at 1..4 warps per SM
// sub-partition. Reports FMA-pipe utilisation = 2 * ops / (4 SMSP * cycles).
//   nvcc -O3 -std=c++17 -gencode arch=compute_100a,code=sm_100a -I paper_2501_08455_b200/csrc tools/pair_step_probe.cu -o tools/pair_step_probe
#include <cstdio>
#include <cuda_runtime.h>

#include <type_traits>

#include "pair_kernel.cuh"

using namespace sigk;

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


// PF: 0 plain loop, 1 software-pipelined loads, 2 operands in registers only (no table loads)
// LEAN: 0 table mode, 1 lean, 2 position table (PosFold)
template <int LEANM>
struct FoldSel;
template <int D, int N, int Q, int LEANM, int PF>
__global__ void __launch_bounds__(512) stepk(float* sink, int steps, int units) {
    using F = std::conditional_t<LEANM == 2, PosFold<D, N, Q>, PairFold<D, N, Q, LEANM == 1>>;
    extern __shared__ __align__(16) unsigned char sm[];
    f2* tab = reinterpret_cast<f2*>(sm);
    constexpr int ROWS = 32;
    for (int i = threadIdx.x; i < ROWS * units * F::RS; i += blockDim.x)
        tab[i] = f2_pack(1e-3f * (i % 7), -1e-3f * (i % 5));
    __syncthreads();
    const int k = threadIdx.x / F::P, pre = threadIdx.x % F::P;
    int dig[F::QS];
    for (int q = 0; q < F::QS; ++q) dig[q] = (Q > 0) ? (pre / ipow(D, Q > 0 ? Q - 1 - q : 0)) % D : 0;
    f2 st[F::S];
    for (int i = 0; i < F::S; ++i) st[i] = f2_pack(1e-3f * i, 2e-3f * i);
    const f2* base = tab + (size_t)(k % units) * F::RS;
    const size_t stride = (size_t)units * F::RS;
    if constexpr (PF == 2) {
        typename F::Ops o;
        F::load(o, base, dig);
#pragma unroll 1
        for (int i = 0; i < steps; ++i) {
            F::step(st, o);
            // loop-carried: the operands cannot be hoisted as constants
            if constexpr (LEANM == 2) o.v[0] = st[3];
            else o.v[0][0] = st[3];
        }
    } else if constexpr (PF == 1) {
        typename F::Ops oa, ob;
        F::load(oa, base, dig);
        for (int i = 0; i + 2 <= steps; i += 2) {
            F::load(ob, base + (size_t)((i + 1) % ROWS) * stride, dig);
            F::step(st, oa);
            F::load(oa, base + (size_t)((i + 2) % ROWS) * stride, dig);
            F::step(st, ob);
        }
    } else {
#pragma unroll 2
        for (int i = 0; i < steps; ++i) {
            typename F::Ops o;
            F::load(o, base + (size_t)(i % ROWS) * stride, dig);
            F::step(st, o);
        }
    }
    float acc = 0.f;
    for (int i = 0; i < F::S; ++i) {
        float lo, hi;
        f2_unpack(st[i], lo, hi);
        acc += lo + hi;
    }
    sink[blockIdx.x * blockDim.x + threadIdx.x] = acc;
}

template <int D, int N, int Q, int LEAN, int PF>
void run(const char* name, float* sink) {
    using F = std::conditional_t<LEAN == 2, PosFold<D, N, Q>, PairFold<D, N, Q, LEAN == 1>>;
    int sms = 0, clk = 0;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, 0);
    for (int w : {1, 2, 3, 4}) {
        const int units = 128 * w / F::P;  // pair-units per CTA: one CTA of 128*w threads per SM
        const int threads = units * F::P;
        const size_t smem = 32ull * units * F::RS * 8;
        cudaFuncSetAttribute(stepk<D, N, Q, LEAN, PF>, cudaFuncAttributeMaxDynamicSharedMemorySize, 200000);
        const int steps = 4000;
        cudaEvent_t e0, e1;
        cudaEventCreate(&e0);
        cudaEventCreate(&e1);
        stepk<D, N, Q, LEAN, PF><<<sms, threads, smem>>>(sink, 10, units);
        cudaEventRecord(e0);
        stepk<D, N, Q, LEAN, PF><<<sms, threads, smem>>>(sink, steps, units);
        cudaEventRecord(e1);
        cudaEventSynchronize(e1);
        float ms;
        cudaEventElapsedTime(&ms, e0, e1);
        cudaGetLastError();
        const double pipe = 2.0 * threads * (double)steps * F::ops_per_step() / 32.0;  // executed warp-pipe cycles per SM
        const double util = pipe / 4.0 / (ms * 1e-3 * clk * 1e3);
        printf("%s warps/SMSP=%.2f threads=%d  executed FMA-pipe util (at max clk)=%.3f  (%.2f ms) %s\n", name, threads / 128.0,
               threads, util, ms, cudaGetErrorString(cudaGetLastError()));
    }
}

int main() {
    float* sink;
    cudaMalloc(&sink, 148 * 1024 * sizeof(float));
    run<5, 4, 2, 1, 2>("d5N4Q2 lean regs    ", sink);
    run<5, 4, 2, 1, 1>("d5N4Q2 lean prefetch", sink);
    run<4, 4, 2, 1, 2>("d4N4Q2 lean regs    ", sink);
    run<4, 4, 2, 1, 1>("d4N4Q2 lean prefetch", sink);
    run<6, 3, 1, 1, 2>("d6N3Q1 lean regs    ", sink);
    run<8, 3, 2, 1, 2>("d8N3Q2 lean regs    ", sink);
    return 0;
}
