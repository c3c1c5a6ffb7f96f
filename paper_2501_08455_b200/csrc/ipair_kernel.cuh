// Inner-pair fold kernel ("pflat" family): the sm_100a fp32 fold for even d
// with packed FP32x2 arithmetic along the LAST tensor index.
//
// Same math as fold.cuh / pair_kernel.cuh (reference detail::sequential_forward,
// /root/reference/proj/include/sigkit/detail/sig_core.hpp:116-147; Horner form
// of exp_into :72-90 + fold_step :92-114). A thread owns
// the prefix slice `pre` (Q leading digits) of ONE path, as in fold.cuh, but
// keeps every vector level T_n[pre, :] as pairs of adjacent last-index
// entries. Each vector stage of the Horner step is then
//     T[J, 2c'..2c'+1] += ua[J] * (δ[2c'], δ[2c'+1])
// i.e. one FFMA2 whose first operand is a broadcast scalar (SASS "R.F32")
// shared by the d/2 consecutive FFMA2 of row J, and whose second operand is a
// δ pair straight from the shared-memory table — no chunk pairing, so the
// state costs no more registers than the scalar fold. Used for large d^N
// where whole paths are the units (BASELINE C4 d=10 N=5, C5 d=8 N=4): no
// sequence chunking, no combine; CTAs of NT consecutive (path, slice) lanes.
#pragma once

#include "pair_kernel.cuh"

namespace sigk {

template <int DIM, int DEPTH, int Q>
struct IPairFold {
    static_assert(DIM % 2 == 0, "inner pairs need an even dimension");
    static_assert(Q >= 1 && Q < DEPTH, "prefix length");
    static constexpr int d = DIM, N = DEPTH, QQ = Q, H = DIM / 2;
    static constexpr int P = ipow(d, Q);  // slices per path
    // pair offset of vector level n (n = Q+1..N)
    __host__ __device__ static constexpr int vo(int n) {
        int o = 0;
        for (int m = Q + 1; m < n; ++m) o += ipow(d, m - Q) / 2;
        return o;
    }
    static constexpr int NVP = vo(N + 1);  // vector state pairs
    static constexpr int FJ = ipow(d, N - Q);
    // FMA-pipe cycles per thread per step (FFMA2 = 2, scalar FFMA/FMUL = 1)
    __host__ __device__ static constexpr int pipe_cycles() {
        int c = 0;
        for (int n = 1; n <= N; ++n) {
            if (n > Q) {
                c += Q;                                            // scalar chain
                for (int k = 2; k <= Q; ++k) c += (n - k + 1 > 1);  // chain scalings
                c += (n - Q > 1);                                  // stage Q+1 prescale
                for (int k = Q + 1; k <= n; ++k) c += ipow(d, k - Q);  // FFMA2: 2 cycles per pair
                for (int k = Q + 2; k <= n - 1; ++k) c += (n - k + 1 > 1) ? ipow(d, k - Q - 1) : 0;  // FMUL2 prescale
            } else {
                c += n;
                for (int k = 2; k <= n - 1; ++k) c += (n - k + 1 > 1);
            }
        }
        return c;
    }

    struct State {
        float sc[Q];     // T_1[p1], ..., T_Q[p1..pQ]
        f2 v[NVP];       // vector levels Q+1..N, pairs along the last index
    };
    struct Ops {
        f2 dv[H];        // δ pairs
        float g[Q];      // δ[p_k]
    };

    __device__ __forceinline__ static float lo(f2 x) {
        float a, b;
        f2_unpack(x, a, b);
        return a;
    }
    __device__ __forceinline__ static float hi(f2 x) {
        float a, b;
        f2_unpack(x, a, b);
        return b;
    }
    template <int SZ>
    __device__ __forceinline__ static float elem(const f2 (&u)[SZ], int J) {
        return (J & 1) ? hi(u[J >> 1]) : lo(u[J >> 1]);
    }

    __device__ __forceinline__ static void load(Ops& o, const float* __restrict__ row, const int (&dig)[Q]) {
#pragma unroll
        for (int c = 0; c + 3 < d; c += 4) {
            const ulonglong2 v = *reinterpret_cast<const ulonglong2*>(row + c);
            o.dv[c / 2] = v.x;
            o.dv[c / 2 + 1] = v.y;
        }
        if constexpr (d % 4) o.dv[H - 1] = *reinterpret_cast<const f2*>(row + d - 2);
#pragma unroll
        for (int k = 0; k < Q; ++k) o.g[k] = row[dig[k]];
    }

    // u * δ[p_k] / m + T
    __device__ __forceinline__ static float chain(float u, const Ops& o, int k, int m, float T) {
        if (m > 1) u *= 1.0f / float(m);
        return fmaf(u, o.g[k - 1], T);
    }

    template <int n>
    __device__ __forceinline__ static void level(State& s, const Ops& o) {
        constexpr float inv_n = 1.0f / float(n);
        if constexpr (n > Q) {
            constexpr int F = n - Q;
            float u = fmaf(o.g[0], inv_n, s.sc[0]);  // δ[p1]/n + T_1[p1]
#pragma unroll
            for (int k = 2; k <= Q; ++k) u = chain(u, o, k, n - k + 1, s.sc[k - 1]);
            if constexpr (F == 1) {
                constexpr int ot = vo(n);
#pragma unroll
                for (int cp = 0; cp < H; ++cp) s.v[ot + cp] = ffma2(f2_bcast(u), o.dv[cp], s.v[ot + cp]);
            } else {
                constexpr int m1 = n - Q;
                const float us = m1 > 1 ? u * (1.0f / float(m1)) : u;
                f2 ua[ipow(d, F - 1) / 2];
                {
                    constexpr int o1 = vo(Q + 1);
#pragma unroll
                    for (int cp = 0; cp < H; ++cp) ua[cp] = ffma2(f2_bcast(us), o.dv[cp], s.v[o1 + cp]);
                }
                stages<n, Q + 2>(s, o, ua);
                constexpr int ot = vo(n);
                constexpr int rows = ipow(d, F - 1);
#pragma unroll
                for (int J = 0; J < rows; ++J) {
                    const float a = elem(ua, J);
#pragma unroll
                    for (int cp = 0; cp < H; ++cp) s.v[ot + J * H + cp] = ffma2(f2_bcast(a), o.dv[cp], s.v[ot + J * H + cp]);
                }
            }
        } else {  // scalar level n <= Q
            if constexpr (n == 1) {
                s.sc[0] += o.g[0];
            } else {
                float u = fmaf(o.g[0], inv_n, s.sc[0]);
#pragma unroll
                for (int k = 2; k <= n - 1; ++k) u = chain(u, o, k, n - k + 1, s.sc[k - 1]);
                s.sc[n - 1] = fmaf(u, o.g[n - 1], s.sc[n - 1]);
            }
        }
    }

    // stage k of level n: ua (d^(k-Q-1) values) -> d^(k-Q) values, in place
    template <int n, int k, int UA>
    __device__ __forceinline__ static void stages(State& s, const Ops& o, f2 (&ua)[UA]) {
        if constexpr (k <= n - 1) {
            constexpr int rows = ipow(d, k - Q - 1);  // values before the stage
            constexpr int ok = vo(k);
            constexpr int m = n - k + 1;
            if constexpr (m > 1) {
#pragma unroll
                for (int i = 0; i < rows / 2; ++i) ua[i] = fmul2(ua[i], f2_bcast(1.0f / float(m)));
            }
#pragma unroll
            for (int J = rows - 1; J >= 0; --J) {
                const float a = elem(ua, J);  // read before the row overwrites its pair
#pragma unroll
                for (int cp = 0; cp < H; ++cp) ua[J * H + cp] = ffma2(f2_bcast(a), o.dv[cp], s.v[ok + J * H + cp]);
            }
            stages<n, k + 1>(s, o, ua);
        }
    }

    template <int n>
    __device__ __forceinline__ static void levels_desc(State& s, const Ops& o) {
        if constexpr (n >= 1) {
            level<n>(s, o);
            levels_desc<n - 1>(s, o);
        }
    }
    __device__ __forceinline__ static void step(State& s, const Ops& o) { levels_desc<N>(s, o); }
};

template <int DIM, int DEPTH, int Q, int NT, int T>
struct IPairGeom {
    using F = IPairFold<DIM, DEPTH, Q>;
    static constexpr int RW = round_up(DIM, 4);                       // floats per table row (16-byte rows)
    static constexpr int NU = F::P >= NT ? 2 : NT / F::P + 2;         // paths one CTA touches
    static constexpr int ENT = NU * T * DIM;                          // producer entries per tile
    static constexpr int EPT = (ENT + NT - 1) / NT;
    static constexpr size_t tab_floats = 2ull * T * NU * RW;
    static constexpr size_t stage_floats = (size_t)NT * F::FJ;
    static constexpr size_t smem = 4 * (tab_floats > stage_floats ? tab_floats : stage_floats);
};

// State of each lane -> out, level by level through a shared-memory stage so
// the stores of consecutive lanes (consecutive slices of <= NU paths) are
// contiguous runs in HBM.
template <typename F, int n>
__device__ __forceinline__ void ipair_store_levels(const typename F::State& s, float* __restrict__ stage, int pre,
                                                   int64_t g0, int nt, float* __restrict__ out) {
    constexpr int d = F::d, Q = F::QQ, P = F::P;
    constexpr int D = level_off(d, F::N);
    if constexpr (n <= F::N) {
        if constexpr (n > Q || n == Q) {
            constexpr int sz = ipow(d, n - Q);
            if constexpr (n == Q) {
                stage[threadIdx.x] = s.sc[Q - 1];
            } else {
                constexpr int o = F::vo(n);
#pragma unroll
                for (int i = 0; i < sz / 2; ++i) {
                    float a, b;
                    f2_unpack(s.v[o + i], a, b);
                    stage[threadIdx.x * sz + 2 * i] = a;
                    stage[threadIdx.x * sz + 2 * i + 1] = b;
                }
            }
            __syncthreads();
            for (int i = threadIdx.x; i < nt * sz; i += blockDim.x) {
                const int lane = i / sz, J = i - lane * sz;
                const int64_t g = g0 + lane;
                const int64_t b = g / P;
                const int p = (int)(g - b * P);
                out[b * D + level_off(d, n - 1) + (int64_t)p * sz + J] = stage[i];
            }
            __syncthreads();
        } else {  // redundant prefix scalar T_n[p_1..p_n], n < Q: one writer each
            constexpr int tail = ipow(d, Q - n);
            if ((int)threadIdx.x < nt && pre % tail == 0) {
                const int64_t b = (g0 + threadIdx.x) / P;
                out[b * D + level_off(d, n - 1) + pre / tail] = s.sc[n - 1];
            }
        }
        ipair_store_levels<F, n + 1>(s, stage, pre, g0, nt, out);
    }
}

// X: (B, L, d) fp32 -> out (B, D). grid = ceil(B * P / NT) CTAs of NT lanes.
template <int DIM, int DEPTH, int Q, int NT, int T, int MINB>
__global__ void __launch_bounds__(NT, MINB) ipair_kernel(const float* __restrict__ X, int64_t B, int64_t L,
                                                         float* __restrict__ out) {
    using G = IPairGeom<DIM, DEPTH, Q, NT, T>;
    using F = typename G::F;
    constexpr int d = DIM, P = F::P, RW = G::RW, NU = G::NU, ENT = G::ENT, EPT = G::EPT;

    extern __shared__ __align__(16) unsigned char smem_raw[];
    float* tab = reinterpret_cast<float*>(smem_raw);  // [2][T][NU][RW], later the store stage

    const int64_t M = L - 1;
    const int64_t lanes = B * (int64_t)P;
    const int64_t g0 = (int64_t)blockIdx.x * NT;
    const int64_t u0 = g0 / P;
    const int64_t gl = g0 + threadIdx.x;
    const int pre = (int)(gl % P);
    const int uu = (int)(gl / P - u0);
    const int nt = (lanes - g0) < NT ? (int)(lanes - g0) : NT;

    int dig[Q];
#pragma unroll
    for (int k = 0; k < Q; ++k) dig[k] = (pre / ipow(d, Q - 1 - k)) % d;
    typename F::State s;
#pragma unroll
    for (int i = 0; i < Q; ++i) s.sc[i] = 0.f;
#pragma unroll
    for (int i = 0; i < F::NVP; ++i) s.v[i] = 0;
    pdl_trigger();

    // producer entries e = (path ue, step st, channel c), c fastest; per-thread
    // offsets relative to the tile start are fixed for the whole kernel
    const float* __restrict__ xc = X + u0 * L * d;
    int eoff[EPT];
#pragma unroll
    for (int i = 0; i < EPT; ++i) {
        const int e = threadIdx.x + i * NT;
        const int c = e % d, st = (e / d) % T, ue = e / (d * T);
        eoff[i] = (e < ENT && (u0 + ue) < B) ? (int)((ue * L + st) * d + c) : -1;
    }
    float xa[EPT], xb[EPT];
    auto load = [&](int tile) {
#pragma unroll
        for (int i = 0; i < EPT; ++i) {
            const int st = ((threadIdx.x + i * NT) / d) % T;
            const bool ok = eoff[i] >= 0 && (tile * T + st < M);
            const float* p = xc + eoff[i] + (int64_t)tile * T * d;
            xa[i] = ok ? __ldg(p) : 0.f;
            xb[i] = ok ? __ldg(p + d) : 0.f;
        }
    };
    auto store = [&](int buf) {
#pragma unroll
        for (int i = 0; i < EPT; ++i) {
            const int e = threadIdx.x + i * NT;
            if (e < ENT) {
                const int c = e % d, st = (e / d) % T, ue = e / (d * T);
                tab[(((size_t)buf * T + st) * NU + ue) * RW + c] = xb[i] - xa[i];
            }
        }
    };

    const int ntiles = (int)((M + T - 1) / T);
    load(0);
    for (int tile = 0; tile < ntiles; ++tile) {
        const int buf = tile & 1;
        store(buf);
        __syncthreads();
        if (tile + 1 < ntiles) load(tile + 1);
        const float* base = tab + (size_t)buf * T * NU * RW + (size_t)uu * RW;
#pragma unroll 2
        for (int i = 0; i < T; ++i) {
            typename F::Ops o;
            F::load(o, base + (size_t)i * NU * RW, dig);
            F::step(s, o);
        }
    }
    pdl_wait();
    __syncthreads();
    if (gl >= lanes) {
#pragma unroll
        for (int i = 0; i < Q; ++i) s.sc[i] = 0.f;
#pragma unroll
        for (int i = 0; i < F::NVP; ++i) s.v[i] = 0;
    }
    ipair_store_levels<F, 1>(s, tab, pre, g0, nt, out);
}

}  // namespace sigk
