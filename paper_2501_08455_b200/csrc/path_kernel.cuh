// Path kernel: one CTA per path, the path's chunks as units inside the CTA.
//
// Used for every variant whose unit (d^Q threads) fits in a CTA: C1, C2, C3
// and C5 of BASELINE.json. The CTA holds U units (chunks of CL = ceil(M/U)
// steps) x P = d^Q threads; each thread folds its prefix slice of its chunk in
// registers (fold.cuh). Increments are produced per tile of T steps into a
// double-buffered shared-memory table: the producer loads of tile t+1 are
// issued before the Horner steps of tile t, so HBM latency hides behind FFMA
// work, and one barrier per tile suffices. When the fold ends the U chunk
// signatures are staged into shared memory (reusing the table space) and
// combined by the per-degree prefix scan over chunks (merge.cuh: N fixed-order
// phases of Chen-identity contributions, not a tree); the path's signature is
// then written to HBM with coalesced stores. Nothing but X is read and nothing
// but the final (B, D) rows is written: no intermediates touch HBM.
#pragma once

#include "fold.cuh"
#include "merge.cuh"

namespace sigk {

template <typename Real, int DIM, int DEPTH, int Q>
struct PathGeom {
    using SF = SliceFold<Real, DIM, DEPTH, Q>;
    static constexpr int D = level_off(DIM, DEPTH);
    // Q == 1: a thread produces T consecutive steps of its own channel (T+1 loads);
    // Q == 0: the thread is the whole unit and produces every channel ((T+1)*d loads);
    // Q >= 2: entries (step, channel) are dealt round-robin over the unit (2 loads each).
    static constexpr bool RUN1 = Q == 1;
    static constexpr bool RUN0 = Q == 0;
    __host__ __device__ static constexpr int ept(int T) { return (T * DIM + SF::P - 1) / SF::P; }
    __host__ __device__ static constexpr int nx(int T) { return RUN1 ? T + 1 : RUN0 ? (T + 1) * DIM : 2 * ept(T); }
    // steps per tile: 8, fewer when the whole-unit (Q == 0) prefetch would cost too many registers
    static constexpr int tile_steps() {
        if (!RUN0) return 8;
        int t = 24 / DIM - 1;
        return t < 1 ? 1 : (t > 8 ? 8 : t);
    }
    __host__ static size_t smem_bytes(int T, int U) {
        const size_t tab = 2ull * T * U * SF::TAB, comb = combine_smem_elems<SF>(U);
        return sizeof(Real) * (tab > comb ? tab : comb);
    }
};

// X: (B, L, d); out: (B, D). grid = B, block = U * d^Q threads.
template <typename Real, int DIM, int DEPTH, int Q, int NTMAX, int T, int MINB, bool PIPE>
__global__ void __launch_bounds__(NTMAX, MINB) path_kernel(const Real* __restrict__ X, int64_t L, int U, int CL,
                                                           Real* __restrict__ out, long long* __restrict__ phases) {
    using G = PathGeom<Real, DIM, DEPTH, Q>;
    using SF = typename G::SF;
    constexpr int d = DIM;
    constexpr int P = SF::P;
    constexpr int TAB = SF::TAB;
    constexpr int D = G::D;
    constexpr bool RUN1 = G::RUN1, RUN0 = G::RUN0;
    constexpr int EPT = G::ept(T);

    extern __shared__ __align__(16) unsigned char smem_raw[];
    Real* tab = reinterpret_cast<Real*>(smem_raw);  // [2][T][U][TAB], later sig[U][D]

    const int64_t b = blockIdx.x;
    const int64_t M = L - 1;
    const int tid = threadIdx.x;
    const int u = tid / P;
    const int tl = tid - u * P;
    const int64_t ustart = (int64_t)u * CL;
    const int64_t rem = M - ustart;  // real steps of this chunk: clamp(rem, 0, CL)
    const int lim = rem <= 0 ? 0 : (rem < CL ? (int)rem : CL);
    const Real* __restrict__ xu = X + (b * L + ustart) * d;              // chunk's first point

    int dig[SF::QS];
    prefix_digits<SF>(tl, dig);
    Real st[SF::S];
#pragma unroll
    for (int i = 0; i < SF::S; ++i) st[i] = Real(0);

    constexpr int NX = G::nx(T);
    Real xr[NX];
    // Q >= 2 producer geometry: thread tl handles channel c0 at steps s0, s0 + P/d, ...
    const int s0 = tl / d, c0 = tl - (tl / d) * d;
    const Real* __restrict__ xg = xu + (int64_t)s0 * d + c0;
    auto load = [&](int tile) {
        const int j0 = tile * T;
        if constexpr (RUN1) {  // channel c = tl, points j0 .. j0+T of the chunk
#pragma unroll
            for (int i = 0; i <= T; ++i) xr[i] = (j0 + i <= lim) ? __ldg(xu + (int64_t)(j0 + i) * d + tl) : Real(0);
        } else if constexpr (RUN0) {  // all channels, points j0 .. j0+T (contiguous)
#pragma unroll
            for (int i = 0; i < (T + 1) * d; ++i) xr[i] = (j0 + i / d <= lim) ? __ldg(xu + (int64_t)j0 * d + i) : Real(0);
        } else {  // entry i: step s0 + i*P/d of channel c0 (P is a multiple of d)
#pragma unroll
            for (int i = 0; i < EPT; ++i) {
                const int s = s0 + i * (P / d);
                const bool ok = (s < T) && (j0 + s < lim);
                const Real* p = xg + (int64_t)j0 * d + i * P;
                xr[2 * i] = ok ? __ldg(p) : Real(0);
                xr[2 * i + 1] = ok ? __ldg(p + d) : Real(0);
            }
        }
    };
    auto store = [&](int buf, int tile) {
        Real* base = tab + (size_t)buf * T * U * TAB;
        if constexpr (RUN1) {
#pragma unroll
            for (int i = 0; i < T; ++i) {
                const Real dl = (tile * T + i < lim) ? xr[i + 1] - xr[i] : Real(0);
                produce_entry<SF>(base + ((size_t)i * U + u) * TAB, tl, dl);
            }
        } else if constexpr (RUN0) {
#pragma unroll
            for (int i = 0; i < T; ++i) {
                const bool ok = tile * T + i < lim;
#pragma unroll
                for (int c = 0; c < d; ++c)
                    produce_entry<SF>(base + ((size_t)i * U + u) * TAB, c, ok ? xr[(i + 1) * d + c] - xr[i * d + c] : Real(0));
            }
        } else {
#pragma unroll
            for (int i = 0; i < EPT; ++i) {
                const int s = s0 + i * (P / d);
                if (s < T) produce_entry<SF>(base + (size_t)s * U * TAB + (size_t)u * TAB, c0, xr[2 * i + 1] - xr[2 * i]);
            }
        }
    };

    // optional phase timestamps (SM clock) of thread 0, for tools/probe.py
    auto phase = [&](int k) {
        if (phases != nullptr && tid == 0) phases[b * 8 + k] = clock64();
    };
    phase(0);
    pdl_trigger();  // the next launch may start folding on free SMs now
    const int ntiles = (CL + T - 1) / T;
    load(0);
    for (int tile = 0; tile < ntiles; ++tile) {
        const int buf = tile & 1;
        store(buf, tile);
        __syncthreads();
        if (tile == 0) phase(1);
        if (tile + 1 < ntiles) load(tile + 1);
        consume_tile<SF, T, PIPE>(st, tab + (size_t)buf * T * U * TAB + (size_t)u * TAB, (size_t)U * TAB, dig);
    }
    phase(2);
    pdl_wait();       // the previous launch has completed: our output writes are ordered after its
    __syncthreads();  // the table is dead; reuse it for the chunk combine
    phase(3);
    combine_chunks<SF>(st, u, tl, U, tab, out + b * D, phase);
    phase(7);
}

}  // namespace sigk
