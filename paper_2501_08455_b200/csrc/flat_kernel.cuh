// Flat kernel: for variants whose unit (d^Q threads) is larger than a CTA —
// C4 (d=10, N=5: Q=3, 1000 threads per path). Whole paths are units (no
// sequence chunking, so no merge and no HBM intermediates); the B * d^Q
// threads are cut into small CTAs of NT consecutive prefixes, so the grid
// load-balances across the 148 SMs at the granularity of one warp. A CTA
// touches at most two paths; it produces the increments of both into its own
// shared-memory table each tile. The final slices are staged level by level
// through shared memory so the stores to the (B, D) output are coalesced.
#pragma once

#include "fold.cuh"

namespace sigk {

template <typename Real, int DIM, int DEPTH, int Q, int NT, int T>
struct FlatGeom {
    using SF = SliceFold<Real, DIM, DEPTH, Q>;
    static constexpr int NU = SF::P >= NT ? 2 : NT / SF::P + 2;  // units one CTA touches
    static constexpr int ENT = NU * T * DIM;
    static constexpr int EPT = (ENT + NT - 1) / NT;
    static constexpr size_t tab_elems = 2ull * T * NU * SF::TAB;
    static constexpr size_t stage_elems = (size_t)NT * ipow(DIM, DEPTH - Q);
    static constexpr size_t smem = sizeof(Real) * (tab_elems > stage_elems ? tab_elems : stage_elems);
};

template <typename SF, int n, typename Real>
__device__ __forceinline__ void flat_store_levels(Real (&st)[SF::S], Real* __restrict__ stage, int pre, int64_t g0,
                                                  int nt, Real* __restrict__ out) {
    constexpr int d = SF::d, Q = SF::QQ, P = SF::P;
    constexpr int D = level_off(d, SF::N);
    if constexpr (n <= SF::N) {
        if constexpr (n >= SF::NMIN) {
            constexpr int sz = ipow(d, n - Q);
            constexpr int o = SF::top_off(n);
#pragma unroll
            for (int J = 0; J < sz; ++J) stage[threadIdx.x * sz + J] = st[o + J];
            __syncthreads();
            // lanes g0 .. g0+nt-1 cover prefixes of <= 2 paths; each run is contiguous in HBM
            for (int i = threadIdx.x; i < nt * sz; i += blockDim.x) {
                const int lane = i / sz, J = i - lane * sz;
                const int64_t g = g0 + lane;
                const int64_t b = g / P;
                const int p = (int)(g - b * P);
                out[b * D + level_off(d, n - 1) + (int64_t)p * sz + J] = stage[i];
            }
            __syncthreads();
        } else {
            constexpr int tail = ipow(d, Q - n);
            if ((int)threadIdx.x < nt && pre % tail == 0) {
                const int64_t b = (g0 + threadIdx.x) / P;
                out[b * D + level_off(d, n - 1) + pre / tail] = st[n - 1];
            }
        }
        flat_store_levels<SF, n + 1>(st, stage, pre, g0, nt, out);
    }
}

template <typename Real, int DIM, int DEPTH, int Q, int NT, int T, int MINB>
__global__ void __launch_bounds__(NT, MINB) flat_kernel(const Real* __restrict__ X, int64_t B, int64_t L,
                                                        Real* __restrict__ out) {
    using G = FlatGeom<Real, DIM, DEPTH, Q, NT, T>;
    using SF = typename G::SF;
    constexpr int d = DIM, P = SF::P, TAB = SF::TAB, NU = G::NU, ENT = G::ENT, EPT = G::EPT;

    extern __shared__ __align__(16) unsigned char smem_raw[];
    Real* tab = reinterpret_cast<Real*>(smem_raw);  // [2][T][NU][TAB], later the store stage

    const int64_t M = L - 1;
    const int64_t lanes = B * (int64_t)P;
    const int64_t g0 = (int64_t)blockIdx.x * NT;
    const int64_t u0 = g0 / P;
    const int64_t g = g0 + threadIdx.x;
    const bool active = g < lanes;
    const int pre = (int)(g % P);
    const int uu = (int)(g / P - u0);
    const int nt = (lanes - g0) < NT ? (int)(lanes - g0) : NT;

    int dig[SF::QS];
    prefix_digits<SF>(pre, dig);
    Real st[SF::S];
#pragma unroll
    for (int i = 0; i < SF::S; ++i) st[i] = Real(0);
    pdl_trigger();

    // producer entries e = (unit ue, step s, channel c), c fastest: per-thread
    // offsets (from the CTA's first path, relative to the tile start) are fixed
    // for the whole kernel; -1 marks entries past the batch
    const Real* __restrict__ xc = X + u0 * L * d;
    int eoff[EPT];
#pragma unroll
    for (int i = 0; i < EPT; ++i) {
        const int e = threadIdx.x + i * NT;
        const int c = e % d, s = (e / d) % T, ue = e / (d * T);
        eoff[i] = (e < ENT && (u0 + ue) < B) ? (int)((ue * L + s) * d + c) : -1;
    }
    Real xa[EPT], xb[EPT];
    auto load = [&](int tile) {
#pragma unroll
        for (int i = 0; i < EPT; ++i) {
            const int s = ((threadIdx.x + i * NT) / d) % T;
            const bool ok = eoff[i] >= 0 && (tile * T + s < M);
            const Real* p = xc + eoff[i] + (int64_t)tile * T * d;
            xa[i] = ok ? __ldg(p) : Real(0);
            xb[i] = ok ? __ldg(p + d) : Real(0);
        }
    };
    auto store = [&](int buf) {
#pragma unroll
        for (int i = 0; i < EPT; ++i) {
            const int e = threadIdx.x + i * NT;
            if (e < ENT) {
                const int c = e % d, s = (e / d) % T, ue = e / (d * T);
                produce_entry<SF>(tab + (((size_t)buf * T + s) * NU + ue) * TAB, c, xb[i] - xa[i]);
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
        consume_tile<SF, T, false>(st, tab + (size_t)buf * T * NU * TAB + (size_t)uu * TAB, (size_t)NU * TAB, dig);
    }
    pdl_wait();
    __syncthreads();
    if (!active) {
#pragma unroll
        for (int i = 0; i < SF::S; ++i) st[i] = Real(0);
    }
    flat_store_levels<SF, 1>(st, tab, pre, g0, nt, out);
}

}  // namespace sigk
