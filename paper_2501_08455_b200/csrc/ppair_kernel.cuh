// Pipelined position-table pair kernel (fp32, packed FP32x2): the pair
// family's fold (pair_kernel.cuh) with
//  * the position-table step (pos_fold.cuh): T_1 and the first stage of every
//    level's Horner chain come from the table (d=5, N=4, Q=2: 39 FFMA2-class
//    ops per thread-step instead of 45, for 38.8 credited);
//  * a producer warp: it TMA-stages the segment's points, then builds the
//    table in tiles of TS steps into a double buffer (full/empty mbarrier
//    pairs), so the fold warps never stop for a table build and the table
//    needs 2 tiles of shared memory instead of the whole segment;
//  * the same chunk / segment combine as pair_kernel (pair_combine_store).
// Same math as the reference fold (sig_core.hpp:116-147) and Chen combine
// (tensor_algebra.cpp:80-102); chunk j folds from A = (1, X[s_j] - X[0], 0, ...).
#pragma once

#include "pos_fold.cuh"

namespace sigk {

__device__ __forceinline__ void mbar_arrive(uint64_t* bar) {
    asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_addr(bar)) : "memory");
}

// Shared memory: [2][TS][UP][RS] table pairs | raw points | 5 mbarriers.
template <int d, int N, int Q>
struct PPairLayout {
    using PF = PosFold<d, N, Q>;
    __host__ __device__ static constexpr size_t tiles_bytes(int TS, int UP) { return (size_t)2 * TS * UP * PF::RS * 8; }
    __host__ __device__ static constexpr size_t raw_off(int TS, int UP) { return tiles_bytes(TS, UP); }
    __host__ __device__ static constexpr size_t bar_off(int TS, int UP, int raw_floats) {
        return (raw_off(TS, UP) + (size_t)(raw_floats + 4) * 4 + 15) / 16 * 16;
    }
    __host__ __device__ static constexpr size_t fold_bytes(int TS, int UP, int raw_floats) {
        return bar_off(TS, UP, raw_floats) + 5 * 8;
    }
};

// Segment smem for the whole CTA life: max(fold phase, combine phases) + the
// cluster segment row + flag (as pair_smem_bytes).
template <int d, int N, int Q>
__host__ __device__ constexpr size_t ppair_segrow_off(int U, int TS, int raw_floats, int G) {
    const size_t seg = G > 1 ? (CombineLayout<d, N>::floats(G, 0) + (size_t)G * ipow(d, N)) * 4 : 0;
    const size_t fold = PPairLayout<d, N, Q>::fold_bytes(TS, U / 2, raw_floats);
    const size_t comb = CombineLayout<d, N>::floats(U, U / 2) * 4;
    const size_t m = fold > comb ? fold : comb;
    return ((m > seg ? m : seg) + 15) / 16 * 16;
}
template <int d, int N, int Q>
__host__ __device__ constexpr size_t ppair_smem_bytes(int U, int TS, int raw_floats, int G, bool cluster) {
    return ppair_segrow_off<d, N, Q>(U, TS, raw_floats, G) + (cluster ? (size_t)level_off(d, N) * 4 : 0) + 16;
}

// grid = B * G CTAs (cluster of G when CLUSTER); block = fold warps + 1
// producer warp; g.threads = fold threads (UP * P rounded up to a warp).
template <int DIM, int DEPTH, int Q, int NT, int MINB, int TS, bool CLUSTER = false>
__global__ void __launch_bounds__(NT, MINB) ppair_kernel(const float* __restrict__ X, int64_t L, PairGeom g,
                                                         float* __restrict__ out) {
    using PF = PosFold<DIM, DEPTH, Q>;
    using LY = PPairLayout<DIM, DEPTH, Q>;
    constexpr bool P1S = true;  // position tables need the (1, X[s_j] - X[0], 0, ...) chunk starts
    constexpr int d = DIM, RS = PF::RS, RP = PF::RP, N = DEPTH;
    extern __shared__ __align__(16) unsigned char smem_raw[];

    const int64_t rowid = blockIdx.x;
    const int64_t b = rowid / g.G, sg = rowid - b * g.G;
    const int64_t M = L - 1;
    const int64_t seg0 = sg * g.SL < M ? sg * g.SL : M;
    const int64_t slen = (seg0 + g.SL < M ? seg0 + g.SL : M) - seg0;
    const int U = g.U, UP = g.UP, CL = g.CL;
    const int tid = threadIdx.x;
    const int nfold = g.threads;  // fold threads (whole warps); the producer warp follows
    const float* __restrict__ xb = X + b * L * d;
    const int ntiles = (CL + TS - 1) / TS;

    f2* tiles = reinterpret_cast<f2*>(smem_raw);  // [2][TS][UP][RS]
    float* raw = reinterpret_cast<float*>(smem_raw + LY::raw_off(TS, UP));
    uint64_t* bars = reinterpret_cast<uint64_t*>(smem_raw + LY::bar_off(TS, UP, g.raw_floats));
    uint64_t* stage_bar = bars;     // points staged (TMA)
    uint64_t* full = bars + 1;      // [2] tile built (32 producer arrivals)
    uint64_t* empty = bars + 3;     // [2] tile consumed (all fold-thread arrivals)

    auto phase = [&](int i) {
        if (g.phases != nullptr && tid == 0) {
            g.phases[rowid * 12 + i] = clock64();
            if (i == 0 || i == 9) {
                unsigned long long t;
                asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
                g.phases[rowid * 12 + 10 + (i == 9)] = (long long)t;
            }
        }
    };
    phase(0);
    pdl_trigger();
    if (tid == 0) {
        mbar_init(stage_bar, 1);
        mbar_init(full, 32);
        mbar_init(full + 1, 32);
        mbar_init(empty, nfold);
        mbar_init(empty + 1, nfold);
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    const bool active = tid < UP * PF::P;
    const int k = active ? tid / PF::P : 0;
    const int pre = active ? tid - (tid / PF::P) * PF::P : 0;
    int dig[PF::QS];
#pragma unroll
    for (int q = 0; q < PF::QS; ++q) dig[q] = (pre / ipow(d, Q - 1 - q)) % d;
    float p10v = 0.f;
    if (tid < d) p10v = __ldg(xb + seg0 * d + tid) - __ldg(xb + tid);  // P^(0)_1
    const float x0d = tid < nfold ? __ldg(xb + dig[0]) : 0.f;             // X[b, 0, p_1]
    __syncthreads();  // barriers initialised

    // raw is shifted so the 16-byte-aligned body of the segment's points is aligned in smem
    const float* src = xb + seg0 * d;
    const int nraw = (int)((slen + 1) * d);
    raw += (reinterpret_cast<uintptr_t>(src) & 15) / 4;

    f2 st[PF::S];
#pragma unroll
    for (int i = 0; i < PF::S; ++i) st[i] = 0;

    if (tid >= nfold) {
        // ------------------------------------------------------- producer warp
        const int lane = tid - nfold;
        {
            const uintptr_t sa = reinterpret_cast<uintptr_t>(src);
            const uintptr_t a = (sa + 15) & ~uintptr_t(15), e = (sa + 4ull * nraw) & ~uintptr_t(15);
            const int h = (int)((a - sa) / 4);
            const int nb = e > a ? (int)((e - a) / 4) : 0;
            const int t0 = nb > 0 ? h + nb : 0;
            if (nb == 0) {
                for (int i = lane; i < nraw; i += 32) raw[i] = src[i];
            } else {
                if (lane == 0) {
                    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_addr(stage_bar)),
                                 "r"((uint32_t)(4 * nb))
                                 : "memory");
                    asm volatile(
                        "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                            smem_addr(raw + h)),
                        "l"(src + h), "r"((uint32_t)(4 * nb)), "r"(smem_addr(stage_bar))
                        : "memory");
                }
                if (lane < h) raw[lane] = src[lane];
                if (lane < nraw - t0) raw[t0 + lane] = src[t0 + lane];
                mbar_wait(stage_bar, 0);
            }
            __syncwarp();
        }
        float x0[d];  // X[b, 0, :]
#pragma unroll
        for (int c = 0; c < d; ++c) x0[c] = __ldg(xb + c);
        const int sl = (int)slen;
        for (int t = 0; t < ntiles; ++t) {
            const int bf = t & 1;
            if (t >= 2) mbar_wait(empty + bf, ((t >> 1) - 1) & 1);
            f2* tab = tiles + (size_t)bf * TS * UP * RS;
            const int s0 = t * TS, ns = min(TS, CL - s0);
            // one (pair-unit, channel) column per lane, walked along the tile's
            // steps: one new point per chunk and step (the previous one carries
            // over in registers), no index division inside the walk; lanes on
            // consecutive channels write consecutive pairs of a row
            for (int pc = lane; pc < UP * d; pc += 32) {
                const int kk = pc / d, c = pc - (pc / d) * d;
                const int cs0 = min(2 * kk * CL, sl), cs1 = min((2 * kk + 1) * CL, sl);
                const int lim0 = min(cs0 + CL, sl) - cs0, lim1 = min(cs1 + CL, sl) - cs1;  // real steps
                float xc = x0[0];
#pragma unroll
                for (int cc = 1; cc < d; ++cc) xc = cc == c ? x0[cc] : xc;
                const f2 nxc = f2_bcast(-xc);
                const float* q0 = raw + cs0 * d + c;
                const float* q1 = raw + cs1 * d + c;
                f2* col = tab + (size_t)kk * RS + c;
                // (chunk 2kk, chunk 2kk+1) pairs throughout: packed FP32x2 arithmetic
                f2 y = f2_pack(q0[min(s0, lim0) * d], q1[min(s0, lim1) * d]);
#pragma unroll 4
                for (int si = 0; si < ns; ++si) {
                    const int s = s0 + si;
                    float ylo, yhi;
                    f2_unpack(y, ylo, yhi);
                    const f2 nx = f2_pack(s < lim0 ? q0[(s + 1) * d] : ylo, s < lim1 ? q1[(s + 1) * d] : yhi);
                    const f2 dl = fadd2(nx, fmul2(y, f2_bcast(-1.0f)));  // 0 past a chunk's end
                    const f2 yr = fadd2(y, nxc);                         // X[t] - X[0]
                    f2* row = col + (size_t)si * UP * RS;
                    row[0] = dl;
#pragma unroll
                    for (int n = 2; n <= N; ++n)  // a_n = (X[t] - X[0] + δ/n) / (n - 1)
                        row[(n - 1) * RP] = fmul2(ffma2(dl, f2_bcast(1.0f / n), yr), f2_bcast(1.0f / (n - 1)));
                    y = nx;
                }
            }
            mbar_arrive(full + bf);  // every producer lane: its rows are written (release)
        }
        if (g.phases != nullptr && lane == 0) g.phases[rowid * 12 + 2] = clock64();  // probes: last tile built
    } else {
        // ---------------------------------------------------------- fold warps
        for (int t = 0; t < ntiles; ++t) {
            const int bf = t & 1;
            mbar_wait(full + bf, (t >> 1) & 1);
            if (t == 0) phase(1);  // first tile ready
            if (active) {
                const f2* base = tiles + (size_t)bf * TS * UP * RS + (size_t)k * RS;
                const size_t stride = (size_t)UP * RS;
                const int ns = min(TS, CL - t * TS);
                typename PF::Ops oa, ob;
                PF::load(oa, base, dig);
                int i = 0;
                for (; i + 2 <= ns; i += 2) {
                    PF::load(ob, base + (size_t)(i + 1) * stride, dig);
                    PF::step(st, oa);
                    if (i + 2 < ns) PF::load(oa, base + (size_t)(i + 2) * stride, dig);
                    PF::step(st, ob);
                }
                if (i < ns) PF::step(st, oa);
            }
            mbar_arrive(empty + bf);  // this thread is done reading the tile
        }
    }
    phase(3);
    __syncthreads();  // points staged and every fold done (raw still intact); no mbarrier in use
    if (tid == 0) {
#pragma unroll
        for (int i = 0; i < 5; ++i) asm volatile("mbarrier.inval.shared::cta.b64 [%0];" ::"r"(smem_addr(bars + i)) : "memory");
    }
    if (active) {
        // T_1 at each chunk's end = X[e_j] - X[0] (the position table kept it implicit)
        const int sl = (int)slen;
        const int e0 = min(min(2 * k * CL, sl) + CL, sl), e1 = min(min((2 * k + 1) * CL, sl) + CL, sl);
        const int c = dig[0];
        PF::scal(st, 1) = f2_pack(raw[e0 * d + c] - x0d, raw[e1 * d + c] - x0d);
    }
    __syncthreads();  // tiles, points and barriers are dead: the combine reuses the buffer
    phase(4);
    pair_combine_store<PF, CLUSTER, P1S>(st, active, k, pre, p10v, g, rowid, b, out, smem_raw, phase);
}

}  // namespace sigk
