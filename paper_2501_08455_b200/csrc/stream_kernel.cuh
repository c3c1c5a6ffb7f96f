// Prefix-stream kernel: every prefix signature of every path, (B, L-1, D)
// (reference signature_stream, /root/reference/proj/src/kernels.cpp:156-198;
// the stream_out rows of detail::sequential_forward, sig_core.hpp:140-143:
// row k = signature of X[0..k+1]).
//
// The output is L-1 times the signature's size, so this path is bound by HBM
// writes, not by the FMA pipe (C2: 399 MB per call). One CTA per path segment,
// the same chunk-pair FFMA2 machinery as pair_kernel.cuh, two passes over the
// shared-memory δ table:
//   pass 1  chunk j folds from A^(j) = (1, P^(j)_1, 0, ...) -> Y^(j); the chunk
//           combine yields the TRUE prefix P^(j) at every chunk start, all
//           levels (levels < N from the fused scan, level N by an exclusive
//           scan of the per-chunk level-N contributions);
//   pass 2  chunk j folds again from P^(j), and after every step each thread
//           drops its slice of the state into a shared-memory row; full rows
//           (D contiguous floats) leave by TMA bulk stores, one per row, issued
//           per tile of TS steps from a double-buffered stage so the copy-out
//           overlaps the next tile's fold.
// The recomputation costs one extra fold (a few µs) against tens of µs of
// writes, and keeps every row exact to the same rounding as the final
// signature path.
#pragma once

#include "pair_kernel.cuh"

namespace sigk {

template <int d, int N, int Q>
__host__ __device__ constexpr size_t stream_smem_bytes(int U, int CL, int raw_floats, int TS) {
    using PF = PairFold<d, N, Q>;
    using CLY = CombineLayout<d, N>;
    const size_t tab = (size_t)CL * (U / 2) * PF::RS * 8;
    const size_t raw = (size_t)raw_floats * 4 + 16 + 16;
    const size_t comb = (CLY::floats(U, 0) + (size_t)(U + 1) * CLY::LNP) * 4;
    const size_t stage = 2ull * U * TS * level_off(d, N) * 4;  // double-buffered
    size_t m = raw > comb ? raw : comb;
    m = m > stage ? m : stage;
    return tab + m;
}

// State slice of one chunk (lo or hi half of the pairs) -> its row in the
// shared-memory stage (redundant prefix scalars written by one thread each).
template <typename PF, int n, bool HI>
__device__ __forceinline__ void stage_slice(const f2 (&st)[PF::S], int pre, float* __restrict__ row) {
    constexpr int d = PF::d, Q = PF::QQ;
    if constexpr (n <= PF::N) {
        if constexpr (n >= PF::NMIN) {
            constexpr int sz = ipow(d, n - Q);
            constexpr int o = PF::top_off(n);
            float* dst = row + level_off(d, n - 1) + pre * sz;
#pragma unroll
            for (int J = 0; J < sz; ++J) {
                float lo, hi;
                f2_unpack(st[o + J], lo, hi);
                dst[J] = HI ? hi : lo;
            }
        } else {
            constexpr int tail = ipow(d, Q - n);
            if (pre % tail == 0) {
                float lo, hi;
                f2_unpack(st[n - 1], lo, hi);
                row[level_off(d, n - 1) + pre / tail] = HI ? hi : lo;
            }
        }
        stage_slice<PF, n + 1, HI>(st, pre, row);
    }
}

// Load a thread's slice of the prefix rows of chunks 2k (lo) and 2k+1 (hi):
// levels < N from pf rows, level N from top rows.
template <typename PF, int n>
__device__ __forceinline__ void load_prefix_slice(f2 (&st)[PF::S], int pre, const float* __restrict__ p0,
                                                  const float* __restrict__ p1, const float* __restrict__ t0,
                                                  const float* __restrict__ t1) {
    constexpr int d = PF::d, Q = PF::QQ, N = PF::N;
    if constexpr (n <= N) {
        const float* a = n < N ? p0 + level_off(d, n - 1) : t0;
        const float* b = n < N ? p1 + level_off(d, n - 1) : t1;
        if constexpr (n >= PF::NMIN) {
            constexpr int sz = ipow(d, n - Q);
            constexpr int o = PF::top_off(n);
#pragma unroll
            for (int J = 0; J < sz; ++J) st[o + J] = f2_pack(a[pre * sz + J], b[pre * sz + J]);
        } else {
            constexpr int tail = ipow(d, Q - n);
            st[n - 1] = f2_pack(a[pre / tail], b[pre / tail]);
        }
        load_prefix_slice<PF, n + 1>(st, pre, p0, p1, t0, t1);
    }
}

// X: (B, L, d) fp32 -> out (B, L-1, D). grid = B CTAs (one segment per path).
template <int DIM, int DEPTH, int Q, int NT, int MINB, bool P1S = (DIM > 1 && DEPTH > 1)>
__global__ void __launch_bounds__(NT, MINB) pair_stream_kernel(const float* __restrict__ X, int64_t L, PairGeom g,
                                                               int TS, float* __restrict__ out) {
    using PF = PairFold<DIM, DEPTH, Q>;
    using CLY = CombineLayout<DIM, DEPTH>;
    constexpr int d = DIM, N = DEPTH, P = PF::P, RS = PF::RS;
    constexpr int D = level_off(DIM, DEPTH);
    constexpr int DL = CLY::DL, LN = CLY::LN, LNP = CLY::LNP, FJ = PF::FJ;
    extern __shared__ __align__(16) unsigned char smem_raw[];

    // CTA (b, sg): steps [sg*SL, (sg+1)*SL) of path b (G > 1: the path is split)
    const int64_t b = blockIdx.x / g.G, sg = blockIdx.x - (blockIdx.x / g.G) * g.G;
    const int64_t M = L - 1;
    const int64_t seg0 = sg * g.SL < M ? sg * g.SL : M;
    const int64_t slen = (seg0 + g.SL < M ? seg0 + g.SL : M) - seg0;
    // P^(0) of the segment: the inclusive prefix published by the path's
    // previous segment CTA (decoupled look-back, same launch); null: identity
    const bool lookback = g.pub != nullptr && sg > 0;
    const float* __restrict__ pre0 = lookback ? g.pub + (b * g.G + sg - 1) * D : nullptr;
    const int U = g.U, UP = g.UP, CL = g.CL;
    const int tid = threadIdx.x, nth = blockDim.x;
    const float* __restrict__ xb = X + b * L * d;

    f2* tab = reinterpret_cast<f2*>(smem_raw);                                    // [CL][UP][RS], both passes
    unsigned char* area = smem_raw + (size_t)CL * UP * RS * 8;                    // raw | combine | stage
    float* raw = reinterpret_cast<float*>(area);
    uint64_t* bar = reinterpret_cast<uint64_t*>(raw + g.raw_floats + 4);

    pdl_trigger();
    const bool active = tid < UP * P;
    const int k = active ? tid / P : 0;
    const int pre = active ? tid - (tid / P) * P : 0;
    int dig[PF::QS];
#pragma unroll
    for (int q = 0; q < PF::QS; ++q) dig[q] = (Q > 0) ? (pre / ipow(d, Q > 0 ? Q - 1 - q : 0)) % d : 0;
    float x0[Q == 0 ? d : 1];
#pragma unroll
    for (int c = 0; c < (Q == 0 ? d : 1); ++c) x0[c] = __ldg(xb + (Q == 0 ? c : dig[0]));

    raw = pair_stage_and_table<PF>(xb, seg0, slen, CL, UP, tab, raw, bar);
    const int64_t c0 = min((int64_t)(2 * k) * CL, slen), c1 = min((int64_t)(2 * k + 1) * CL, slen);
    f2 st[PF::S];
#pragma unroll
    for (int i = 0; i < PF::S; ++i) st[i] = 0;
    if (P1S && active) {
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
    const f2* base = tab + (size_t)k * RS;
    const size_t stride = (size_t)UP * RS;
    // ---- pass 1: chunk results Y^(j)
    if (active) {
#pragma unroll 2
        for (int i = 0; i < CL; ++i) {
            typename PF::Ops o;
            PF::load(o, base + (size_t)i * stride, dig);
            PF::step(st, o);
        }
    }
    __syncthreads();  // raw is dead: the combine area takes its place
    // ---- true prefixes P^(j), j = 0..U-1, all levels
    CombineSmem<d, N, P1S> S(reinterpret_cast<float*>(area), U);
    float* top = reinterpret_cast<float*>(area) + CLY::floats(U, 0);  // [U+1][LNP]: P^(j)_N
    if (lookback) {  // wait for the previous segment of this path (same launch)
        if (tid == 0) {
            const int* f = g.flags + b * g.G + sg - 1;
            int v;
            for (;;) {
                asm volatile("ld.acquire.gpu.global.b32 %0, [%1];" : "=r"(v) : "l"(f) : "memory");
                if (v == g.epoch) break;
                __nanosleep(64);
            }
        }
        __syncthreads();
    }
    if (active) store_low_levels<PF, 1>(st, k, pre, S.ylow);
    if (tid < d) S.p10[tid] = __ldg(xb + seg0 * d + tid) - __ldg(xb + tid);  // P^(0)_1 = X[seg0] - X[0] (raw is dead)
    S.p0 = pre0;                                            // P^(0), levels 2..N-1 (null: zero)
    __syncthreads();
    fused_scan<d, N, P1S>(S, U, tid, nth);
    build_c<d, N, P1S>(S, U, tid, nth);
    __syncthreads();
    if (active) {  // per-chunk level-N contributions -> top rows j+1
        constexpr int ot = PF::top_off(N);
#pragma unroll
        for (int h = 0; h < 2; ++h) {
            const int j = 2 * k + h;
            float acc[FJ];
#pragma unroll
            for (int J = 0; J < FJ; ++J) {
                float lo, hi;
                f2_unpack(st[ot + J], lo, hi);
                acc[J] = h ? hi : lo;
                if constexpr (N == 1 && P1S) acc[J] -= S.p1(j, pre * FJ + J);  // Y_1 - P_1 = C_1
            }
            top_cross_slice<d, N, Q, P1S, P1S ? 2 : 1>(S, j, pre, acc);
            float* r = top + (size_t)(j + 1) * LNP + (size_t)pre * FJ;
#pragma unroll
            for (int J = 0; J < FJ; ++J) r[J] = acc[J];
        }
    }
    __syncthreads();
    for (int F = tid; F < LN; F += nth) {  // exclusive scan over chunks, fixed order
        float run = pre0 != nullptr ? __ldcg(pre0 + DL + F) : 0.f;  // P^(0)_N (another CTA's output: via L2)
        top[F] = run;
        for (int j = 1; j <= U; ++j) {
            run += top[(size_t)j * LNP + F];
            top[(size_t)j * LNP + F] = run;
        }
    }
    __syncthreads();
    if (g.pub != nullptr && sg + 1 < g.G) {
        // publish P^(U) = signature of X[0 .. segment end] for the next segment CTA;
        // the previous launch is complete first (it may still read these rows)
        pdl_wait();
        float* prow = g.pub + (b * g.G + sg) * D;
        const float* pU = S.pf + (size_t)U * DL;
        for (int i = tid; i < DL; i += nth) prow[i] = pU[i];
        for (int F = tid; F < LN; F += nth) prow[DL + F] = top[(size_t)U * LNP + F];
        __threadfence();
        __syncthreads();
        if (tid == 0) asm volatile("st.release.gpu.global.b32 [%0], %1;" ::"l"(g.flags + b * g.G + sg), "r"(g.epoch) : "memory");
    }
    // ---- pass 2: fold every chunk again from its true prefix, streaming rows
#pragma unroll
    for (int i = 0; i < PF::S; ++i) st[i] = 0;
    if (active)
        load_prefix_slice<PF, 1>(st, pre, S.pf + (size_t)(2 * k) * DL, S.pf + (size_t)(2 * k + 1) * DL,
                                 top + (size_t)(2 * k) * LNP, top + (size_t)(2 * k + 1) * LNP);
    __syncthreads();  // prefixes are in registers: the stage takes the area over
    // double-buffered stage [2][U][TS][D]; full rows leave by TMA bulk stores
    // (cp.async.bulk.global.shared::cta) issued by one thread, so the copy-out
    // of tile t overlaps the fold of tile t+1
    float* stage = reinterpret_cast<float*>(area);
    const size_t sbuf = (size_t)U * TS * D;
    pdl_wait();  // output writes are ordered after the previous launch
    float* ob = out + (b * M + seg0) * D;
    const bool bulk = (D * 4) % 16 == 0 && (reinterpret_cast<uintptr_t>(out) & 15) == 0;
    const int warp = tid >> 5, lane = tid & 31, nwarps = nth >> 5;
    const int sl = (int)slen;
    for (int t0 = 0, it = 0; t0 < CL; t0 += TS, ++it) {
        const int ts = min(TS, CL - t0);
        float* sb = stage + (size_t)(it & 1) * sbuf;
        // every issuing lane waits for its own bulk stores that read this buffer two tiles ago
        if (bulk && lane == 0 && it >= 2) asm volatile("cp.async.bulk.wait_group.read 1;" ::: "memory");
        __syncthreads();
        if (active) {
            for (int i = 0; i < ts; ++i) {
                typename PF::Ops o;
                PF::load(o, base + (size_t)(t0 + i) * stride, dig);
                PF::step(st, o);
                stage_slice<PF, 1, false>(st, pre, sb + ((size_t)(2 * k) * TS + i) * D);
                stage_slice<PF, 1, true>(st, pre, sb + ((size_t)(2 * k + 1) * TS + i) * D);
            }
        }
        if (bulk) asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
        __syncthreads();
        // rows (chunk j, step t0+i) -> out[b, s_j + t0 + i] for real steps only. A
        // chunk's rows of the tile are contiguous both in the stage and in the
        // output, so each chunk leaves as ONE bulk copy of up to TS rows (chunks
        // dealt over the warps, one lane per warp issues: bulk groups are per thread)
        for (int j = warp; j < U; j += nwarps) {
            const int cs = min(j * CL, sl), ce = min(cs + CL, sl);
            const int nrows = max(0, min(ts, ce - (cs + t0)));
            if (nrows == 0) continue;
            const float* srow = sb + (size_t)j * TS * D;
            float* drow = ob + (int64_t)(cs + t0) * D;
            if (bulk) {
                if (lane == 0)
                    asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], %2;" ::"l"(drow),
                                 "r"(smem_addr(srow)), "r"((uint32_t)(nrows * D * 4))
                                 : "memory");
            } else {
                for (int c = lane; c < nrows * D; c += 32) drow[c] = srow[c];
            }
        }
        if (bulk && lane == 0) asm volatile("cp.async.bulk.commit_group;" ::: "memory");
    }
    if (bulk && lane == 0) asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");  // writes done before exit
}

}  // namespace sigk
