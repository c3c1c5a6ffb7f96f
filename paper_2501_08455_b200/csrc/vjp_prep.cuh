// Reverse mode's producer in one launch (fp32, pair family, one CTA per path):
// the forward pair fold of the path's U chunks from the identity (each thread
// holds its prefix slice of chunks 2k and 2k+1 as FP32x2 pairs, exactly the
// fold of pair_kernel.cuh), the chunk signatures C^(j) written from registers
// into shared memory, then both chunk passes there (scan_passes_smem: the
// forward prefix E^(j) at every chunk end -> `ends`, the cotangent pulled back
// to every chunk end -> `cbars`). Replaces the chunk-signature launch, its
// global rows and the pass launch for paths whose chunks are short enough to
// fold in one CTA (sigk_abi.cu decides); the slice walk (vjp_slice.cuh) follows.
#pragma once

#include "pair_kernel.cuh"
#include "vjp_slice.cuh"

namespace sigk {

// Levels 1..N of both chunks of a thread's slice -> rows 2k, 2k+1 of `rows`
// (row stride D; rows >= R are not written; redundant prefix scalars by one thread each).
template <typename PF, int n>
__device__ __forceinline__ void store_chunk_rows(const f2 (&st)[PF::S], int k, int pre, float* __restrict__ rows, int R) {
    constexpr int d = PF::d, Q = PF::QQ;
    constexpr int D = level_off(d, PF::N);
    if constexpr (n <= PF::N) {
        float* y0 = rows + (size_t)(2 * k) * D + level_off(d, n - 1);
        float* y1 = y0 + D;
        const bool w0 = 2 * k < R, w1 = 2 * k + 1 < R;
        if constexpr (n >= PF::NMIN) {
            constexpr int sz = ipow(d, n - Q);
            constexpr int o = PF::top_off(n);
#pragma unroll
            for (int J = 0; J < sz; ++J) {
                float lo, hi;
                f2_unpack(st[o + J], lo, hi);
                if (w0) y0[pre * sz + J] = lo;
                if (w1) y1[pre * sz + J] = hi;
            }
        } else {
            constexpr int tail = ipow(d, Q - n);
            if (pre % tail == 0) {
                float lo, hi;
                f2_unpack(st[n - 1], lo, hi);
                if (w0) y0[pre / tail] = lo;
                if (w1) y1[pre / tail] = hi;
            }
        }
        store_chunk_rows<PF, n + 1>(st, k, pre, rows, R);
    }
}

// Shared memory of one CTA: the fold (table + staged points) or, after it,
// the passes' rows (ScanPasses::smem), whichever is larger.
template <int d, int N, int Q>
__host__ __device__ constexpr size_t vjp_prep_smem(int U, int CL, int raw_floats) {
    using PF = PairFold<d, N, Q>;
    const size_t fold = (size_t)CL * (U / 2) * PF::RS * 8 + (size_t)raw_floats * 4 + 16 + 16;
    const size_t passes = ScanPasses<float, d, N>::smem(U);
    return ((fold > passes ? fold : passes) + 15) / 16 * 16;
}

// grid = B; block = g.threads (>= U/2 * P). Path b: M = L-1 steps as U chunks of
// CL (U even; the last chunks may be short or empty), R = ceil(M / CL) of them real.
template <int DIM, int DEPTH, int Q, int NT>
__global__ void __launch_bounds__(NT, 1) pair_vjp_prep_kernel(const float* __restrict__ X, int64_t L, PairGeom g,
                                                              int R, const float* __restrict__ cot,
                                                              float* __restrict__ ends, float* __restrict__ cbars,
                                                              float* __restrict__ grad) {
    using PF = PairFold<DIM, DEPTH, Q>;
    constexpr int d = DIM, N = DEPTH, P = PF::P, RS = PF::RS;
    constexpr int D = level_off(d, N), DL = level_off(d, N - 1);
    extern __shared__ __align__(16) unsigned char smem_raw[];
    const int64_t b = blockIdx.x;
    const int64_t M = L - 1;
    const int UP = g.UP, CL = g.CL;
    const int tid = threadIdx.x, nth = blockDim.x;
    const float* __restrict__ xb = X + b * L * d;
    f2* tab = reinterpret_cast<f2*>(smem_raw);                                   // [CL][UP][RS]
    float* raw = reinterpret_cast<float*>(smem_raw + (size_t)CL * UP * RS * 8);  // [(M+1)*d + 4]
    uint64_t* bar = reinterpret_cast<uint64_t*>(raw + g.raw_floats + 4);
    const bool active = tid < UP * P;
    const int k = active ? tid / P : 0;
    const int pre = active ? tid - (tid / P) * P : 0;
    int dig[PF::QS];
#pragma unroll
    for (int q = 0; q < PF::QS; ++q) dig[q] = (Q > 0) ? (pre / ipow(d, Q > 0 ? Q - 1 - q : 0)) % d : 0;
    pair_stage_and_table<PF>(xb, 0, M, CL, UP, tab, raw, bar);
    f2 st[PF::S];
#pragma unroll
    for (int i = 0; i < PF::S; ++i) st[i] = 0;  // chunks fold from the identity: st = C^(j)
    __syncthreads();
    if (tid == 0) asm volatile("mbarrier.inval.shared::cta.b64 [%0];" ::"r"(smem_addr(bar)) : "memory");
    if (active) {
        const f2* base = tab + (size_t)k * RS;
        const size_t stride = (size_t)UP * RS;
        if constexpr (PF::PREFETCH) {
            typename PF::Ops oa, ob;
            PF::load(oa, base, dig);
            int i = 0;
            for (; i + 2 <= CL; i += 2) {
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
    __syncthreads();  // table and staged points are dead: the rows take their place
    float* Cs = reinterpret_cast<float*>(smem_raw);  // [R][D]
    float* Es = Cs + (size_t)R * D;                   // [R][DL]
    float* Ts = Es + (size_t)R * DL;                  // [R][DL]
    float* cs = Ts + (size_t)R * DL;                  // [D]
    if (active) store_chunk_rows<PF, 1>(st, k, pre, Cs, R);
    for (int i = tid; i < D; i += nth) cs[i] = __ldg(cot + b * D + i);
    {  // the walk adds the two chunks' terms of every shared chunk point onto zeros
        float* gb = grad + b * L * d;
        for (int i = tid; i < (R - 1) * d; i += nth) {
            const int j = i / d;
            gb[(int64_t)(j + 1) * CL * d + (i - j * d)] = 0.f;
        }
    }
    __syncthreads();
    scan_passes_smem<float, d, N, true, true>(Cs, Es, Ts, cs, R, ends + b * (int64_t)R * D, cbars + b * (int64_t)R * D,
                                              tid, nth);
}

}  // namespace sigk
