// Shape-generic fold for (d, N) pairs without a register-sliced instantiation.
//
// Same recurrence as fold.cuh (reference sig_core.hpp:92-114), evaluated
// element-parallel instead of slice-parallel: one CTA per path keeps the flat
// state row in global memory (L2-resident), and for each step updates the
// levels in descending order, one CTA barrier per level:
//     T_n[I] += Σ_{j=1}^{n} T_{n-j}[I / d^j] · Π_{last j digits c of I} δ[c] / j!
// with T_0 = 1. Slow (O(N·D) work and N barriers per step) but correct for
// any shape; the dispatcher only routes here when no fast variant exists.
#pragma once

#include "sigk_common.cuh"

namespace sigk {

constexpr int kGenericMaxDepth = 16;

template <typename Real>
__global__ void __launch_bounds__(256) generic_fold_kernel(const Real* __restrict__ X, int64_t L, int d, int N,
                                                           int64_t D, Real* __restrict__ out) {
    extern __shared__ __align__(16) unsigned char smem_raw[];
    Real* dl = reinterpret_cast<Real*>(smem_raw);  // [d]
    __shared__ int64_t off[kGenericMaxDepth + 1];
    __shared__ Real invfact[kGenericMaxDepth + 1];
    const int64_t b = blockIdx.x;
    Real* S = out + b * D;
    if (threadIdx.x == 0) {
        off[0] = 0;
        int64_t p = 1;
        Real f = 1;
        invfact[0] = 1;
        for (int n = 1; n <= N; ++n) {
            p *= d;
            off[n] = off[n - 1] + p;
            f *= Real(n);
            invfact[n] = Real(1) / f;
        }
    }
    for (int64_t i = threadIdx.x; i < D; i += blockDim.x) S[i] = Real(0);
    const Real* row = X + b * L * d;
    for (int64_t t = 0; t + 1 < L; ++t) {
        __syncthreads();
        for (int c = threadIdx.x; c < d; c += blockDim.x) dl[c] = row[(t + 1) * d + c] - row[t * d + c];
        __syncthreads();
        for (int n = N; n >= 1; --n) {
            const int64_t lsz = off[n] - off[n - 1];
            for (int64_t I = threadIdx.x; I < lsz; I += blockDim.x) {
                Real acc = S[off[n - 1] + I];
                Real e = 1;
                int64_t rem = I;
                for (int j = 1; j <= n; ++j) {
                    e *= dl[rem % d];
                    rem /= d;
                    const Real lower = (j < n) ? S[off[n - j - 1] + rem] : Real(1);
                    acc = fma(lower, e * invfact[j], acc);
                }
                S[off[n - 1] + I] = acc;
            }
            __syncthreads();
        }
    }
}

// Synthetic Brownian paths for the benchmark: X[b,0,:] = 0,
// X[b,t,c] = X[b,t-1,c] + σ·Z, σ = 1/sqrt(L-1), Z ~ N(0,1) from a
// counter-based Philox4x32-10 keyed by (seed, global row b, t, c), so a row's
// values do not depend on how the batch is sharded. (Mirrors the reference's
// make_bench_paths distribution, bench.cpp:134-161; the stream itself differs.)
__device__ __forceinline__ void philox4x32_10(uint32_t (&ctr)[4], uint32_t k0, uint32_t k1) {
#pragma unroll
    for (int r = 0; r < 10; ++r) {
        const uint64_t p0 = (uint64_t)0xD2511F53u * ctr[0];
        const uint64_t p1 = (uint64_t)0xCD9E8D57u * ctr[2];
        const uint32_t hi0 = (uint32_t)(p0 >> 32), lo0 = (uint32_t)p0;
        const uint32_t hi1 = (uint32_t)(p1 >> 32), lo1 = (uint32_t)p1;
        const uint32_t n0 = hi1 ^ ctr[1] ^ k0;
        const uint32_t n2 = hi0 ^ ctr[3] ^ k1;
        ctr[0] = n0;
        ctr[1] = lo1;
        ctr[2] = n2;
        ctr[3] = lo0;
        k0 += 0x9E3779B9u;
        k1 += 0xBB67AE85u;
    }
}

template <typename Real>
__global__ void brownian_kernel(Real* __restrict__ X, int64_t B, int64_t L, int d, uint64_t seed, int64_t row0) {
    const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;  // (b, c)
    if (i >= B * d) return;
    const int64_t b = i / d;
    const int c = (int)(i % d);
    const int64_t gb = row0 + b;
    const double sigma = L > 1 ? 1.0 / sqrt((double)(L - 1)) : 1.0;
    Real* row = X + b * L * d + c;
    double acc = 0.0;
    row[0] = Real(0);
    for (int64_t t = 1; t < L; ++t) {
        uint32_t ctr[4] = {(uint32_t)t, (uint32_t)(t >> 32) ^ ((uint32_t)c << 16), (uint32_t)gb, (uint32_t)(gb >> 32)};
        philox4x32_10(ctr, (uint32_t)seed, (uint32_t)(seed >> 32));
        const double u1 = ((double)ctr[0] + 1.0) * (1.0 / 4294967296.0);  // (0, 1]
        const double u2 = (double)ctr[1] * (1.0 / 4294967296.0);
        const double z = sqrt(-2.0 * log(u1)) * cospi(2.0 * u2);
        acc += sigma * z;
        row[t * d] = Real(acc);
    }
}

}  // namespace sigk

namespace sigk {

// Prefix stream for shapes / precisions without the pair-family stream kernel:
// out (B, L-1, D), row t = signature of X[0..t+1]. Row t is computed from row
// t-1 (element-parallel, one barrier per step, no level ordering needed since
// the previous state is a separate row):
//     T_n(t)[I] = T_n(t-1)[I] + Σ_{j=1}^{n} T_{n-j}(t-1)[I / d^j] · Π_{last j digits c} δ[c] / j!
//
// Chunk-parallel: CTA (b, u) of a grid of B*U walks steps [u*CL, min((u+1)*CL,
// M)) of path b, starting from `starts` row b*U + u (the signature of X[0 ..
// u*CL], from chunk_prefix_kernel; u = 0 starts from the identity), so the
// walk's serial length is CL instead of L-1.
template <typename Real>
__global__ void __launch_bounds__(256) generic_stream_kernel(const Real* __restrict__ X, int64_t L, int d, int N,
                                                             int64_t D, Real* __restrict__ out, int U, int64_t CL,
                                                             const Real* __restrict__ starts) {
    extern __shared__ __align__(16) unsigned char smem_raw[];
    Real* dl = reinterpret_cast<Real*>(smem_raw);  // [d]
    __shared__ int64_t off[kGenericMaxDepth + 1];
    __shared__ Real invfact[kGenericMaxDepth + 1];
    const int64_t b = blockIdx.x / U, u = blockIdx.x - (blockIdx.x / U) * U;
    const int64_t M = L - 1;
    const int64_t t0 = u * CL < M ? u * CL : M, t1 = t0 + CL < M ? t0 + CL : M;
    Real* ob = out + b * M * D;
    if (threadIdx.x == 0) {
        off[0] = 0;
        int64_t p = 1;
        Real f = 1;
        invfact[0] = 1;
        for (int n = 1; n <= N; ++n) {
            p *= d;
            off[n] = off[n - 1] + p;
            f *= Real(n);
            invfact[n] = Real(1) / f;
        }
    }
    pdl_trigger();
    pdl_wait();
    const Real* row = X + b * L * d;
    const Real* start = u > 0 ? starts + (b * U + u) * D : nullptr;
    for (int64_t t = t0; t < t1; ++t) {
        __syncthreads();
        for (int c = threadIdx.x; c < d; c += blockDim.x) dl[c] = row[(t + 1) * d + c] - row[t * d + c];
        __syncthreads();
        const Real* prev = t > t0 ? ob + (t - 1) * D : start;
        Real* cur = ob + t * D;
        for (int64_t F = threadIdx.x; F < D; F += blockDim.x) {
            int n = 1;
            while (F >= off[n]) ++n;
            const int64_t I = F - off[n - 1];
            Real acc = prev ? prev[F] : Real(0);
            Real e = 1;
            int64_t rem = I;
            for (int j = 1; j <= n; ++j) {
                e *= dl[rem % d];
                rem /= d;
                const Real lower = (j < n) ? (prev ? prev[off[n - j - 1] + rem] : Real(0)) : Real(1);
                acc = fma(lower, e * invfact[j], acc);
            }
            cur[F] = acc;
        }
    }
}

// The same walk for small signatures (D <= 1024, d <= 16): one thread per
// entry (block = D rounded up to a warp), its index data in registers — the
// degree, the trailing digits (4 bits each) and the offsets of the NM
// lower-degree entries it multiplies — so a step costs loads and FMAs only,
// no integer division; the running row is double-buffered in shared memory
// and the chunk's points are staged once, so a step touches global memory
// only to store its row.
// final_rows != null: signature mode — no row per step; the chunk's own
// signature (walked from the identity when starts == null) goes to row
// b*U + u of final_rows.
template <typename Real, int NM>
__global__ void __launch_bounds__(1024) generic_stream_small_kernel(const Real* __restrict__ X, int64_t L, int d, int N,
                                                                    int64_t D, Real* __restrict__ out, int U, int64_t CL,
                                                                    const Real* __restrict__ starts,
                                                                    Real* __restrict__ final_rows) {
    extern __shared__ __align__(16) unsigned char smem_raw[];
    Real* dl = reinterpret_cast<Real*>(smem_raw);  // [d]
    __shared__ Real invfact[NM + 1];
    const int64_t b = blockIdx.x / U, u = blockIdx.x - (blockIdx.x / U) * U;
    const int64_t M = L - 1;
    const int64_t t0 = u * CL < M ? u * CL : M, t1 = t0 + CL < M ? t0 + CL : M;
    Real* ob = out + b * M * D;
    if (threadIdx.x == 0) {
        Real f = 1;
        invfact[0] = 1;
        for (int n = 1; n <= N; ++n) {
            f *= Real(n);
            invfact[n] = Real(1) / f;
        }
    }
    const int F = (int)threadIdx.x;
    int deg = 0;
    uint32_t digs = 0;
    int lo[NM];
#pragma unroll
    for (int j = 0; j < NM; ++j) lo[j] = 0;
    if (F < D) {
        int n = 1, off0 = 0, sz = d;  // level n occupies [off0, off0 + sz)
        while (F >= off0 + sz) {
            off0 += sz;
            sz *= d;
            ++n;
        }
        deg = n;
        int rem = F - off0;
#pragma unroll
        for (int j = 1; j <= NM; ++j) {
            if (j <= n) {
                digs |= (uint32_t)(rem % d) << (4 * (j - 1));
                rem /= d;
                int offl = 0, p = 1;  // entry I / d^j of level n - j starts at off(n - j - 1)
                for (int m = 1; m < n - j; ++m) {
                    p *= d;
                    offl += p;
                }
                lo[j - 1] = offl + rem;
            }
        }
    }
    pdl_trigger();
    pdl_wait();
    const Real* row = X + b * L * d;
    Real* rows = dl + 16;      // [2][D]
    Real* pts = rows + 2 * D;  // X[t0 .. t1]
    const Real* start = u > 0 ? starts + (b * U + u) * D : nullptr;
    for (int i = threadIdx.x; i < D; i += blockDim.x) rows[i] = start ? start[i] : Real(0);
    for (int64_t i = threadIdx.x; i < (t1 - t0 + 1) * d; i += blockDim.x) pts[i] = row[t0 * d + i];
    for (int64_t t = t0; t < t1; ++t) {
        __syncthreads();
        const Real* pt = pts + (t - t0) * d;
        for (int c = threadIdx.x; c < d; c += blockDim.x) dl[c] = pt[d + c] - pt[c];
        __syncthreads();
        const int par = (int)((t - t0) & 1);
        const Real* prev = rows + par * D;
        if (deg > 0) {
            Real acc = prev[F];
            Real e = 1;
#pragma unroll
            for (int j = 1; j <= NM; ++j) {
                if (j <= deg) {
                    e *= dl[(digs >> (4 * (j - 1))) & 15u];
                    const Real lower = (j < deg) ? prev[lo[j - 1]] : Real(1);
                    acc = fma(lower, e * invfact[j], acc);
                }
            }
            rows[(1 - par) * D + F] = acc;
            if (!final_rows) ob[t * D + F] = acc;
        }
    }
    if (final_rows && F < D) final_rows[(b * U + u) * D + F] = rows[((t1 - t0) & 1) * D + F];
}

// The chunk walk for larger signatures or depths (any D whose two rows and the
// chunk's points fit shared memory, N <= 16): 1024 threads, entries strided
// over them, index data recomputed per step in 32-bit arithmetic; rows and
// points in shared memory as above. final_rows as generic_stream_small_kernel.
template <typename Real>
__global__ void __launch_bounds__(1024) generic_walk_kernel(const Real* __restrict__ X, int64_t L, int d, int N, int64_t D,
                                                            Real* __restrict__ out, int U, int64_t CL,
                                                            const Real* __restrict__ starts,
                                                            Real* __restrict__ final_rows) {
    extern __shared__ __align__(16) unsigned char smem_raw[];
    Real* dl = reinterpret_cast<Real*>(smem_raw);  // [d] (<= 16)
    __shared__ int off[kGenericMaxDepth + 1];
    __shared__ Real invfact[kGenericMaxDepth + 1];
    const int64_t b = blockIdx.x / U, u = blockIdx.x - (blockIdx.x / U) * U;
    const int64_t M = L - 1;
    const int64_t t0 = u * CL < M ? u * CL : M, t1 = t0 + CL < M ? t0 + CL : M;
    Real* ob = out ? out + b * M * D : nullptr;
    if (threadIdx.x == 0) {
        off[0] = 0;
        int p = 1;
        Real f = 1;
        invfact[0] = 1;
        for (int n = 1; n <= N; ++n) {
            p *= d;
            off[n] = off[n - 1] + p;
            f *= Real(n);
            invfact[n] = Real(1) / f;
        }
    }
    pdl_trigger();
    pdl_wait();
    const Real* row = X + b * L * d;
    Real* rows = dl + 16;      // [2][D]
    Real* pts = rows + 2 * D;  // X[t0 .. t1]
    const Real* start = u > 0 && starts ? starts + (b * U + u) * D : nullptr;
    for (int64_t i = threadIdx.x; i < D; i += blockDim.x) rows[i] = start ? start[i] : Real(0);
    for (int64_t i = threadIdx.x; i < (t1 - t0 + 1) * d; i += blockDim.x) pts[i] = row[t0 * d + i];
    for (int64_t t = t0; t < t1; ++t) {
        __syncthreads();
        const Real* pt = pts + (t - t0) * d;
        for (int c = threadIdx.x; c < d; c += blockDim.x) dl[c] = pt[d + c] - pt[c];
        __syncthreads();
        const int par = (int)((t - t0) & 1);
        const Real* prev = rows + par * D;
        Real* nxt = rows + (1 - par) * D;
        for (int F = threadIdx.x; F < (int)D; F += blockDim.x) {
            int n = 1;
            while (F >= off[n]) ++n;
            int rem = F - off[n - 1];
            Real acc = prev[F], e = 1;
            for (int j = 1; j <= n; ++j) {
                e *= dl[rem % d];
                rem /= d;
                const Real lower = (j < n) ? prev[off[n - j - 1] + rem] : Real(1);
                acc = fma(lower, e * invfact[j], acc);
            }
            nxt[F] = acc;
            if (!final_rows) ob[t * D + F] = acc;
        }
    }
    if (final_rows) {
        __syncthreads();
        const Real* fin = rows + ((t1 - t0) & 1) * D;
        for (int64_t F = threadIdx.x; F < D; F += blockDim.x) final_rows[(b * U + u) * D + F] = fin[F];
    }
}

// Prefixes at the chunk starts for the chunk-parallel stream: row b*U + u of
// `starts` = C_0 ⊠ ... ⊠ C_{u-1} (u >= 1; Chen's identity,
// tensor_algebra.cpp:80-102), from the chunk signatures C (B*U, D). One CTA
// per path, one product per chunk, element-parallel (row 0 is not written:
// chunk 0 starts from the identity).
template <typename Real>
__global__ void __launch_bounds__(256) chunk_prefix_kernel(const Real* __restrict__ C, int64_t D, int d, int N, int U,
                                                           Real* __restrict__ starts) {
    __shared__ int64_t off[kGenericMaxDepth + 1], pw[kGenericMaxDepth + 1];
    if (threadIdx.x == 0) {
        off[0] = 0;
        pw[0] = 1;
        for (int n = 1; n <= N; ++n) {
            pw[n] = pw[n - 1] * d;
            off[n] = off[n - 1] + pw[n];
        }
    }
    pdl_trigger();
    pdl_wait();
    __syncthreads();
    const int64_t b = blockIdx.x;
    const Real* Cb = C + b * U * D;
    Real* Sb = starts + b * U * D;
    for (int u = 1; u < U; ++u) {
        const Real* a = u > 1 ? Sb + (int64_t)(u - 1) * D : nullptr;  // P_{u-1} (identity for u = 1)
        const Real* c = Cb + (int64_t)(u - 1) * D;                    // C_{u-1}
        Real* o = Sb + (int64_t)u * D;
        for (int64_t F = threadIdx.x; F < D; F += blockDim.x) {
            int n = 1;
            while (F >= off[n]) ++n;
            const int64_t I = F - off[n - 1];
            Real v = (a ? a[F] : Real(0)) + c[F];
            if (a)
                for (int k = 1; k < n; ++k)  // a_k ⊗ c_{n-k}
                    v = fma(a[off[k - 1] + I / pw[n - k]], c[off[n - k - 1] + I % pw[n - k]], v);
            o[F] = v;
        }
        __syncthreads();  // row u is read by the next product
    }
}

// Signature of each path from its U chunk signatures (rows b*U .. b*U+U-1 of
// C): out[b] = C_0 ⊠ C_1 ⊠ ... ⊠ C_{U-1}, left to right in a fixed order
// (Chen's identity, tensor_algebra.cpp:80-102). One CTA per path, the running
// product double-buffered in shared memory (2 D values).
template <typename Real>
__global__ void __launch_bounds__(256) chunk_product_kernel(const Real* __restrict__ C, int64_t D, int d, int N, int U,
                                                            Real* __restrict__ out) {
    extern __shared__ __align__(16) unsigned char smem_raw[];
    Real* acc = reinterpret_cast<Real*>(smem_raw);  // [2][D]
    __shared__ int64_t off[kGenericMaxDepth + 1], pw[kGenericMaxDepth + 1];
    if (threadIdx.x == 0) {
        off[0] = 0;
        pw[0] = 1;
        for (int n = 1; n <= N; ++n) {
            pw[n] = pw[n - 1] * d;
            off[n] = off[n - 1] + pw[n];
        }
    }
    pdl_trigger();
    pdl_wait();
    const int64_t b = blockIdx.x;
    const Real* Cb = C + b * U * D;
    for (int64_t F = threadIdx.x; F < D; F += blockDim.x) acc[F] = Cb[F];
    __syncthreads();
    for (int u = 1; u < U; ++u) {
        const Real* a = acc + ((u - 1) & 1) * D;
        Real* o = acc + (u & 1) * D;
        const Real* c = Cb + (int64_t)u * D;
        for (int64_t F = threadIdx.x; F < D; F += blockDim.x) {
            int n = 1;
            while (F >= off[n]) ++n;
            const int64_t I = F - off[n - 1];
            Real v = a[F] + c[F];
            for (int k = 1; k < n; ++k) v = fma(a[off[k - 1] + I / pw[n - k]], c[off[n - k - 1] + I % pw[n - k]], v);
            o[F] = v;
        }
        __syncthreads();
    }
    const Real* fin = acc + ((U - 1) & 1) * D;
    for (int64_t F = threadIdx.x; F < D; F += blockDim.x) out[b * D + F] = fin[F];
}

}  // namespace sigk
