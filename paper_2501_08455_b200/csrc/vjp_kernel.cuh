// Reverse mode: gradient of <cotangent, Sig(X)> with respect to every path
// point (reference signature_vjp, /root/reference/proj/src/autodiff.cpp:218-224;
// the fold adjoint vjp_sequential :31-107).
//
// The forward states (every prefix signature) come from the prefix-stream
// kernels; one CTA per path then walks the steps backwards, element-parallel
// over the D coefficients, with exactly the reference's adjoint of
// C = A ⊠ exp(δ):
//     Ā_i[I]  = C̄_i[I] + Σ_j Σ_J C̄_{i+j}[I J] E_j[J]            (A = state before)
//     Ē_j[J]  = C̄_j[J] + Σ_i Σ_I C̄_{i+j}[I J] A_i[I]            (E = exp(δ))
// then through e_n = e_{n-1} ⊗ δ / n from the top degree down, and
// ∂L/∂X_t = δ̄_{t-1} − δ̄_t. Reductions over a leading index (the δ̄ terms)
// are warp shuffles in a fixed order: deterministic.
#pragma once

#include "generic.cuh"

namespace sigk {

template <typename Real>
__device__ __forceinline__ Real warp_sum(Real v) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
    return v;
}

// X (B, L, d); states (B, L-1, D) = prefix signatures (row t after step t);
// cot (B, D); grad (B, L, d). work: per-CTA scratch of vjp_work_elems(D, d)
// Reals (shared memory when it fits, else `gwork` + blockIdx * that). The
// state row of the next step is prefetched with cp.async into a second
// buffer while the current step computes.
__host__ __device__ constexpr int64_t vjp_horner_elems(int d, int N) {
    int64_t p = 1;
    for (int n = 1; n < N; ++n) p *= d;
    return N > 2 ? 2 * (N - 2) * p : 0;  // Ā Horner chains: two buffers of d^(N-1) per target n < N-1
}
__host__ __device__ constexpr int64_t vjp_work_elems(int64_t D, int d, int N) {
    return 6 * D + 3 * d + 4 + vjp_horner_elems(d, N);
}

template <typename Real>
__device__ __forceinline__ void prefetch_row(Real* dst, const Real* src, int64_t n) {
    for (int64_t i = threadIdx.x; i < n; i += blockDim.x) {
        if constexpr (sizeof(Real) == 8)
            asm volatile("cp.async.ca.shared.global [%0], [%1], 8;" ::"r"(static_cast<uint32_t>(__cvta_generic_to_shared(dst + i))),
                         "l"(src + i)
                         : "memory");
        else
            asm volatile("cp.async.ca.shared.global [%0], [%1], 4;" ::"r"(static_cast<uint32_t>(__cvta_generic_to_shared(dst + i))),
                         "l"(src + i)
                         : "memory");
    }
    asm volatile("cp.async.commit_group;" ::: "memory");
}
// CTA (b, j) of the grid walks chunk j = steps [j*CL, min((j+1)*CL, M)) of
// path b backwards, starting from the cotangent of the state at the chunk's
// end (cbars row b*U + j; the boundary kernel below), and writes δ̄_s of its
// steps to dbar (B, M, d); vjp_grad_kernel turns those into ∂/∂X.
template <typename Real, int DD = 0, int NN = 0>
__global__ void __launch_bounds__(256) vjp_kernel(const Real* __restrict__ X, int64_t L, int d_, int N_, int64_t D,
                                                  const Real* __restrict__ states, const Real* __restrict__ cbars,
                                                  int U, int64_t CL, Real* __restrict__ dbar,
                                                  Real* __restrict__ gwork, int use_smem) {
    extern __shared__ __align__(16) unsigned char smem_raw[];
    // DD/NN > 0: compile-time shape (loops unroll, offsets fold); 0: runtime
    const int d = DD > 0 ? DD : d_;
    const int N = NN > 0 ? NN : N_;
    __shared__ int64_t off[kGenericMaxDepth + 1];
    auto OFF = [&](int n) -> int { return (int)off[n]; };
    __shared__ Real invfact[kGenericMaxDepth + 1];
    const int64_t b = blockIdx.x / U, j = blockIdx.x - (blockIdx.x / U) * U;
    const int64_t M = L - 1;
    const int64_t s_lo = j * CL < M ? j * CL : M, s_hi = (j + 1) * CL < M ? (j + 1) * CL : M;
    const int tid = threadIdx.x, nth = blockDim.x, lane = tid & 31, warp = tid >> 5, nw = nth >> 5;
    Real* work = use_smem ? reinterpret_cast<Real*>(smem_raw) : gwork + (int64_t)blockIdx.x * vjp_work_elems(D, d, N);
    Real* cbar = work;            // [D] cotangent of the state after the step
    Real* abar = cbar + D;        // [D] ... of the state before it
    Real* ebar = abar + D;        // [D] ... of exp(δ)
    Real* E = ebar + D;           // [D] exp(δ)
    Real* Ab[2] = {E + D, E + 2 * D};  // [2][D] state rows (current, next)
    Real* dl = E + 3 * D;         // [d] δ
    Real* db = dl + d;            // [d] δ̄ of this step
    Real* dbn = db + d;           // [d] δ̄ of the next step
    Real* gh = dbn + d + 4;       // [N-2][2][d^(N-1)] Ā Horner chains
    if (tid == 0) {
        off[0] = 0;
        int64_t p = 1;
        Real f = 1;
        invfact[0] = 1;
#pragma unroll
        for (int n = 1; n <= N; ++n) {
            p *= d;
            off[n] = off[n - 1] + p;
            f *= Real(n);
            invfact[n] = Real(1) / f;
        }
    }
    pdl_trigger();
    pdl_wait();
    const Real* xb = X + b * L * d;
    const Real* sb = states + b * M * D;
    Real* db_out = dbar + b * M * d;
    for (int64_t i = tid; i < D; i += nth) cbar[i] = cbars[(int64_t)blockIdx.x * D + i];
    const bool async_rows = use_smem;
    if (async_rows && s_hi > s_lo && s_hi >= 2) prefetch_row(Ab[(s_hi - 1) & 1], sb + (s_hi - 2) * D, D);
    __syncthreads();
    for (int64_t s = s_hi - 1; s >= s_lo; --s) {
        // state before step s (null: identity); the row for step s-1 streams in meanwhile
        const Real* A = nullptr;
        if (s > 0) {
            if (async_rows) {
                asm volatile("cp.async.wait_all;" ::: "memory");
                A = Ab[s & 1];
                if (s >= 2 && s - 1 >= s_lo) prefetch_row(Ab[(s - 1) & 1], sb + (s - 2) * D, D);
            } else {
                A = sb + (s - 1) * D;
            }
        }
        for (int c = tid; c < d; c += nth) {
            dl[c] = xb[(s + 1) * d + c] - xb[s * d + c];
            db[c] = Real(0);
        }
        __syncthreads();
        // E_n[P d + c] = E_{n-1}[P] δ[c] / n, levels ascending
#pragma unroll
        for (int n = 1; n <= N; ++n) {
            const int psz = n == 1 ? 1 : (int)(OFF(n - 1) - OFF(n - 2));  // d^(n-1)
            const Real inv = Real(1) / Real(n);
            for (int P = tid; P < psz; P += nth) {
                const Real e = (n == 1 ? Real(1) : E[OFF(n - 2) + P]) * inv;
                Real* dst = E + OFF(n - 1) + P * d;
                for (int c = 0; c < d; ++c) dst[c] = e * dl[c];
            }
            __syncthreads();
        }
        // Ā_n[I] = C̄_n[I] + Σ_j Σ_J C̄_{n+j}[I J] E_j[J] by Horner over the trailing
        // index, all targets n at once, one stage per level m (descending):
        //   G_{n,m}[I] = C̄_m[I] + Σ_c G_{n,m+1}[I c] δ[c] / (m-n+1),  G_{n,N} = C̄_N,  Ā_n = G_{n,n}
        // (d FMAs per output, every output of a stage in parallel)
        if (A != nullptr) {
            const int dN1 = OFF(N - 1) - OFF(N - 2);  // d^(N-1)
            int cur = 0;
            for (int m = N - 1; m >= 1; --m) {
                const int szm = OFF(m) - OFF(m - 1), om = OFF(m - 1);
                for (int item = tid; item < m * szm; item += nth) {
                    const int n = 1 + item / szm, I = item - (item / szm) * szm;
                    const Real* src = (m + 1 == N) ? cbar + OFF(N - 1) + I * d
                                                   : gh + ((n - 1) * 2 + (cur ^ 1)) * dN1 + I * d;
                    Real acc = Real(0);
#pragma unroll
                    for (int c = 0; c < (DD > 0 ? DD : d); ++c) acc = fma(src[c], dl[c], acc);
                    const Real v = fma(acc, Real(1) / Real(m - n + 1), cbar[om + I]);
                    if (n == m) abar[om + I] = v;
                    else gh[((n - 1) * 2 + cur) * dN1 + I] = v;
                }
                __syncthreads();
                cur ^= 1;
            }
        }
        // Ē_n[J] = C̄_n[J] + Σ_i Σ_I C̄_{i+n}[I J] A_i[I] (leading-index contractions:
        // long dot products by a whole warp, short ones by a thread)
        for (int n = 1; n <= N; ++n) {
            const int sz = (int)(OFF(n) - OFF(n - 1));
            const int on = (int)OFF(n - 1);
            const int len = (int)(OFF(N - n) - 0);  // Σ_{i=1}^{N-n} d^i
            if (A == nullptr || n == N) {
                for (int i = tid; i < sz; i += nth) {
                    if (A == nullptr || n == N) abar[on + i] = cbar[on + i];
                    ebar[on + i] = cbar[on + i];
                }
            } else if (len >= 64) {
                for (int I = warp; I < sz; I += nw) {
                    Real acc = Real(0);
                    for (int i = 1; i + n <= N; ++i) {
                        const int wi = (int)(OFF(i) - OFF(i - 1));
                        const Real* cr = cbar + OFF(i + n - 1) + I;
                        const Real* ar = A + OFF(i - 1);
                        for (int P = lane; P < wi; P += 32) acc = fma(cr[P * sz], ar[P], acc);
                    }
                    acc = warp_sum(acc);
                    if (lane == 0) ebar[on + I] = cbar[on + I] + acc;
                }
            } else {
                for (int I = tid; I < sz; I += nth) {
                    Real acc = cbar[on + I];
                    for (int i = 1; i + n <= N; ++i) {
                        const int wi = (int)(OFF(i) - OFF(i - 1));
                        const Real* cr = cbar + OFF(i + n - 1) + I;
                        const Real* ar = A + OFF(i - 1);
                        for (int P = 0; P < wi; ++P) acc = fma(cr[P * sz], ar[P], acc);
                    }
                    ebar[on + I] = acc;
                }
            }
        }
        __syncthreads();
        // e_n = e_{n-1} ⊗ δ / n, top degree down (autodiff.cpp:86-98)
#pragma unroll
        for (int n = N; n >= 2; --n) {
            const int psz = (int)(OFF(n - 1) - OFF(n - 2));
            const Real inv = Real(1) / Real(n);
            const Real* en = ebar + OFF(n - 1);
            for (int P = tid; P < psz; P += nth) {
                Real acc = Real(0);
                for (int c = 0; c < d; ++c) acc = fma(en[P * d + c], dl[c], acc);
                ebar[OFF(n - 2) + P] = fma(acc, inv, ebar[OFF(n - 2) + P]);
            }
            for (int c = warp; c < d; c += nw) {
                Real acc = Real(0);
                for (int P = lane; P < psz; P += 32) acc = fma(en[P * d + c], E[OFF(n - 2) + P], acc);
                acc = warp_sum(acc);
                if (lane == 0) db[c] = fma(acc, inv, db[c]);
            }
            __syncthreads();
        }
        for (int c = tid; c < d; c += nth) db_out[s * d + c] = db[c] + ebar[c];  // δ̄_s
        Real* t = cbar;
        cbar = abar;
        abar = t;
        __syncthreads();
    }
}

template <typename Real>
using VjpKernelFn = void (*)(const Real*, int64_t, int, int, int64_t, const Real*, const Real*, int, int64_t, Real*,
                             Real*, int);
// compile-time (d, N) instantiations (csrc/vjp_inst.cu); the runtime kernel otherwise
VjpKernelFn<float> vjp_kernel_for_f32(int d, int N);
VjpKernelFn<double> vjp_kernel_for_f64(int d, int N);

// slice-parallel adjoint (vjp_slice.cuh) where a prefix length fits a warp
template <typename Real>
struct VjpSlice {
    void (*fn)(const Real*, int64_t, int64_t, int, int64_t, const Real*, const Real*, Real*) = nullptr;
    int slots = 0;  // (path, chunk) items per warp
    // compile-time boundary + ends pass (vjp_chunk_passes_kernel); null: the runtime kernels
    void (*passes)(const Real*, const Real*, int, int, Real*, Real*, int64_t, int64_t, Real*) = nullptr;
    // the same passes by degree, all chunks at once (vjp_scan_passes_kernel; 512 threads,
    // (U D + 2 U DL + D) values of shared memory, DL = the signature size below level N)
    void (*scan)(const Real*, const Real*, int, int, Real*, Real*, int64_t, int64_t, Real*) = nullptr;
};
VjpSlice<float> vjp_slice_for_f32(int d, int N);
VjpSlice<double> vjp_slice_for_f64(int d, int N);

// Xseg (B*U, CL+1, d): chunk j of path b as its own path (the last point is
// repeated past the end: zero increments, identity factors).
template <typename Real>
__global__ void segment_gather_kernel(const Real* __restrict__ X, int64_t B, int64_t L, int d, int U, int64_t CL,
                                      Real* __restrict__ Xseg) {
    // chunk (b, j) is the contiguous run of points j*CL .. j*CL+CL of path b
    // (the last point repeated past the path's end): a row copy per chunk
    const int per = (int)((CL + 1) * d);
    for (int64_t r = blockIdx.x; r < B * U; r += gridDim.x) {
        const int64_t b = r / U, j = r - b * U;
        const Real* __restrict__ src = X + (b * L + j * CL) * d;
        const Real* __restrict__ last = X + (b * L + L - 1) * d;
        const int64_t left = (L - j * CL) * d;
        const int valid = left < per ? (int)left : per;
        Real* __restrict__ dst = Xseg + r * per;
        for (int q = threadIdx.x; q < per; q += blockDim.x) dst[q] = q < valid ? src[q] : last[q % d];
    }
}

// Cotangents of the state at every chunk end, one CTA per path: row U-1 is
// the output cotangent, row j-1 = row j pulled back through right
// multiplication by chunk j's signature C_j (the adjoint the per-step loop
// applies with exp(δ)): Ā_n[I] = Ā'_n[I] + Σ_k Σ_J Ā'_{n+k}[I J] C_k[J].
template <typename Real>
__global__ void __launch_bounds__(256) vjp_boundary_kernel(const Real* __restrict__ C, const Real* __restrict__ cot,
                                                           Real* __restrict__ cbars, int U, int d, int N, int64_t D) {
    // dynamic shared memory: the running cotangent row and the chunk signature
    // row (2 D values), staged once per chunk so the contractions read shared
    // memory rather than chains of dependent global loads
    extern __shared__ __align__(16) unsigned char smem_raw[];
    Real* cur = reinterpret_cast<Real*>(smem_raw);
    Real* sig = cur + D;
    Real* nxt = sig + D;
    __shared__ int64_t off[kGenericMaxDepth + 1];
    const int64_t b = blockIdx.x;
    const int tid = threadIdx.x, nth = blockDim.x;
    if (tid == 0) {
        off[0] = 0;
        int64_t p = 1;
        for (int n = 1; n <= N; ++n) {
            p *= d;
            off[n] = off[n - 1] + p;
        }
    }
    pdl_trigger();
    pdl_wait();
    Real* cb = cbars + b * U * D;
    for (int64_t i = tid; i < D; i += nth) {
        const Real v = __ldcg(cot + b * D + i);
        cur[i] = v;
        cb[(int64_t)(U - 1) * D + i] = v;
    }
    for (int j = U - 1; j >= 1; --j) {
        const Real* cj = C + (b * U + j) * D;
        for (int64_t i = tid; i < D; i += nth) sig[i] = __ldcg(cj + i);  // a previous launch's output: via L2
        __syncthreads();
        for (int n = 1; n <= N; ++n) {
            const int64_t sz = off[n] - off[n - 1];
            for (int64_t I = tid; I < sz; I += nth) {
                Real acc = cur[off[n - 1] + I];
                int64_t w = 1;
                for (int k = 1; n + k <= N; ++k) {
                    w *= d;
                    const Real* cr = cur + off[n + k - 1] + I * w;
                    const Real* er = sig + off[k - 1];
                    for (int64_t J = 0; J < w; ++J) acc = fma(cr[J], er[J], acc);
                }
                nxt[off[n - 1] + I] = acc;
            }
        }
        __syncthreads();
        for (int64_t i = tid; i < D; i += nth) {
            cur[i] = nxt[i];
            cb[(int64_t)(j - 1) * D + i] = nxt[i];
        }
        __syncthreads();
    }
}

// ∂/∂X_t = δ̄_{t-1} - δ̄_t (δ̄_{-1} = δ̄_M = 0), grad (B, L, d)
template <typename Real>
__global__ void vjp_grad_kernel(const Real* __restrict__ dbar, int64_t B, int64_t L, int d, Real* __restrict__ grad) {
    const int64_t M = L - 1, n = B * L * d;
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
        const int64_t b = i / (L * d), q = i - b * L * d, t = q / d, c = q - t * d;
        const Real* db = dbar + b * M * d;
        grad[i] = (t >= 1 ? db[(t - 1) * d + c] : Real(0)) - (t < M ? db[t * d + c] : Real(0));
    }
}

}  // namespace sigk
