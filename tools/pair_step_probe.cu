// Microbenchmark: issue rate of the pair-fold Horner step (pair_kernel.cuh,
// PairFold::step) with operands streamed from a shared-memory table exactly as
// the kernel's fold loop does (software-pipelined loads), at 1..4 warps per SM
// sub-partition. Reports FMA-pipe utilisation = 2 * ops / (4 SMSP * cycles).
//   nvcc -O3 -std=c++17 -gencode arch=compute_100a,code=sm_100a -I paper_2501_08455_b200/csrc tools/pair_step_probe.cu -o tools/pair_step_probe
#include <cstdio>
#include <cuda_runtime.h>

#include <type_traits>

#include "pos_fold.cuh"

using namespace sigk;



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
