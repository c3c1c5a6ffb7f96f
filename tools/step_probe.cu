// Microbenchmark: issue rate of the register-resident Horner step alone
// (SliceFold::step with operands already in registers; no shared memory, no
// barriers) at 1/2/4 warps per SM sub-partition. Reports FFMA-pipe ops/cycle.
//   nvcc -O3 -std=c++17 -gencode arch=compute_100a,code=sm_100a -I paper_2501_08455_b200/csrc tools/step_probe.cu -o tools/step_probe
#include <cstdio>
#include <cuda_runtime.h>

#include "fold.cuh"

using namespace sigk;

template <int D, int N, int Q>
__global__ void __launch_bounds__(256) stepk(float* sink, const float* __restrict__ in, int steps) {
    using SF = SliceFold<float, D, N, Q>;
    float st[SF::S];
#pragma unroll
    for (int i = 0; i < SF::S; ++i) st[i] = 0.f;
    StepRegs<SF, float> r;
#pragma unroll
    for (int i = 0; i < SF::VEC; ++i) r.vs[i] = in[(threadIdx.x + i) & 63] * 1e-3f;
#pragma unroll
    for (int k = 0; k < SF::QS; ++k)
#pragma unroll
        for (int i = 0; i < (SF::SCW > 0 ? SF::SCW : 1); ++i) r.sc[k][i] = in[(threadIdx.x * 3 + i + k) & 63] * 1e-3f;
#pragma unroll 1
    for (int s = 0; s < steps; ++s) {
        SF::step(st, r.vs, r.sc);
        r.vs[0] = -r.vs[0];  // keep the loop honest
    }
    float acc = 0.f;
#pragma unroll
    for (int i = 0; i < SF::S; ++i) acc += st[i];
    sink[blockIdx.x * blockDim.x + threadIdx.x] = acc;
}

template <int D, int N, int Q>
void run(const char* name, float* sink, const float* in) {
    using SF = SliceFold<float, D, N, Q>;
    int sms = 0, clk = 0;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, 0);
    for (int w : {1, 2, 3, 4}) {
        const int threads = 128 * w > 256 ? 256 : 128 * w;
        const int blocks = sms * (128 * w) / threads;
        const int steps = 2000;
        cudaEvent_t e0, e1;
        cudaEventCreate(&e0);
        cudaEventCreate(&e1);
        stepk<D, N, Q><<<blocks, threads>>>(sink, in, 10);
        cudaEventRecord(e0);
        stepk<D, N, Q><<<blocks, threads>>>(sink, in, steps);
        cudaEventRecord(e1);
        cudaEventSynchronize(e1);
        float ms;
        cudaEventElapsedTime(&ms, e0, e1);
        const double ops = (double)blocks * threads * steps * SF::ops_per_step();
        const double per_sm_cycle = ops / (ms * 1e-3) / sms / (clk * 1e3);
        printf("%s warps/SMSP=%d  ops/SM/cycle(at max clk)=%.1f of 128  (%.2f ms) %s\n", name, w, per_sm_cycle, ms,
               cudaGetErrorString(cudaGetLastError()));
    }
}

int main() {
    float *sink, *in;
    cudaMalloc(&sink, 148 * 1024 * sizeof(float));
    cudaMalloc(&in, 64 * sizeof(float));
    float h[64];
    for (int i = 0; i < 64; ++i) h[i] = 0.01f * (i % 7);
    cudaMemcpy(in, h, sizeof(h), cudaMemcpyHostToDevice);
    run<5, 4, 1>("d5N4Q1", sink, in);
    run<5, 4, 2>("d5N4Q2", sink, in);
    run<8, 4, 2>("d8N4Q2", sink, in);
    run<2, 4, 0>("d2N4Q0", sink, in);
    return 0;
}
