// Microbenchmark: FFMA issue rate for the operand patterns the fold uses.
//   mode 0: fma(r, const, const)            (constant-bank operands)
//   mode 1: acc[j] = fma(u, v[j], acc[j])   (3 register sources, u reusable)
//   mode 2: acc[j] = fma(u[j%4], v[j/4], acc[j]) (outer-product 4x8 tile)
// for 1, 2, 4, 8 warps per SMSP. nvcc -O3 -gencode arch=compute_100a,code=sm_100a tools/ffma_probe.cu -o tools/ffma_probe
#include <cstdio>
#include <cuda_runtime.h>

template <int MODE>
__global__ void k(float* sink, const float* __restrict__ in, int iters) {
    float acc[32];
    float v[8], u[4];
#pragma unroll
    for (int j = 0; j < 32; ++j) acc[j] = in[(threadIdx.x + j) & 255];
#pragma unroll
    for (int j = 0; j < 8; ++j) v[j] = in[(threadIdx.x * 3 + j) & 255];
#pragma unroll
    for (int j = 0; j < 4; ++j) u[j] = in[(threadIdx.x * 5 + j) & 255];
    const float a = in[1], b = in[2];
#pragma unroll 1
    for (int i = 0; i < iters; ++i) {
        if (MODE == 0) {
#pragma unroll
            for (int j = 0; j < 32; ++j) acc[j] = fmaf(acc[j], 0.999f, 1e-6f);
        } else if (MODE == 1) {
#pragma unroll
            for (int j = 0; j < 32; ++j) acc[j] = fmaf(u[0], v[j & 7], acc[j]);
            u[0] = acc[5];
        } else {
#pragma unroll
            for (int j = 0; j < 32; ++j) acc[j] = fmaf(u[j & 3], v[j >> 2], acc[j]);
            u[0] = acc[3] * a + b;
        }
    }
    float s = 0;
#pragma unroll
    for (int j = 0; j < 32; ++j) s += acc[j];
    sink[blockIdx.x * blockDim.x + threadIdx.x] = s;
}

template <int MODE>
double run(int warps_per_smsp, float* sink, const float* in) {
    const int threads = 128 * warps_per_smsp > 1024 ? 1024 : 128 * warps_per_smsp;
    const int blocks = 148 * (128 * warps_per_smsp) / threads;
    const int iters = 4000;
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    k<MODE><<<blocks, threads>>>(sink, in, 10);
    cudaEventRecord(e0);
    k<MODE><<<blocks, threads>>>(sink, in, iters);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms;
    cudaEventElapsedTime(&ms, e0, e1);
    const double flops = 2.0 * blocks * threads * (double)iters * 32;
    return flops / (ms * 1e-3) / 1e12;
}

int main() {
    float *sink, *in;
    cudaMalloc(&sink, 148 * 1024 * 8 * sizeof(float));
    cudaMalloc(&in, 256 * sizeof(float));
    float h[256];
    for (int i = 0; i < 256; ++i) h[i] = 1e-3f * (i % 17);
    cudaMemcpy(in, h, sizeof(h), cudaMemcpyHostToDevice);
    for (int w : {1, 2, 4, 8}) {
        printf("warps/SMSP=%d  const %.1f  reg-reuse %.1f  outer4x8 %.1f TFLOP/s\n", w, run<0>(w, sink, in),
               run<1>(w, sink, in), run<2>(w, sink, in));
    }
    return 0;
}
