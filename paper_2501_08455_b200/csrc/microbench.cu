// FP32 FFMA-pipe peak microbenchmark (the roofline denominator for the fold
// kernels; MEASURED_PEAKS.json carries HBM and bf16 tensor peaks only).
// Register-resident: 8 independent FMA chains per thread, no memory traffic
// except one store per thread so the chains are not dead code.
#include <cuda_runtime.h>

#include "../../include/sigk.h"

namespace {

__global__ void __launch_bounds__(256) ffma_kernel(float* __restrict__ sink, int iters, float a, float b) {
    float r0 = threadIdx.x * 1e-7f, r1 = r0 + 1e-3f, r2 = r0 + 2e-3f, r3 = r0 + 3e-3f;
    float r4 = r0 + 4e-3f, r5 = r0 + 5e-3f, r6 = r0 + 6e-3f, r7 = r0 + 7e-3f;
#pragma unroll 1
    for (int i = 0; i < iters; ++i) {
#pragma unroll
        for (int j = 0; j < 16; ++j) {
            r0 = fmaf(r0, a, b); r1 = fmaf(r1, a, b); r2 = fmaf(r2, a, b); r3 = fmaf(r3, a, b);
            r4 = fmaf(r4, a, b); r5 = fmaf(r5, a, b); r6 = fmaf(r6, a, b); r7 = fmaf(r7, a, b);
        }
    }
    sink[blockIdx.x * blockDim.x + threadIdx.x] = r0 + r1 + r2 + r3 + r4 + r5 + r6 + r7;
}

}  // namespace

extern "C" {

/* Launch ffma_kernel on `stream`: grid = blocks x 256 threads, each thread
 * iters*16*8 FFMAs. *flops receives 2 * total FFMAs. sink: blocks*256 floats. */
int sigk_bench_ffma(float* sink, int blocks, int iters, double* flops, void* stream) {
    ffma_kernel<<<blocks, 256, 0, static_cast<cudaStream_t>(stream)>>>(sink, iters, 0.999999f, 1e-6f);
    if (flops) *flops = 2.0 * blocks * 256.0 * iters * 16.0 * 8.0;
    return cudaGetLastError() == cudaSuccess ? SIGK_OK : SIGK_EDEVICE;
}

}  // extern "C"
