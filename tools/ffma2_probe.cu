// Microbenchmark: packed FP32 (FFMA2, PTX fma.rn.f32x2, sm_100a) vs scalar
// FFMA issue/FMA rates for the operand patterns a Horner step could use.
//   mode 0: scalar  r = fma(r, a, b)                 (uniform operands: the FFMA peak)
//   mode 1: scalar  acc[j] = fma(u[j%4], v[j/4], acc[j])   (outer-product tile)
//   mode 2: packed  r2 = fma2(r2, a2, b2)             (loop-invariant pairs)
//   mode 3: packed  acc2[j] = fma2(u2[j%4], v2[j/4], acc2[j])  (outer-product tile of pairs)
//   mode 4: packed  acc2[j] = fma2(u2[j%4], {v[j/4], v[j/4]}, acc2[j])  (broadcast operand)
// FMAs counted per lane: 1 per FFMA, 2 per FFMA2.
//   nvcc -O3 -gencode arch=compute_100a,code=sm_100a tools/ffma2_probe.cu -o tools/ffma2_probe
#include <cstdio>
#include <cuda_runtime.h>

__device__ __forceinline__ unsigned long long pk(float lo, float hi) {
    unsigned long long r;
    asm("mov.b64 %0, {%1, %2};" : "=l"(r) : "f"(lo), "f"(hi));
    return r;
}
__device__ __forceinline__ void upk(unsigned long long v, float& lo, float& hi) {
    asm("mov.b64 {%0, %1}, %2;" : "=f"(lo), "=f"(hi) : "l"(v));
}
__device__ __forceinline__ unsigned long long fma2(unsigned long long a, unsigned long long b, unsigned long long c) {
    unsigned long long r;
    asm("fma.rn.f32x2 %0, %1, %2, %3;" : "=l"(r) : "l"(a), "l"(b), "l"(c));
    return r;
}

template <int MODE>
__global__ void k(float* sink, const float* __restrict__ in, int iters) {
    const int t = threadIdx.x;
    float s = 0.f;
    if (MODE == 0) {
        float r[16];
#pragma unroll
        for (int j = 0; j < 16; ++j) r[j] = in[(t + j) & 255];
        const float a = in[1], b = in[2];
#pragma unroll 1
        for (int i = 0; i < iters; ++i)
#pragma unroll
            for (int rep = 0; rep < 2; ++rep)
#pragma unroll
                for (int j = 0; j < 16; ++j) r[j] = fmaf(r[j], a, b);
#pragma unroll
        for (int j = 0; j < 16; ++j) s += r[j];
    } else if (MODE == 1) {
        float acc[32], u[4], v[8];
#pragma unroll
        for (int j = 0; j < 32; ++j) acc[j] = in[(t + j) & 255];
#pragma unroll
        for (int j = 0; j < 8; ++j) v[j] = in[(t * 3 + j) & 255];
#pragma unroll
        for (int j = 0; j < 4; ++j) u[j] = in[(t * 5 + j) & 255];
        const float a = in[1], b = in[2];
#pragma unroll 1
        for (int i = 0; i < iters; ++i) {
#pragma unroll
            for (int j = 0; j < 32; ++j) acc[j] = fmaf(u[j & 3], v[j >> 2], acc[j]);
            u[0] = acc[3] * a + b;
        }
#pragma unroll
        for (int j = 0; j < 32; ++j) s += acc[j];
    } else if (MODE == 2) {
        unsigned long long r[16];
#pragma unroll
        for (int j = 0; j < 16; ++j) r[j] = pk(in[(t + j) & 255], in[(t + j + 1) & 255]);
        const unsigned long long a = pk(in[1], in[3]), b = pk(in[2], in[4]);
#pragma unroll 1
        for (int i = 0; i < iters; ++i)
#pragma unroll
            for (int j = 0; j < 16; ++j) r[j] = fma2(r[j], a, b);
#pragma unroll
        for (int j = 0; j < 16; ++j) { float lo, hi; upk(r[j], lo, hi); s += lo + hi; }
    } else if (MODE == 3 || MODE == 4) {
        unsigned long long acc[16], u[4], v[4];
        float vs[4];
#pragma unroll
        for (int j = 0; j < 16; ++j) acc[j] = pk(in[(t + j) & 255], in[(t + j + 7) & 255]);
#pragma unroll
        for (int j = 0; j < 4; ++j) { v[j] = pk(in[(t * 3 + j) & 255], in[(t * 3 + j + 1) & 255]); vs[j] = in[(t * 7 + j) & 255]; }
#pragma unroll
        for (int j = 0; j < 4; ++j) u[j] = pk(in[(t * 5 + j) & 255], in[(t * 5 + j + 2) & 255]);
        const unsigned long long ab = pk(in[1], in[1]), bb = pk(in[2], in[2]);
#pragma unroll 1
        for (int i = 0; i < iters; ++i) {
#pragma unroll
            for (int j = 0; j < 16; ++j) {
                if (MODE == 3) acc[j] = fma2(u[j & 3], v[j >> 2], acc[j]);
                else acc[j] = fma2(u[j & 3], pk(vs[j >> 2], vs[j >> 2]), acc[j]);
            }
            u[0] = fma2(acc[3], ab, bb);
        }
#pragma unroll
        for (int j = 0; j < 16; ++j) { float lo, hi; upk(acc[j], lo, hi); s += lo + hi; }
    }
    sink[blockIdx.x * blockDim.x + t] = s;
}

// FMAs per lane per iteration
constexpr double fmas(int mode) { return mode == 0 ? 32 : mode == 1 ? 32 : 32; }

template <int MODE>
double run(int warps_per_smsp, float* sink, const float* in, int sms) {
    const int threads = 128 * warps_per_smsp > 1024 ? 1024 : 128 * warps_per_smsp;
    const int blocks = sms * (128 * warps_per_smsp) / threads;
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
    const double flops = 2.0 * blocks * threads * (double)iters * fmas(MODE);
    return flops / (ms * 1e-3) / 1e12;
}

int main() {
    float *sink, *in;
    int sms = 0;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    cudaMalloc(&sink, sms * 1024 * 8 * sizeof(float));
    cudaMalloc(&in, 256 * sizeof(float));
    float h[256];
    for (int i = 0; i < 256; ++i) h[i] = 1e-3f * (i % 17);
    cudaMemcpy(in, h, sizeof(h), cudaMemcpyHostToDevice);
    printf("TFLOP/s  (FMA=2 flops; FFMA2 = 2 FMAs)\n");
    for (int w : {1, 2, 4, 8}) {
        printf("warps/SMSP=%d  ffma-uniform %.1f  ffma-outer %.1f  ffma2-uniform %.1f  ffma2-outer %.1f  ffma2-bcast %.1f\n", w,
               run<0>(w, sink, in, sms), run<1>(w, sink, in, sms), run<2>(w, sink, in, sms), run<3>(w, sink, in, sms),
               run<4>(w, sink, in, sms));
    }
    printf("%s\n", cudaGetErrorString(cudaGetLastError()));
    return 0;
}
