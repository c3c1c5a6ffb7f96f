// Microbenchmark: FMA-pipe rate of scalar FFMA vs packed FFMA2 (fma.rn.f32x2)
// for operand patterns of a rank-1 update acc[j] += a * b, at 2 and 8 warps
// per SM sub-partition. Prints TFLOP/s (1 FFMA = 2 flops, 1 FFMA2 = 4).
//   P0 ffma  acc[j] = fma(acc[j], a, b)           uniform (peak reference)
//   P1 ffma  acc[j] = fma(a, v[j%8], acc[j])      a reused, v fresh
//   P2 ffma  acc[j] = fma(u[j/4], v[j%4], acc[j]) outer 4x4
//   P3 ffma2 acc[j] = fma2(acc[j], a2, b2)        uniform pairs
//   P4 ffma2 acc[j] = fma2(a2, v2[j%8], acc[j])   a2 reused, v2 fresh pairs
//   P5 ffma2 acc[j] = fma2(v2[j%8], s, acc[j])    scalar broadcast s reused
//   P6 ffma2 acc[j] = fma2(a2, s[j%8], acc[j])    a2 reused, broadcast s fresh
//   P7 ffma2 acc[j] = fma2(u2[j/4], v2[j%4], acc) outer 4x4 of pairs
//   nvcc -O3 -gencode arch=compute_100a,code=sm_100a tools/ffma_pattern_probe.cu -o tools/ffma_pattern_probe
#include <cstdio>
#include <cuda_runtime.h>

typedef unsigned long long u64;
__device__ __forceinline__ u64 pk(float lo, float hi) {
    u64 r;
    asm("mov.b64 %0, {%1, %2};" : "=l"(r) : "f"(lo), "f"(hi));
    return r;
}
__device__ __forceinline__ float sum2(u64 v) {
    float lo, hi;
    asm("mov.b64 {%0, %1}, %2;" : "=f"(lo), "=f"(hi) : "l"(v));
    return lo + hi;
}
__device__ __forceinline__ u64 fma2(u64 a, u64 b, u64 c) {
    u64 r;
    asm("fma.rn.f32x2 %0, %1, %2, %3;" : "=l"(r) : "l"(a), "l"(b), "l"(c));
    return r;
}

template <int P>
__global__ void k(float* sink, const float* __restrict__ in, int iters) {
    const int t = threadIdx.x;
    auto ld = [&](int i) { return in[(t * 7 + i) & 255]; };
    float s = 0.f;
    if constexpr (P <= 2) {
        float acc[32], v[8], u[8];
#pragma unroll
        for (int j = 0; j < 32; ++j) acc[j] = ld(j);
#pragma unroll
        for (int j = 0; j < 8; ++j) { v[j] = ld(40 + j); u[j] = ld(60 + j); }
        float a = ld(90), b = ld(91);
#pragma unroll 1
        for (int i = 0; i < iters; ++i) {
#pragma unroll
            for (int j = 0; j < 32; ++j) {
                if (P == 0) acc[j] = fmaf(acc[j], a, b);
                if (P == 1) acc[j] = fmaf(a, v[j & 7], acc[j]);
                if (P == 2) acc[j] = fmaf(u[(j >> 2) & 7], v[j & 3], acc[j]);
            }
            if (P == 1) a = acc[1];
            if (P == 2) u[0] = acc[1];
        }
#pragma unroll
        for (int j = 0; j < 32; ++j) s += acc[j];
    } else {
        u64 acc[16], v2[8], u2[4];
        float sc[8];
#pragma unroll
        for (int j = 0; j < 16; ++j) acc[j] = pk(ld(j), ld(j + 17));
#pragma unroll
        for (int j = 0; j < 8; ++j) { v2[j] = pk(ld(40 + j), ld(50 + j)); sc[j] = ld(70 + j); }
#pragma unroll
        for (int j = 0; j < 4; ++j) u2[j] = pk(ld(80 + j), ld(85 + j));
        u64 a2 = pk(ld(90), ld(92)), b2 = pk(ld(91), ld(93));
        float sb = ld(95);
#pragma unroll 1
        for (int i = 0; i < iters; ++i) {
#pragma unroll
            for (int j = 0; j < 16; ++j) {
                if (P == 3) acc[j] = fma2(acc[j], a2, b2);
                if (P == 4) acc[j] = fma2(a2, v2[j & 7], acc[j]);
                if (P == 5) acc[j] = fma2(v2[j & 7], pk(sb, sb), acc[j]);
                if (P == 6) acc[j] = fma2(a2, pk(sc[j & 7], sc[j & 7]), acc[j]);
                if (P == 7) acc[j] = fma2(u2[j >> 2], v2[j & 3], acc[j]);
            }
            if (P == 4 || P == 6) a2 = acc[1];
            if (P == 5) sb = sum2(acc[1]);
            if (P == 7) u2[0] = acc[1];
        }
#pragma unroll
        for (int j = 0; j < 16; ++j) s += sum2(acc[j]);
    }
    sink[blockIdx.x * blockDim.x + t] = s;
}

template <int P>
double run(int w, float* sink, const float* in, int sms) {
    const int threads = 128 * w > 1024 ? 1024 : 128 * w;
    const int blocks = sms * (128 * w) / threads;
    const int iters = 4000;
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    k<P><<<blocks, threads>>>(sink, in, 10);
    cudaEventRecord(e0);
    k<P><<<blocks, threads>>>(sink, in, iters);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms;
    cudaEventElapsedTime(&ms, e0, e1);
    return 2.0 * 32 * blocks * threads * (double)iters / (ms * 1e-3) / 1e12;
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
    for (int w : {1, 2, 4, 8}) {
        printf("w=%d P0 %.1f P1 %.1f P2 %.1f | P3 %.1f P4 %.1f P5 %.1f P6 %.1f P7 %.1f\n", w, run<0>(w, sink, in, sms),
               run<1>(w, sink, in, sms), run<2>(w, sink, in, sms), run<3>(w, sink, in, sms), run<4>(w, sink, in, sms),
               run<5>(w, sink, in, sms), run<6>(w, sink, in, sms), run<7>(w, sink, in, sms));
    }
    printf("%s\n", cudaGetErrorString(cudaGetLastError()));
    return 0;
}
