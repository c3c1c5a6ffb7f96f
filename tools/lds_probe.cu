// Microbenchmark: shared-memory load throughput (warp instructions per SM
// cycle) for broadcast patterns like the fold's table reads.
//   mode 0: LDS.32 one address per warp     mode 1: LDS.64 one address
//   mode 2: LDS.128 one address             mode 3: LDS.128 two addresses (25 + 7 lanes)
//   mode 4: LDS.64 two addresses            mode 5: LDS.128 32 consecutive addresses
//   nvcc -O3 -gencode arch=compute_100a,code=sm_100a tools/lds_probe.cu -o tools/lds_probe
#include <cstdio>
#include <cuda_runtime.h>

template <int MODE>
__global__ void __launch_bounds__(512) k(float* sink, int iters) {
    __shared__ __align__(16) float sm[4096];
    for (int i = threadIdx.x; i < 4096; i += blockDim.x) sm[i] = i * 1e-3f;
    __syncthreads();
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    int a;
    if (MODE == 3 || MODE == 4) a = (lane < 25 ? 0 : 48) + warp * 96;
    else if (MODE == 5) a = lane * 4;
    else a = warp * 96;
    float acc = 0.f;
    const float* p = sm + a;
#pragma unroll 1
    for (int i = 0; i < iters; ++i) {
        const int o = (i & 7) * 8;
#pragma unroll
        for (int j = 0; j < 8; ++j) {
            if (MODE == 0) acc += p[o + j];
            else if (MODE == 1 || MODE == 4) {
                const float2 v = *reinterpret_cast<const float2*>(p + o + 2 * (j & 3));
                acc += v.x + v.y;
            } else {
                const float4 v = *reinterpret_cast<const float4*>(p + o + 4 * (j & 1));
                acc += v.x + v.w;
            }
        }
    }
    sink[blockIdx.x * blockDim.x + threadIdx.x] = acc;
}

template <int MODE>
void run(const char* name, float* sink, int sms, int clk) {
    const int threads = 512, iters = 4000;
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    k<MODE><<<sms, threads>>>(sink, 10);
    cudaEventRecord(e0);
    k<MODE><<<sms, threads>>>(sink, iters);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms;
    cudaEventElapsedTime(&ms, e0, e1);
    const double winst = (double)(threads / 32) * iters * 8;  // per SM
    printf("%s: %.3f warp-LDS per SM cycle (at max clk)\n", name, winst / (ms * 1e-3 * clk * 1e3));
}

int main() {
    int sms = 0, clk = 0;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, 0);
    float* sink;
    cudaMalloc(&sink, sms * 512 * sizeof(float));
    run<0>("LDS.32  1 addr ", sink, sms, clk);
    run<1>("LDS.64  1 addr ", sink, sms, clk);
    run<2>("LDS.128 1 addr ", sink, sms, clk);
    run<3>("LDS.128 2 addrs", sink, sms, clk);
    run<4>("LDS.64  2 addrs", sink, sms, clk);
    run<5>("LDS.128 32 addrs", sink, sms, clk);
    return 0;
}
