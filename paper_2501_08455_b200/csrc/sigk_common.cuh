// Shared helpers for the sm_100a signature kernels.
#pragma once

#include <cstddef>
#include <cstdint>
#include <cuda_runtime.h>

namespace sigk {

__host__ __device__ constexpr int ipow(int b, int e) {
    int r = 1;
    for (int i = 0; i < e; ++i) r *= b;
    return r;
}

__host__ __device__ constexpr int round_up(int x, int m) { return (x + m - 1) / m * m; }

// Flat signature layout (reference tensor_algebra.hpp:25-42, sig_core.hpp:7-10):
// level n occupies [off(n-1), off(n)) with off(0) = 0, off(N) = D; inside a
// level the multi-index (i_1..i_n) sits at sum_m i_m d^(n-m), i_1 = earliest
// increment, last index fastest.
__host__ __device__ constexpr int level_off(int d, int n) {  // start of degree n+1
    int o = 0, p = 1;
    for (int m = 1; m <= n; ++m) {
        p *= d;
        o += p;
    }
    return o;
}

// Programmatic dependent launch (sm_90+): let the next kernel on the stream be
// scheduled now / wait until the previous kernel on the stream has completed
// and its memory is visible. Both are no-ops for an ordinary launch.
__device__ __forceinline__ void pdl_trigger() { asm volatile("griddepcontrol.launch_dependents;" ::: "memory"); }
__device__ __forceinline__ void pdl_wait() { asm volatile("griddepcontrol.wait;" ::: "memory"); }

// Vector width (in elements) of one 16-byte shared-memory access.
template <typename Real>
struct Vec16;
template <>
struct Vec16<float> {
    using type = float4;
    static constexpr int n = 4;
};
template <>
struct Vec16<double> {
    using type = double2;
    static constexpr int n = 2;
};

}  // namespace sigk
