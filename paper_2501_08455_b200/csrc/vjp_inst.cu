// Compile-time (d, N) instantiations of the reverse-mode kernel (loops over
// levels unroll, level offsets fold to constants); shapes outside the list
// use the runtime-shape kernel.
#include "vjp_slice.cuh"

namespace sigk {

#define SIGK_VJP_SHAPES(X) \
    X(1, 1) X(1, 2) X(1, 3) X(1, 4) X(1, 5) X(1, 6) \
    X(2, 1) X(2, 2) X(2, 3) X(2, 4) X(2, 5) X(2, 6) \
    X(3, 1) X(3, 2) X(3, 3) X(3, 4) X(3, 5) X(3, 6) \
    X(4, 1) X(4, 2) X(4, 3) X(4, 4) X(4, 5) X(4, 6) \
    X(5, 1) X(5, 2) X(5, 3) X(5, 4) X(5, 5) \
    X(6, 1) X(6, 2) X(6, 3) X(6, 4) \
    X(7, 1) X(7, 2) X(7, 3) X(7, 4) \
    X(8, 1) X(8, 2) X(8, 3) X(8, 4) \
    X(10, 1) X(10, 2) X(10, 3)

template <typename Real>
static VjpKernelFn<Real> pick(int d, int N) {
#define SIGK_VJP_CASE(DD, NN) \
    if (d == DD && N == NN) return vjp_kernel<Real, DD, NN>;
    SIGK_VJP_SHAPES(SIGK_VJP_CASE)
#undef SIGK_VJP_CASE
    return vjp_kernel<Real, 0, 0>;
}

template <typename Real, int DD, int NN>
static void slice_case(int d, int N, VjpSlice<Real>& out) {
    constexpr int Q = vjp_slice_q(DD, NN);
    if constexpr (Q > 0) {
        if (d == DD && N == NN) {
            out.fn = vjp_slice_kernel<Real, DD, NN, Q>;
            out.slots = SliceLayout<DD, NN, Q>::SLOTS;
            out.passes = vjp_chunk_passes_kernel<Real, DD, NN>;
            out.scan = vjp_scan_passes_kernel<Real, DD, NN>;
        }
    }
}

template <typename Real>
static VjpSlice<Real> pick_slice(int d, int N) {
    VjpSlice<Real> r;
#define SIGK_VJP_SLICE(DD, NN) slice_case<Real, DD, NN>(d, N, r);
    SIGK_VJP_SHAPES(SIGK_VJP_SLICE)
#undef SIGK_VJP_SLICE
    return r;
}

#if SIGK_VJP_REAL_F32
VjpKernelFn<float> vjp_kernel_for_f32(int d, int N) { return pick<float>(d, N); }
VjpSlice<float> vjp_slice_for_f32(int d, int N) { return pick_slice<float>(d, N); }
#else
VjpKernelFn<double> vjp_kernel_for_f64(int d, int N) { return pick<double>(d, N); }
VjpSlice<double> vjp_slice_for_f64(int d, int N) { return pick_slice<double>(d, N); }
#endif

}  // namespace sigk
