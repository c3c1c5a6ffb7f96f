// Compile-time variant table: one register-sliced fold kernel per
// (precision, d, N), with the prefix length Q picked so the per-thread slice
// fits the register budget, and the kernel family picked by unit size.
#pragma once

#include <cuda_runtime.h>

#include <atomic>
#include <cstdint>

#include "flat_kernel.cuh"
#include "ipair_kernel.cuh"
#include "pair_kernel.cuh"
#include "ppair_kernel.cuh"
#include "path_kernel.cuh"
#include "stream_kernel.cuh"
#include "variants.h"
#include "vjp_prep.cuh"

namespace sigk {

// Smallest Q whose per-thread state (in 32-bit registers) fits the budget.
template <typename Real>
constexpr int pick_q(int d, int N) {
    constexpr int budget = 160;  // 32-bit registers of state per thread
    for (int q = 0; q < N; ++q) {
        int s = q > 1 ? q - 1 : 0;
        for (int n = (q > 1 ? q : 1); n <= N; ++n) s += ipow(d, n - q);
        if (s * (int)(sizeof(Real) / 4) <= budget) return q;
    }
    return N - 1;
}

// Opt a kernel in to > 48 KB of dynamic shared memory once per device (not
// stream-ordered, so it must not be repeated inside a graph capture).
template <typename K>
cudaError_t opt_in_smem(K kern, size_t bytes, std::atomic<uint64_t>& done) {
    int dev = 0;
    cudaGetDevice(&dev);
    const uint64_t bit = 1ull << (dev & 63);
    if (bytes <= 48 * 1024 || (done.load() & bit)) return cudaSuccess;
    int optin = 0;
    cudaDeviceGetAttribute(&optin, cudaDevAttrMaxSharedMemoryPerBlockOptin, dev);
    cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, optin);
    if (e == cudaSuccess) done.fetch_or(bit);
    return e;
}

// Launch, optionally as a programmatic dependent launch (PDL): the grid may
// start while the previous kernel on the stream is still running. The fold
// kernels trigger their dependents at entry and execute griddepcontrol.wait
// before their first global write, so only the output write is ordered after
// the predecessor; the caller (sigk_abi.cu) enables this only when the input
// cannot be the predecessor's output.
template <typename K, typename... Args>
cudaError_t launch_maybe_overlapped(K kern, dim3 grid, dim3 block, size_t smem, cudaStream_t s, bool overlap,
                                    Args... args) {
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = grid;
    cfg.blockDim = block;
    cfg.dynamicSmemBytes = smem;
    cfg.stream = s;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    attr[0].val.programmaticStreamSerializationAllowed = 1;
    cfg.attrs = attr;
    cfg.numAttrs = overlap ? 1 : 0;
    return cudaLaunchKernelEx(&cfg, kern, args...);
}

template <typename Real, int DIM, int DEPTH, int Q>
struct PathVariant {
    using G = PathGeom<Real, DIM, DEPTH, Q>;
    using SF = typename G::SF;
    // Register budget from the slice size: small slices get 512-thread CTAs, mid
    // slices 256 threads at >= 2 CTAs/SM (both <= 128 registers per thread), big
    // slices 256 threads with up to 255 registers.
    static constexpr int S32 = SF::S * (int)(sizeof(Real) / 4);
    static constexpr int NTMAX = S32 <= 48 ? 512 : 256;
    static constexpr int MINB = (S32 > 48 && S32 <= 96) ? 2 : 1;
    static constexpr int T = G::tile_steps();
    static constexpr bool PIPE = !(S32 > 48 && S32 <= 96);  // mid slices: more warps instead
    static constexpr auto kernel = path_kernel<Real, DIM, DEPTH, Q, NTMAX, T, MINB, PIPE>;
    static std::atomic<uint64_t> smem_done;

    static cudaError_t launch(const void* X, int64_t B, int64_t L, int U, void* out, cudaStream_t s, void* phases,
                              bool overlap) {
        const int64_t M = L - 1;
        const int CL = (int)((M + U - 1) / U);
        const size_t smem = G::smem_bytes(T, U);
        cudaError_t e = opt_in_smem(kernel, smem, smem_done);
        if (e != cudaSuccess) return e;
        return launch_maybe_overlapped(kernel, dim3((unsigned)B), dim3(U * SF::P), smem, s, overlap,
                                       static_cast<const Real*>(X), L, U, CL, static_cast<Real*>(out),
                                       static_cast<long long*>(phases));
    }
    static cudaError_t occupancy(int U, int* blocks) {
        const size_t smem = G::smem_bytes(T, U);
        cudaError_t e = opt_in_smem(kernel, smem, smem_done);
        if (e != cudaSuccess) return e;
        return cudaOccupancyMaxActiveBlocksPerMultiprocessor(blocks, kernel, U * SF::P, smem);
    }
};
template <typename Real, int DIM, int DEPTH, int Q>
std::atomic<uint64_t> PathVariant<Real, DIM, DEPTH, Q>::smem_done{0};

template <typename Real, int DIM, int DEPTH, int Q>
struct FlatVariant {
    static constexpr int NT = 32;
    static constexpr int T = 8;
    static constexpr int MINB = 14;
    using G = FlatGeom<Real, DIM, DEPTH, Q, NT, T>;
    using SF = typename G::SF;
    static constexpr auto kernel = flat_kernel<Real, DIM, DEPTH, Q, NT, T, MINB>;
    static std::atomic<uint64_t> smem_done;

    static cudaError_t launch(const void* X, int64_t B, int64_t L, int, void* out, cudaStream_t s, void*,
                              bool overlap) {
        cudaError_t e = opt_in_smem(kernel, G::smem, smem_done);
        if (e != cudaSuccess) return e;
        const int64_t lanes = B * (int64_t)SF::P;
        return launch_maybe_overlapped(kernel, dim3((unsigned)((lanes + NT - 1) / NT)), dim3(NT), G::smem, s, overlap,
                                       static_cast<const Real*>(X), B, L, static_cast<Real*>(out));
    }
    static cudaError_t occupancy(int, int* blocks) {
        cudaError_t e = opt_in_smem(kernel, G::smem, smem_done);
        if (e != cudaSuccess) return e;
        return cudaOccupancyMaxActiveBlocksPerMultiprocessor(blocks, kernel, NT, G::smem);
    }
};
template <typename Real, int DIM, int DEPTH, int Q>
std::atomic<uint64_t> FlatVariant<Real, DIM, DEPTH, Q>::smem_done{0};

// Pair family (fp32 only): 256-thread CTAs, two per SM (<= 128 registers).
template <int DIM, int DEPTH, int Q>
struct PairVariant {
    using PF = PairFold<DIM, DEPTH, Q>;
    static constexpr int NT = 256;
    static constexpr int MINB = 2;
    static constexpr auto kernel = pair_kernel<DIM, DEPTH, Q, NT, MINB>;
    static constexpr auto ckernel = pair_kernel<DIM, DEPTH, Q, NT, MINB, true>;  // cluster segment combine
    static std::atomic<uint64_t> smem_done, csmem_done, psmem_done, pcsmem_done;
    // position-table fold with a producer warp (ppair_kernel.cuh): Q >= 1, P1S shapes
    static constexpr bool HAS_POS = Q >= 1 && Q < DEPTH && DIM > 1 && ipow(DIM, Q) <= 128;
    static constexpr int QP = HAS_POS ? Q : 1;
    static constexpr int NFP = 128;  // fold threads of a position-table CTA (+ 1 producer warp)
    static constexpr int TSP = 16;   // steps per table tile
    static constexpr auto pkernel = ppair_kernel<HAS_POS ? DIM : 2, HAS_POS ? DEPTH : 2, QP, NFP + 32, 3, TSP>;
    static constexpr auto pckernel = ppair_kernel<HAS_POS ? DIM : 2, HAS_POS ? DEPTH : 2, QP, NFP + 32, 3, TSP, true>;
    static size_t psmem(int U, int64_t SL, int G, bool cluster) {
        return ppair_smem_bytes<HAS_POS ? DIM : 2, HAS_POS ? DEPTH : 2, QP>(U, TSP, raw_floats(SL), G, cluster);
    }

    static int raw_floats(int64_t SL) { return (int)(((SL + 1) * DIM + 3) / 4 * 4); }
    static size_t smem(int U, int CL, int64_t SL, int G, bool cluster = false) {
        return pair_smem_bytes<DIM, DEPTH, Q>(U, CL, raw_floats(SL), G, cluster);
    }
    static int threads(int U) { return (U / 2 * PF::P + 31) / 32 * 32; }

    static cudaError_t launch(const PairLaunch& a) {
        PairGeom g;
        g.G = a.G;
        g.SL = a.SL;
        g.U = a.U;
        g.UP = a.U / 2;
        g.CL = a.CL;
        g.threads = threads(a.U);
        g.raw_floats = raw_floats(a.SL);
        g.phases = static_cast<long long*>(a.phases);
        g.counters = static_cast<int*>(a.counters);
        g.final_out = static_cast<float*>(a.out);
        g.sub_U = a.sub_U;
        g.sub_CL = a.sub_CL;
        g.sub_L = a.sub_L;
        const bool cl = a.cluster && a.G > 1;
        if (a.sub_U > 0 && a.pos) return cudaErrorInvalidValue;  // chunk paths: the table-fold kernel only
        if (a.pos) {  // position-table fold, producer warp
            if (!HAS_POS || g.threads > NFP) return cudaErrorInvalidValue;
            const size_t sm = psmem(a.U, a.SL, a.G, cl);
            g.smem_bytes = (int)sm;
            g.segrow_off = (int)ppair_segrow_off<HAS_POS ? DIM : 2, HAS_POS ? DEPTH : 2, QP>(a.U, TSP, raw_floats(a.SL), a.G);
            cudaError_t e = cl ? opt_in_smem(pckernel, sm, pcsmem_done) : opt_in_smem(pkernel, sm, psmem_done);
            if (e != cudaSuccess) return e;
            if (a.ev_fold_start) {
                if (a.capturing) cudaEventRecordWithFlags(static_cast<cudaEvent_t>(a.ev_fold_start), a.s, cudaEventRecordExternal);
                else cudaEventRecord(static_cast<cudaEvent_t>(a.ev_fold_start), a.s);
            }
            cudaLaunchConfig_t cfg = {};
            cfg.gridDim = dim3((unsigned)(a.B * a.G));
            cfg.blockDim = dim3(g.threads + 32);
            cfg.dynamicSmemBytes = sm;
            cfg.stream = a.s;
            cudaLaunchAttribute attr[2];
            int na = 0;
            if (cl) {
                attr[na].id = cudaLaunchAttributeClusterDimension;
                attr[na].val.clusterDim.x = (unsigned)a.G;
                attr[na].val.clusterDim.y = 1;
                attr[na].val.clusterDim.z = 1;
                ++na;
            }
            if (a.overlap && !a.ev_fold_start) {
                attr[na].id = cudaLaunchAttributeProgrammaticStreamSerialization;
                attr[na].val.programmaticStreamSerializationAllowed = 1;
                ++na;
            }
            cfg.attrs = attr;
            cfg.numAttrs = na;
            float* dst = static_cast<float*>(a.G > 1 && !cl ? a.scratch : a.out);
            e = cudaLaunchKernelEx(&cfg, cl ? pckernel : pkernel, static_cast<const float*>(a.X), a.L, g, dst);
            if (a.ev_fold_stop) {
                if (a.capturing) cudaEventRecordWithFlags(static_cast<cudaEvent_t>(a.ev_fold_stop), a.s, cudaEventRecordExternal);
                else cudaEventRecord(static_cast<cudaEvent_t>(a.ev_fold_stop), a.s);
            }
            return e;
        }
        if (g.threads > NT) return cudaErrorInvalidValue;
        const size_t sm = smem(a.U, a.CL, a.SL, a.G, cl);
        g.smem_bytes = (int)sm;
        g.segrow_off = (int)pair_segrow_off<DIM, DEPTH, Q>(a.U, a.CL, raw_floats(a.SL), a.G);
        cudaError_t e = cl ? opt_in_smem(ckernel, sm, csmem_done) : opt_in_smem(kernel, sm, smem_done);
        if (e != cudaSuccess) return e;
        auto record = [&](void* ev) {
            if (!ev) return;
            if (a.capturing) cudaEventRecordWithFlags(static_cast<cudaEvent_t>(ev), a.s, cudaEventRecordExternal);
            else cudaEventRecord(static_cast<cudaEvent_t>(ev), a.s);
        };
        record(a.ev_fold_start);
        if (cl) {  // the path's G segment CTAs form one cluster
            cudaLaunchConfig_t cfg = {};
            cfg.gridDim = dim3((unsigned)(a.B * a.G));
            cfg.blockDim = dim3(g.threads);
            cfg.dynamicSmemBytes = sm;
            cfg.stream = a.s;
            cudaLaunchAttribute attr[2];
            attr[0].id = cudaLaunchAttributeClusterDimension;
            attr[0].val.clusterDim.x = (unsigned)a.G;
            attr[0].val.clusterDim.y = 1;
            attr[0].val.clusterDim.z = 1;
            attr[1].id = cudaLaunchAttributeProgrammaticStreamSerialization;
            attr[1].val.programmaticStreamSerializationAllowed = 1;
            cfg.attrs = attr;
            cfg.numAttrs = (a.overlap && !a.ev_fold_start) ? 2 : 1;
            e = cudaLaunchKernelEx(&cfg, ckernel, static_cast<const float*>(a.X), a.L, g, static_cast<float*>(a.out));
        } else {
            float* dst = static_cast<float*>(a.G > 1 ? a.scratch : a.out);
            e = launch_maybe_overlapped(kernel, dim3((unsigned)(a.B * a.G)), dim3(g.threads), sm, a.s,
                                        a.overlap && !a.ev_fold_start, static_cast<const float*>(a.X), a.L, g, dst);
        }
        record(a.ev_fold_stop);
        return e;
    }
    static cudaError_t pos_occupancy(int U, int CL, int64_t SL, int G, bool cluster, int* blocks) {
        (void)CL;
        const bool cl = cluster && G > 1 && G <= kMaxPairCluster;
        const size_t sm = psmem(U, SL, G, cl);
        *blocks = 0;
        if (!HAS_POS || sm > 227 * 1024 || threads(U) > NFP) return cudaSuccess;
        cudaError_t e = cl ? opt_in_smem(pckernel, sm, pcsmem_done) : opt_in_smem(pkernel, sm, psmem_done);
        if (e != cudaSuccess) return e;
        return cudaOccupancyMaxActiveBlocksPerMultiprocessor(blocks, cl ? pckernel : pkernel, threads(U) + 32, sm);
    }
    static cudaError_t occupancy(int U, int CL, int64_t SL, int G, bool cluster, int* blocks) {
        const bool cl = cluster && G > 1 && G <= kMaxPairCluster;
        const size_t sm = smem(U, CL, SL, G, cl);
        *blocks = 0;
        if (sm > 227 * 1024 || threads(U) > NT) return cudaSuccess;
        cudaError_t e = cl ? opt_in_smem(ckernel, sm, csmem_done) : opt_in_smem(kernel, sm, smem_done);
        if (e != cudaSuccess) return e;
        return cudaOccupancyMaxActiveBlocksPerMultiprocessor(blocks, cl ? ckernel : kernel, threads(U), sm);
    }

    // reverse mode's producer (vjp_prep.cuh), shapes with a slice walk only
    static constexpr bool HAS_VJP = vjp_slice_q(DIM, DEPTH) > 0;
    static std::atomic<uint64_t> vsmem_done;
    static size_t vjp_smem(int U, int CL, int64_t L) { return vjp_prep_smem<DIM, DEPTH, Q>(U, CL, raw_floats(L - 1)); }
    template <bool E = HAS_VJP>
    static cudaError_t vjp_launch(const void* X, int64_t B, int64_t L, int U, int CL, int R, const void* cot,
                                  void* ends, void* cbars, void* grad, cudaStream_t s) {
        if constexpr (E) {
            // 512 threads: the fold uses U/2 * P of them, the chunk passes all (<= 128 registers)
            constexpr int NTV = 512;
            constexpr auto k = pair_vjp_prep_kernel<DIM, DEPTH, Q, NTV>;
            PairGeom g{};
            g.G = 1;
            g.SL = L - 1;
            g.U = U;
            g.UP = U / 2;
            g.CL = CL;
            g.threads = threads(U);
            g.raw_floats = raw_floats(L - 1);
            if (U % 2 || g.threads > NT) return cudaErrorInvalidValue;
            const size_t sm = vjp_smem(U, CL, L);
            cudaError_t e = opt_in_smem(k, sm, vsmem_done);
            if (e != cudaSuccess) return e;
            k<<<(unsigned)B, NTV, sm, s>>>(static_cast<const float*>(X), L, g, R, static_cast<const float*>(cot),
                                                  static_cast<float*>(ends), static_cast<float*>(cbars),
                                                  static_cast<float*>(grad));
            return cudaGetLastError();
        } else {
            return cudaErrorNotSupported;
        }
    }

    // prefix stream: one CTA per path; the largest stage tile TS in {8, 4, 2, 1} that fits
    static constexpr auto skernel = pair_stream_kernel<DIM, DEPTH, Q, NT, MINB>;
    static std::atomic<uint64_t> ssmem_done;
    // stage tile (steps per chunk staged before the copy-out) the stream launch uses, 0 if nothing fits
    static int stream_tile_steps(int64_t L, int G, int U) {
        const int64_t M = L - 1;
        G = std::max(1, G);
        const int64_t SL = (M + G - 1) / G;
        U = std::max(2, U / 2 * 2);
        const int CL = (int)((SL + U - 1) / U);
        for (int TS = 8; TS >= 1; TS /= 2)
            if (stream_smem_bytes<DIM, DEPTH, Q>(U, CL, raw_floats(SL), TS) <= 227 * 1024) return TS;
        return 0;
    }
    static cudaError_t stream_launch(const void* X, int64_t B, int64_t L, int U, void* out, cudaStream_t s,
                                     bool overlap, int G, void* pub, int* flags, int epoch) {
        const int64_t M = L - 1;
        G = std::max(1, G);
        const int64_t SL = (M + G - 1) / G;
        U = std::max(2, U / 2 * 2);
        const int CL = (int)((SL + U - 1) / U);
        int TS = 8;
        size_t sm = 0;
        for (; TS >= 1; TS /= 2) {
            sm = stream_smem_bytes<DIM, DEPTH, Q>(U, CL, raw_floats(SL), TS);
            if (sm <= 227 * 1024) break;
        }
        if (TS < 1) return cudaErrorInvalidValue;
        cudaError_t e = opt_in_smem(skernel, sm, ssmem_done);
        if (e != cudaSuccess) return e;
        PairGeom g{};
        g.G = G;
        g.SL = SL;
        g.U = U;
        g.UP = U / 2;
        g.CL = CL;
        g.threads = threads(U);
        g.raw_floats = raw_floats(SL);
        g.pub = G > 1 ? static_cast<float*>(pub) : nullptr;
        g.flags = flags;
        g.epoch = epoch;
        return launch_maybe_overlapped(skernel, dim3((unsigned)(B * G)), dim3(g.threads), sm, s, overlap,
                                       static_cast<const float*>(X), L, g, TS, static_cast<float*>(out));
    }
};
template <int DIM, int DEPTH, int Q>
std::atomic<uint64_t> PairVariant<DIM, DEPTH, Q>::smem_done{0};
template <int DIM, int DEPTH, int Q>
std::atomic<uint64_t> PairVariant<DIM, DEPTH, Q>::csmem_done{0};
template <int DIM, int DEPTH, int Q>
std::atomic<uint64_t> PairVariant<DIM, DEPTH, Q>::psmem_done{0};
template <int DIM, int DEPTH, int Q>
std::atomic<uint64_t> PairVariant<DIM, DEPTH, Q>::pcsmem_done{0};
template <int DIM, int DEPTH, int Q>
std::atomic<uint64_t> PairVariant<DIM, DEPTH, Q>::ssmem_done{0};
template <int DIM, int DEPTH, int Q>
std::atomic<uint64_t> PairVariant<DIM, DEPTH, Q>::vsmem_done{0};

// Smallest Q whose pair state (two chunks) fits ~80 registers, or -1.
constexpr int pick_q_pair(int d, int N) {
    for (int q = 0; q < N && q <= 2; ++q) {
        int s = q > 1 ? q - 1 : 0;
        for (int n = (q > 1 ? q : 1); n <= N; ++n) s += ipow(d, n - q);
        if (2 * s <= 80 && ipow(d, q) <= 128) return q;
    }
    return -1;
}

template <int DIM, int DEPTH, int Q>
Variant make_pair_variant() {
    using PF = PairFold<DIM, DEPTH, Q>;
    using V = PairVariant<DIM, DEPTH, Q>;
    int chen = 0;
    for (int n = 2; n <= DEPTH; ++n) chen += (n - 2) * ipow(DIM, n);
    Variant v{DIM, DEPTH, Q, PF::P, PF::ops_per_step(), PF::loads_per_step(), chen, KernelFamily::Pair, V::NT, 0,
              nullptr, nullptr, nullptr, nullptr, 0, nullptr, 0, 0, nullptr, nullptr};
    v.pair_launch = &V::launch;
    v.pair_occupancy = &V::occupancy;
    v.pair_units_max = V::NT / PF::P;
    if constexpr (V::HAS_POS) {
        v.pos_ops = PosFold<DIM, DEPTH, V::QP>::ops_per_step();
        v.pos_units_max = V::NFP / PF::P;
        v.pair_pos_occupancy = &V::pos_occupancy;
    }
    v.stream_launch = &V::stream_launch;
    v.stream_tile_steps = &V::stream_tile_steps;
    if constexpr (V::HAS_VJP) {
        v.vjp_prep_launch = &V::template vjp_launch<true>;
        v.vjp_prep_smem = &V::vjp_smem;
    }
    return v;
}

// Inner-pair flat family (fp32, even d): 128-lane CTAs over (path, slice)
// lanes, no chunking; 4 CTAs/SM for small states, 3 for large ones.
template <int DIM, int DEPTH, int Q>
struct IPairVariant {
    using F = IPairFold<DIM, DEPTH, Q>;
    static constexpr int NT = 128;
    // steps per table tile: 32 (fewer barriers) unless the register-staged
    // producer entries per thread would exceed 8
    static constexpr int T = IPairGeom<DIM, DEPTH, Q, NT, 32>::EPT <= 8 ? 32 : 8;
    static constexpr int SF = Q + 2 * F::NVP;  // state floats
    static constexpr int MINB = SF <= 80 ? 4 : 3;
    using G = IPairGeom<DIM, DEPTH, Q, NT, T>;
    static constexpr auto kernel = ipair_kernel<DIM, DEPTH, Q, NT, T, MINB>;
    static std::atomic<uint64_t> smem_done;

    static cudaError_t launch(const void* X, int64_t B, int64_t L, int, void* out, cudaStream_t s, void*,
                              bool overlap) {
        cudaError_t e = opt_in_smem(kernel, G::smem, smem_done);
        if (e != cudaSuccess) return e;
        const int64_t lanes = B * (int64_t)F::P;
        return launch_maybe_overlapped(kernel, dim3((unsigned)((lanes + NT - 1) / NT)), dim3(NT), G::smem, s, overlap,
                                       static_cast<const float*>(X), B, L, static_cast<float*>(out));
    }
    static cudaError_t occupancy(int, int* blocks) {
        cudaError_t e = opt_in_smem(kernel, G::smem, smem_done);
        if (e != cudaSuccess) return e;
        return cudaOccupancyMaxActiveBlocksPerMultiprocessor(blocks, kernel, NT, G::smem);
    }
};
template <int DIM, int DEPTH, int Q>
std::atomic<uint64_t> IPairVariant<DIM, DEPTH, Q>::smem_done{0};

// Smallest Q >= 1 whose inner-pair state fits ~120 registers (even d only), or -1.
constexpr int pick_q_ipair(int d, int N) {
    if (d % 2 || d < 2 || N < 2) return -1;
    for (int q = 1; q < N; ++q) {
        int s = q;
        for (int n = q + 1; n <= N; ++n) s += ipow(d, n - q);
        if (s <= 120) return ipow(d, q) <= 4096 ? q : -1;
    }
    return -1;
}

template <int DIM, int DEPTH, int Q>
Variant make_ipair_variant() {
    using V = IPairVariant<DIM, DEPTH, Q>;
    using F = typename V::F;
    Variant v{DIM, DEPTH, Q, F::P, F::pipe_cycles(), 0, 0, KernelFamily::PFlat, V::NT, V::T,
              &V::launch, &V::occupancy, nullptr, nullptr, 0, nullptr, 0, 0, nullptr, nullptr};
    return v;
}

template <typename Real, int DIM, int DEPTH, int Q>
Variant make_variant() {
    using SF = SliceFold<Real, DIM, DEPTH, Q>;
    int chen = 0;
    for (int n = 2; n <= DEPTH; ++n) chen += (n - 1) * ipow(DIM, n);
    const int loads = SF::VEC / SF::VW + Q * (SF::SCW / SF::VW);
    if constexpr (SF::P > 256) {
        using V = FlatVariant<Real, DIM, DEPTH, Q>;
        return Variant{DIM, DEPTH, Q, SF::P, SF::ops_per_step(), loads, chen, KernelFamily::Flat, V::NT, V::T,
                       &V::launch, &V::occupancy, nullptr, nullptr, 0, nullptr, 0, 0, nullptr, nullptr};
    } else {
        using V = PathVariant<Real, DIM, DEPTH, Q>;
        return Variant{DIM, DEPTH, Q, SF::P, SF::ops_per_step(), loads, chen, KernelFamily::Path, V::NTMAX, V::T,
                       &V::launch, &V::occupancy, nullptr, nullptr, 0, nullptr, 0, 0, nullptr, nullptr};
    }
}

// Candidates per (precision, d, N): the smallest register-feasible prefix
// length Q0 and, when it still fits a CTA, Q0 + 1 (more threads per unit, so
// fewer sequence chunks and a cheaper merge tree at some redundant work). The
// planner (sigk_abi.cu) picks per call from a cycle model.
template <typename Real, int DIM, int DEPTH>
struct VariantImpl {
    static constexpr int Q0 = pick_q<Real>(DIM, DEPTH);
    static constexpr bool SECOND = DIM > 1 && Q0 + 1 < DEPTH && ipow(DIM, Q0 + 1) <= 256 && ipow(DIM, Q0) <= 256;
    static constexpr int QP = pick_q_pair(DIM, DEPTH);
    static constexpr bool PAIR = sizeof(Real) == 4 && QP >= 0;
    static constexpr int QI = pick_q_ipair(DIM, DEPTH);
    static constexpr bool IPAIR = sizeof(Real) == 4 && QI >= 1;
    static constexpr int count = (SECOND ? 2 : 1) + (PAIR ? 1 : 0) + (IPAIR ? 1 : 0);
    static void fill(Variant* out) {
        int i = 0;
        out[i++] = make_variant<Real, DIM, DEPTH, Q0>();
        if constexpr (SECOND) out[i++] = make_variant<Real, DIM, DEPTH, Q0 + 1>();
        if constexpr (PAIR) out[i++] = make_pair_variant<DIM, DEPTH, QP < 0 ? 0 : QP>();
        if constexpr (IPAIR) out[i++] = make_ipair_variant<DIM, DEPTH, QI < 1 ? 1 : QI>();
    }
};

// Registry filled by the per-(precision, d) translation units at load time.
void register_variants(const Variant* table, int n, bool is_f64);

template <typename Real, int DIM, int... Ns>
struct DimTable {
    static constexpr int count = (VariantImpl<Real, DIM, Ns>::count + ...);
    static const Variant* table() {
        static Variant t[count];
        static bool done = false;
        if (!done) {
            int i = 0;
            ((VariantImpl<Real, DIM, Ns>::fill(t + i), i += VariantImpl<Real, DIM, Ns>::count), ...);
            done = true;
        }
        return t;
    }
};

}  // namespace sigk

// (d, N) pairs with a register-sliced instantiation (anything else runs the
// shape-generic kernel). Each (precision, d) row is compiled as its own
// translation unit (variants_inst.cu) so the build parallelises.
#define SIGK_DEPTHS_1 1, 2, 3, 4, 5, 6
#define SIGK_DEPTHS_2 1, 2, 3, 4, 5, 6
#define SIGK_DEPTHS_3 1, 2, 3, 4, 5, 6
#define SIGK_DEPTHS_4 1, 2, 3, 4, 5, 6
#define SIGK_DEPTHS_5 1, 2, 3, 4, 5, 6
#define SIGK_DEPTHS_6 1, 2, 3, 4
#define SIGK_DEPTHS_7 1, 2, 3, 4
#define SIGK_DEPTHS_8 1, 2, 3, 4
#define SIGK_DEPTHS_10 1, 2, 3, 4, 5
#define SIGK_FAST_DIMS 1, 2, 3, 4, 5, 6, 7, 8, 10
