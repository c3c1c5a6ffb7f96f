// C ABI (include/sigk.h): validation, dispatch, chunk planning, host staging
// and the multi-GPU batch-sharded driver.
//
// Validation mirrors the reference boundary (kernels.cpp:13-26,
// tensor_algebra.cpp:10-20): batch/len/dim >= 1 and depth >= 1 else
// SIGK_EDOMAIN; L == 1 returns the identity (zero rows, sig_core.hpp:201-206).
#include <algorithm>
#include <atomic>
#include <cmath>
#include <cstdio>
#include <cstring>
#include <mutex>
#include <string>
#include <thread>
#include <vector>

#include "../../include/sigk.h"
#include "generic.cuh"
#include "variants.h"

namespace sigk {

namespace {

thread_local std::string g_err;

int fail(int code, const std::string& msg) {
    g_err = msg;
    return code;
}

int cuda_fail(cudaError_t e, const char* what) {
    const int code = (e == cudaErrorMemoryAllocation) ? SIGK_ERESOURCE : SIGK_EDEVICE;
    return fail(code, std::string(what) + ": " + cudaGetErrorName(e) + " (" + cudaGetErrorString(e) + ")");
}

struct Registry {
    std::mutex mu;
    std::vector<Variant> f32, f64;
};

Registry& registry() {
    static Registry r;
    return r;
}

// Per-device cache of SM count and fold occupancy.
struct DeviceInfo {
    int sms = 0;
};

DeviceInfo device_info(int dev) {
    static std::mutex mu;
    static std::vector<DeviceInfo> cache;
    std::lock_guard<std::mutex> g(mu);
    if ((int)cache.size() <= dev) cache.resize(dev + 1);
    if (cache[dev].sms == 0) cudaDeviceGetAttribute(&cache[dev].sms, cudaDevAttrMultiProcessorCount, dev);
    return cache[dev];
}

}  // namespace

void register_variants(const Variant* table, int n, bool is_f64) {
    Registry& r = registry();
    std::lock_guard<std::mutex> g(r.mu);
    auto& v = is_f64 ? r.f64 : r.f32;
    for (int i = 0; i < n; ++i) v.push_back(table[i]);
}

static const Variant* find_variant(int d, int N, bool is_f64) {
    Registry& r = registry();
    std::lock_guard<std::mutex> g(r.mu);
    for (const Variant& v : is_f64 ? r.f64 : r.f32)
        if (v.d == d && v.N == N) return &v;
    return nullptr;
}

// Chunk count K for a (B, M) problem: minimise a cycle model of
//   fold  = ceil(CTAs / SMs) * NT * ceil(M/K) * ops / 128       (FFMA-pipe bound)
//   merge = K>1: ceil(B / SMs) * ((K-1) * chen * 4 / 128 + rounds * N * 600) + 4000
// where the merge term charges ~4 issue slots per Chen FMA (3 loads + fma),
// a barrier-plus-latency cost per tree level and one extra launch.
static int plan_chunks(const Variant& v, int64_t B, int64_t M, int sms, int occ) {
    if (M <= 1) return 1;
    const int kmax = (int)std::min<int64_t>(M, 512);
    double best = 1e300;
    int bestk = 1;
    for (int K = 1; K <= kmax; ++K) {
        const int64_t CL = (M + K - 1) / K;
        const int64_t lanes = B * K * (int64_t)v.P;
        const int64_t ctas = (lanes + v.NT - 1) / v.NT;
        const int64_t per_sm = (ctas + sms - 1) / sms;
        // partial residency: fewer resident warps than the FMA latency needs
        const double fill = std::min(1.0, (double)std::min<int64_t>(per_sm, occ) * v.NT / 256.0);
        double t = (double)per_sm * v.NT * CL * v.ops / 128.0 / std::max(fill, 0.25);
        if (K > 1) {
            int rounds = 0;
            while ((1 << rounds) < K) ++rounds;
            t += (double)((B + sms - 1) / sms) * ((K - 1) * (double)v.chen * 4.0 / 128.0 + rounds * v.N * 600.0) + 4000.0;
        }
        if (t < best * 0.999) {
            best = t;
            bestk = K;
        }
    }
    return bestk;
}

template <typename Real>
static int run_device(const Real* X, int64_t B, int64_t L, int d, int N, Real* out, cudaStream_t s,
                      const sigk_tuning* tun, sigk_stats* st) {
    const bool is_f64 = sizeof(Real) == 8;
    const int64_t D = [&] {
        int64_t t = 0, p = 1;
        for (int n = 0; n < N; ++n) {
            p *= d;
            t += p;
        }
        return t;
    }();
    sigk_stats local{};
    const int64_t M = L - 1;
    cudaError_t e;
    if (M == 0) {  // identity signature
        e = cudaMemsetAsync(out, 0, sizeof(Real) * B * D, s);
        if (e != cudaSuccess) return cuda_fail(e, "memset");
        local.chunks = 1;
        local.prefix_len = 0;
        local.threads_per_unit = 1;
        if (st) *st = local;
        return SIGK_OK;
    }
    const Variant* v = (tun && tun->force_generic) ? nullptr : find_variant(d, N, is_f64);
    if (v == nullptr) {
        e = is_f64 ? launch_generic_f64(X, B, L, d, N, out, s) : launch_generic_f32(X, B, L, d, N, out, s);
        if (e != cudaSuccess) return cuda_fail(e, "generic fold launch");
        local.fold_steps = M;
        local.chunks = 1;
        local.prefix_len = -1;
        local.threads_per_unit = 0;
        local.launches = 1;
        if (st) *st = local;
        return SIGK_OK;
    }
    int dev = 0;
    cudaGetDevice(&dev);
    const DeviceInfo di = device_info(dev);
    int occ = 1;
    e = v->occupancy(&occ);
    if (e != cudaSuccess) return cuda_fail(e, "occupancy query");
    if (occ < 1) return fail(SIGK_ERESOURCE, "fold variant does not fit on this device");
    const int64_t plan_rows = (tun && tun->plan_rows > 0) ? tun->plan_rows : B;
    int K = (tun && tun->chunks > 0) ? tun->chunks : plan_chunks(*v, plan_rows, M, di.sms, occ);
    K = (int)std::max<int64_t>(1, std::min<int64_t>(K, M));
    const int CL = (int)((M + K - 1) / K);
    K = (int)((M + CL - 1) / CL);  // drop empty trailing chunks
    cudaEvent_t ev0 = tun ? static_cast<cudaEvent_t>(tun->fold_event_start) : nullptr;
    cudaEvent_t ev1 = tun ? static_cast<cudaEvent_t>(tun->fold_event_stop) : nullptr;
    cudaStreamCaptureStatus cap = cudaStreamCaptureStatusNone;
    if (ev0 || ev1) cudaStreamIsCapturing(s, &cap);
    auto record = [&](cudaEvent_t ev) {  // an event-record node when captured into a graph
        if (cap == cudaStreamCaptureStatusActive) cudaEventRecordWithFlags(ev, s, cudaEventRecordExternal);
        else cudaEventRecord(ev, s);
    };
    auto fold = [&](void* dst, int k) {
        if (ev0) record(ev0);
        cudaError_t r = v->fold(X, B, L, k, CL, dst, s);
        if (ev1) record(ev1);
        return r;
    };
    if (K == 1) {
        e = fold(out, 1);
        if (e != cudaSuccess) return cuda_fail(e, "fold launch");
        local.launches = 1;
    } else {
        Real* ws = nullptr;
        e = cudaMallocAsync(reinterpret_cast<void**>(&ws), sizeof(Real) * B * K * D, s);
        if (e != cudaSuccess) return cuda_fail(e, "workspace allocation");
        e = fold(ws, K);
        if (e == cudaSuccess) e = v->merge(ws, K, out, B, s);
        cudaError_t e2 = cudaFreeAsync(ws, s);
        if (e != cudaSuccess) return cuda_fail(e, "fold/merge launch");
        if (e2 != cudaSuccess) return cuda_fail(e2, "workspace free");
        local.launches = 2;
    }
    int rounds = 0;
    while ((1 << rounds) < K) ++rounds;
    local.fold_steps = CL;
    local.scan_passes = rounds;
    local.chunks = K;
    local.prefix_len = v->Q;
    local.threads_per_unit = v->P;
    if (st) *st = local;
    return SIGK_OK;
}

static int validate(const void* X, size_t B, size_t L, int d, int N, const void* out) {
    if (B < 1 || L < 1 || d < 1)
        return fail(SIGK_EDOMAIN, "paths: batch, len and dim must all be >= 1");
    if (N < 1) return fail(SIGK_EDOMAIN, "depth must be >= 1, got " + std::to_string(N));
    if (X == nullptr || out == nullptr) return fail(SIGK_EDOMAIN, "paths/out pointer is null");
    long double D = 0, p = 1;
    for (int n = 0; n < N; ++n) {
        p *= d;
        D += p;
    }
    if (D * (long double)B > 9.0e18L || (long double)B * L * d > 9.0e18L)
        return fail(SIGK_ERESOURCE, "signature size overflows 64-bit indexing");
    if (D > 2147483647.0L) return fail(SIGK_ERESOURCE, "signature width exceeds 2^31 coefficients");
    return SIGK_OK;
}

template <typename Real>
static int signature_impl(const Real* X, size_t B, size_t L, int d, int N, Real* out, unsigned flags,
                          void* stream, const sigk_tuning* tun, sigk_stats* st) {
    g_err.clear();
    int rc = validate(X, B, L, d, N, out);
    if (rc != SIGK_OK) return rc;
    cudaStream_t s = static_cast<cudaStream_t>(stream);
    size_t D = 0;
    sigk_sig_dim(d, N, &D);
    const size_t xbytes = sizeof(Real) * B * L * d, obytes = sizeof(Real) * B * D;
    const bool xdev = flags & SIGK_X_ON_DEVICE, odev = flags & SIGK_OUT_ON_DEVICE;
    const Real* Xd = X;
    Real* Od = out;
    Real* xbuf = nullptr;
    Real* obuf = nullptr;
    cudaError_t e;
    if (!xdev) {
        e = cudaMallocAsync(reinterpret_cast<void**>(&xbuf), xbytes, s);
        if (e != cudaSuccess) return cuda_fail(e, "input staging allocation");
        e = cudaMemcpyAsync(xbuf, X, xbytes, cudaMemcpyHostToDevice, s);
        if (e != cudaSuccess) return cuda_fail(e, "H2D copy");
        Xd = xbuf;
    }
    if (!odev) {
        e = cudaMallocAsync(reinterpret_cast<void**>(&obuf), obytes, s);
        if (e != cudaSuccess) return cuda_fail(e, "output staging allocation");
        Od = obuf;
    }
    rc = run_device<Real>(Xd, (int64_t)B, (int64_t)L, d, N, Od, s, tun, st);
    if (rc == SIGK_OK && !odev) {
        e = cudaMemcpyAsync(out, obuf, obytes, cudaMemcpyDeviceToHost, s);
        if (e != cudaSuccess) rc = cuda_fail(e, "D2H copy");
    }
    if (xbuf) cudaFreeAsync(xbuf, s);
    if (obuf) cudaFreeAsync(obuf, s);
    if (!xdev || !odev) {
        e = cudaStreamSynchronize(s);
        if (e != cudaSuccess && rc == SIGK_OK) rc = cuda_fail(e, "stream synchronize");
    }
    if (rc == SIGK_OK && (xdev && odev)) {
        e = cudaPeekAtLastError();
        if (e != cudaSuccess) rc = cuda_fail(e, "kernel launch");
    }
    return rc;
}

template <typename Real>
static int sharded_impl(const Real* X, size_t B, size_t L, int d, int N, Real* out, int num_gpus, sigk_stats* st) {
    g_err.clear();
    int rc = validate(X, B, L, d, N, out);
    if (rc != SIGK_OK) return rc;
    int ndev = 0;
    cudaError_t e = cudaGetDeviceCount(&ndev);
    if (e != cudaSuccess || ndev < 1) return cuda_fail(e == cudaSuccess ? cudaErrorNoDevice : e, "device query");
    int G = num_gpus <= 0 ? ndev : std::min(num_gpus, ndev);
    G = (int)std::min<size_t>((size_t)G, B);
    size_t D = 0;
    sigk_sig_dim(d, N, &D);
    const size_t per = (B + G - 1) / G;
    std::vector<int> rcs(G, SIGK_OK);
    std::vector<std::string> errs(G);
    std::vector<sigk_stats> sts(G);
    std::vector<std::thread> th;
    for (int g = 0; g < G; ++g) {
        const size_t b0 = g * per;
        if (b0 >= B) break;
        const size_t nb = std::min(per, B - b0);
        th.emplace_back([&, g, b0, nb] {
            cudaError_t ee = cudaSetDevice(g);
            if (ee != cudaSuccess) {
                rcs[g] = cuda_fail(ee, "cudaSetDevice");
                errs[g] = g_err;
                return;
            }
            cudaStream_t s;
            cudaStreamCreateWithFlags(&s, cudaStreamNonBlocking);
            sigk_tuning tun{};
            tun.plan_rows = (int64_t)B;  // same chunking on every shard -> bitwise equal to G = 1
            rcs[g] = signature_impl<Real>(X + b0 * L * d, nb, L, d, N, out + b0 * D, 0u, s, &tun, &sts[g]);
            errs[g] = g_err;
            cudaStreamDestroy(s);
        });
    }
    for (auto& t : th) t.join();
    for (int g = 0; g < (int)th.size(); ++g)
        if (rcs[g] != SIGK_OK) return fail(rcs[g], "device " + std::to_string(g) + ": " + errs[g]);
    if (st) {
        *st = sts[0];
        st->launches = 0;
        for (int g = 0; g < (int)th.size(); ++g) st->launches += sts[g].launches;
    }
    return SIGK_OK;
}

}  // namespace sigk

extern "C" {

int sigk_sig_dim(int d, int N, size_t* D) {
    if (d < 1) return sigk::fail(SIGK_EDOMAIN, "sig_dim: dim must be >= 1, got " + std::to_string(d));
    if (N < 1) return sigk::fail(SIGK_EDOMAIN, "sig_dim: depth must be >= 1, got " + std::to_string(N));
    size_t t = 0, p = 1;
    for (int n = 1; n <= N; ++n) {
        p *= (size_t)d;
        t += p;
    }
    if (D) *D = t;
    return SIGK_OK;
}

int sigk_level_offsets(int d, int N, size_t* offsets) {
    int rc = sigk_sig_dim(d, N, nullptr);
    if (rc != SIGK_OK) return rc;
    size_t p = 1;
    offsets[0] = 0;
    for (int n = 1; n <= N; ++n) {
        p *= (size_t)d;
        offsets[n] = offsets[n - 1] + p;
    }
    return SIGK_OK;
}

int sigk_signature_f32(const float* X, size_t B, size_t L, int d, int N, float* out, unsigned flags, void* stream,
                       const sigk_tuning* tuning, sigk_stats* stats) {
    return sigk::signature_impl<float>(X, B, L, d, N, out, flags, stream, tuning, stats);
}

int sigk_signature_f64(const double* X, size_t B, size_t L, int d, int N, double* out, unsigned flags, void* stream,
                       const sigk_tuning* tuning, sigk_stats* stats) {
    return sigk::signature_impl<double>(X, B, L, d, N, out, flags, stream, tuning, stats);
}

int sigk_signature_sharded_f32(const float* X, size_t B, size_t L, int d, int N, float* out, int num_gpus,
                               sigk_stats* stats) {
    return sigk::sharded_impl<float>(X, B, L, d, N, out, num_gpus, stats);
}

int sigk_signature_sharded_f64(const double* X, size_t B, size_t L, int d, int N, double* out, int num_gpus,
                               sigk_stats* stats) {
    return sigk::sharded_impl<double>(X, B, L, d, N, out, num_gpus, stats);
}

int sigk_brownian_f32(float* X, size_t B, size_t L, int d, uint64_t seed, size_t row0, void* stream) {
    if (B < 1 || L < 1 || d < 1 || !X) return sigk::fail(SIGK_EDOMAIN, "brownian: bad shape");
    cudaError_t e = sigk::launch_brownian_f32(X, (int64_t)B, (int64_t)L, d, seed, (int64_t)row0,
                                              static_cast<cudaStream_t>(stream));
    return e == cudaSuccess ? SIGK_OK : sigk::cuda_fail(e, "brownian launch");
}

int sigk_brownian_f64(double* X, size_t B, size_t L, int d, uint64_t seed, size_t row0, void* stream) {
    if (B < 1 || L < 1 || d < 1 || !X) return sigk::fail(SIGK_EDOMAIN, "brownian: bad shape");
    cudaError_t e = sigk::launch_brownian_f64(X, (int64_t)B, (int64_t)L, d, seed, (int64_t)row0,
                                              static_cast<cudaStream_t>(stream));
    return e == cudaSuccess ? SIGK_OK : sigk::cuda_fail(e, "brownian launch");
}

int sigk_has_fast_variant(int d, int N, int is_f64, int* Q) {
    const sigk::Variant* v = sigk::find_variant(d, N, is_f64 != 0);
    if (Q) *Q = v ? v->Q : -1;
    return v != nullptr;
}

const char* sigk_last_error(void) { return sigk::g_err.c_str(); }

int sigk_version(void) { return 100; }

}  // extern "C"

// Generic / brownian launchers (templates live in generic.cuh).
namespace sigk {
template <typename Real>
static cudaError_t gen(const void* X, int64_t B, int64_t L, int d, int N, void* out, cudaStream_t s) {
    const int64_t D = level_off(d, N);
    if (N > kGenericMaxDepth) return cudaErrorInvalidValue;
    generic_fold_kernel<Real><<<(unsigned)B, 256, sizeof(Real) * d, s>>>(static_cast<const Real*>(X), L, d, N, D,
                                                                          static_cast<Real*>(out));
    return cudaGetLastError();
}
template <typename Real>
static cudaError_t brown(void* X, int64_t B, int64_t L, int d, uint64_t seed, int64_t row0, cudaStream_t s) {
    const int64_t n = B * d;
    brownian_kernel<Real><<<(unsigned)((n + 127) / 128), 128, 0, s>>>(static_cast<Real*>(X), B, L, d, seed, row0);
    return cudaGetLastError();
}
cudaError_t launch_generic_f32(const void* X, int64_t B, int64_t L, int d, int N, void* out, cudaStream_t s) {
    return gen<float>(X, B, L, d, N, out, s);
}
cudaError_t launch_generic_f64(const void* X, int64_t B, int64_t L, int d, int N, void* out, cudaStream_t s) {
    return gen<double>(X, B, L, d, N, out, s);
}
cudaError_t launch_brownian_f32(void* X, int64_t B, int64_t L, int d, uint64_t seed, int64_t row0, cudaStream_t s) {
    return brown<float>(X, B, L, d, seed, row0, s);
}
cudaError_t launch_brownian_f64(void* X, int64_t B, int64_t L, int d, uint64_t seed, int64_t row0, cudaStream_t s) {
    return brown<double>(X, B, L, d, seed, row0, s);
}
}  // namespace sigk
