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
#include "vjp_kernel.cuh"
#include "increments.cuh"
#include "bruteforce.cuh"
#include "scan_kernel.cuh"
#include "scan_vjp.cuh"

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

const Variant* find_variant(int d, int N, bool is_f64) {
    Registry& r = registry();
    std::lock_guard<std::mutex> g(r.mu);
    const Variant* best = nullptr;
    for (const Variant& v : is_f64 ? r.f64 : r.f32)
        if (v.d == d && v.N == N && (!best || v.Q < best->Q)) best = &v;
    return best;
}

int find_variants(int d, int N, bool is_f64, const Variant** out, int max) {
    Registry& r = registry();
    std::lock_guard<std::mutex> g(r.mu);
    int n = 0;
    for (const Variant& v : is_f64 ? r.f64 : r.f32)
        if (v.d == d && v.N == N && n < max) out[n++] = &v;
    return n;
}

// Issue efficiency of the FFMA pipe vs resident warps per SM sub-partition
// (measured on B200 with tools/ffma_probe.cu: ~0.62 at 1 warp, ~0.85 at 2).
static double issue_eff(double warps_per_smsp) {
    // saturates near 0.8: the fold's 3-register FFMAs dispatch at ~0.75/cycle/SMSP
    // (tools/step_probe.cu), and the in-kernel loop adds shared-memory traffic
    if (warps_per_smsp <= 1.0) return 0.55 * std::max(warps_per_smsp, 0.05);
    if (warps_per_smsp <= 2.0) return 0.55 + 0.2 * (warps_per_smsp - 1.0);
    return std::min(0.8, 0.75 + 0.05 * (warps_per_smsp - 2.0));
}

// Cycle model of one launch (SM cycles). Path kernel: a wave puts c CTAs of
// U*P threads on each SM; a thread issues CL * (ops + loads + producer + 2)
// slots for the fold, the Chen tree issues ~12 slots per output element per
// product ((U-1) products of D elements) plus barriers per level and round.
static double model_cycles(const Variant& v, int64_t B, int64_t M, int sms, int U, int occ, int64_t D) {
    const double prod = (double)((v.T * v.d + v.P - 1) / v.P) * (v.N + (v.N - v.Q) + 4) / v.T;
    const double per_step = v.ops + v.loads + prod + 2.0;
    if (v.family == KernelFamily::Flat) {
        const int64_t ctas = (B * v.P + v.nt - 1) / v.nt;
        const int64_t per_sm = (ctas + sms - 1) / sms;
        const int64_t c = std::min<int64_t>(occ, per_sm);
        const int64_t waves = (per_sm + c - 1) / c;
        const double eff = issue_eff(c * (v.nt / 32.0) / 4.0);
        return waves * (c * v.nt * (double)M * per_step / 128.0 / eff);
    }
    const int64_t CL = (M + U - 1) / U;
    const int64_t c = std::min<int64_t>(occ, (B + sms - 1) / sms);  // CTAs per SM per wave
    const int64_t waves = (B + sms * c - 1) / (sms * c);
    const double threads = (double)U * v.P;
    const double eff = issue_eff(c * std::ceil(threads / 32.0) / 4.0);
    const double fold = c * threads * CL * per_step / 128.0 / eff;
    int rounds = 0;
    while ((1 << rounds) < U) ++rounds;
    // combine (merge.cuh): ~20 issue slots per chunk per signature element, plus
    // a barrier-bound latency per degree
    const double merge = c * (U - 1) * (double)D * 20.0 / 128.0 / eff + rounds * v.N * 120.0;
    const double sync = (double)((CL + v.T - 1) / v.T) * 100.0;
    return waves * (fold + merge + sync);
}

// Pair family (pair_kernel.cuh), modelled for back-to-back launches (the
// serving / benchmark regime, where programmatic dependent launch keeps every
// SM's CTA slots filled across calls): B*G segment CTAs of w = ceil(U/2*P/32)
// warps; each CTA's fold keeps the FMA pipe busy for fold_pipe cycles (an
// FFMA2 is 2 pipe cycles per warp) and spends `fixed` cycles in staging, table
// build and chunk combine with the pipe mostly idle. With c CTAs resident per
// SM the SM retires a CTA every max(pipe-bound, latency-bound) cycles.
static double pair_eff(double warps_per_smsp) {
    if (warps_per_smsp >= 3.0) return 0.92;
    if (warps_per_smsp >= 2.0) return 0.85 + 0.07 * (warps_per_smsp - 2.0);
    if (warps_per_smsp >= 1.0) return 0.6 + 0.25 * (warps_per_smsp - 1.0);
    return 0.6 * warps_per_smsp;
}

static double model_pair(const Variant& v, int64_t B, int64_t M, int sms, int G, int U, int occ) {
    const int64_t SL = (M + G - 1) / G;
    const int64_t CL = (SL + U - 1) / U;
    const int64_t ctas = B * G;
    const int warps = (int)((U / 2 * v.P + 31) / 32);
    const double fold_pipe = warps * (double)CL * v.ops * 2.0 / 4.0;
    const double fixed = 2500.0 + 60.0 * U + 300.0 * v.N + 4.0 * CL;
    const double c = (double)std::max(1, occ);
    const double per_cta = std::max(fold_pipe / pair_eff(c * warps / 4.0),
                                    (fixed + fold_pipe / pair_eff(warps / 4.0)) / c);
    double t = (double)ctas / sms * per_cta;
    if (G > 1) t += (double)B / sms * (1000.0 + 60.0 * G);  // last-CTA segment combine
    return t;
}

// Pair family, one call with nothing to overlap (a synchronous call, the
// first launch on an idle GPU, a training step): every CTA of the launch
// starts together, so phases do not hide each other. Time = the busiest
// SM's fold (c CTAs of `warps` warps folding CL steps; FMA-pipe efficiency by
// warps per SMSP, measured with tools/pair_step_probe.cu: 0.5 / 0.67 / 0.7 /
// 0.73 at 1 / 2 / 3 / 4) plus the serial phases of one CTA (staging latency,
// table build, chunk combine, output, the cluster combine when G > 1).
static double lat_eff(double wps) {
    if (wps >= 4.0) return 0.73;
    if (wps >= 3.0) return 0.70 + 0.03 * (wps - 3.0);
    if (wps >= 2.0) return 0.67 + 0.03 * (wps - 2.0);
    if (wps >= 1.0) return 0.5 + 0.17 * (wps - 1.0);
    return 0.5 * wps;
}

static double model_pair_latency(const Variant& v, int64_t B, int64_t M, int sms, int G, int U, int occ) {
    const int64_t SL = (M + G - 1) / G;
    const int64_t CL = (SL + U - 1) / U;
    const int64_t ctas = B * G;
    const int warps = (int)((U / 2 * v.P + 31) / 32);
    const int64_t per_sm = (ctas + sms - 1) / sms;
    const int64_t c = std::min<int64_t>(per_sm, std::max(1, occ));
    const int64_t waves = (per_sm + c - 1) / c;
    const double wps = c * warps / 4.0;
    const double fold = c * warps * (double)CL * v.ops * 2.0 / 4.0 / lat_eff(wps);
    const double table = (double)CL * (U / 2) * v.d * 6.0 / (warps * 32.0) * c;
    const double fixed = 1500.0 + table + 400.0 + 40.0 * U + 800.0 + (G > 1 ? 6000.0 : 0.0);  // cluster sync + combine: measured
    return waves * (fold + fixed);
}

struct Plan {
    const Variant* v = nullptr;
    int U = 1;
    int G = 1;
    bool pos = false;  // pair family: position-table fold with a producer warp (ppair_kernel.cuh)
};

static const int kSegCands[] = {1, 2, 3, 4, 5, 6, 8, 10, 12, 14, 16, 20, 24, 28, 32, 40, 48, 56, 64, 80, 96, 112, 128,
                                160, 192, 256, 320, 384, 512, 640, 768, 1024};

// Pick the variant, chunks per path (or per segment) U and segments G.
static Plan plan_launch(int d, int N, bool is_f64, int64_t B, int64_t M, int sms, int64_t D, const sigk_tuning* tun) {
    const Variant* cands[8];
    const int nc = find_variants(d, N, is_f64, cands, 8);
    const int fam = tun ? tun->family : 0;
    const int fq = tun ? tun->prefix_len : 0;
    const int fU = tun ? tun->chunks : 0;
    const int fG = tun ? tun->segments : 0;
    const bool latency = tun && tun->mode == SIGK_MODE_LATENCY;
    const bool use_cluster = tun && tun->cluster;
    const int fvar = tun ? tun->fold_variant : 0;
    bool have_pair = false;
    for (int k = 0; k < nc; ++k)
        if (cands[k]->family == KernelFamily::Pair && (fam == 0 || fam == SIGK_FAMILY_PAIR) && (fq == 0 || fq == cands[k]->Q))
            have_pair = true;
    // inner-pair flat family: whole paths as units, so only when the batch
    // alone fills the GPU (>= 2 CTAs of 128 lanes per SM), and only where the
    // scalar kernels need the flat (unchunked, register-heavy) form anyway —
    // measured on B200: C4 (d=10, N=5) 2x faster than flat; C5 (d=8, N=4)
    // 6% slower than the chunk-capable path kernel
    bool scalar_flat = false;
    for (int k = 0; k < nc; ++k)
        if (cands[k]->family == KernelFamily::Flat) scalar_flat = true;
    bool use_pflat = false;
    for (int k = 0; k < nc; ++k)
        if (cands[k]->family == KernelFamily::PFlat && (fq == 0 || fq == cands[k]->Q) &&
            (fam == SIGK_FAMILY_PFLAT ||
             (fam == 0 && !have_pair && scalar_flat && B * cands[k]->P >= (int64_t)sms * 256)))
            use_pflat = true;
    Plan best;
    double best_t = 1e300;
    for (int k = 0; k < nc; ++k) {
        const Variant& v = *cands[k];
        if (fam != 0 && (int)v.family != fam) continue;
        if (fq > 0 && v.Q != fq) continue;
        if ((v.family == KernelFamily::PFlat) != use_pflat) continue;
        if (v.family == KernelFamily::PFlat) {
            int occ = 0;
            if (v.occupancy(1, &occ) != cudaSuccess || occ < 1) continue;
            best.v = &v;
            best.U = 1;
            best.G = 1;
            break;
        }
        if (v.family == KernelFamily::Pair) {
            const int gforce[1] = {fG};
            const int* gl = fG > 0 ? gforce : kSegCands;
            const int ng = fG > 0 ? 1 : (int)(sizeof(kSegCands) / sizeof(int));
            for (int gi = 0; gi < ng; ++gi) {
                const int G = gl[gi];
                if (G > 1 && (N < 2 || (fG == 0 && (int64_t)G * 4 > M) || G > M)) continue;
                const int64_t SL = (M + G - 1) / G;
                const int umax = std::max(2, 2 * v.pair_units_max);
                // a forced chunk count is rounded down to even (>= 2) and clamped to one CTA
                const int uforce = fU > 0 ? std::min(umax, std::max(2, fU / 2 * 2)) : 0;
                for (int U = 2; U <= umax; U += 2) {
                    if (uforce > 0 && U != uforce) continue;
                    if (uforce == 0 && U > 2 && U > SL + 1) break;  // whole empty pair-units
                    const int CL = (int)((SL + U - 1) / U);
                    for (int pos = 0; pos < 2; ++pos) {
                        // the position-table fold is opt-in (fold_variant = 2): measured on B200 it
                        // does not beat the register-table fold (profiles/r02/pos_fold_probe.txt)
                        if (pos && (v.pos_ops == 0 || U / 2 > v.pos_units_max || fvar != 2)) continue;
                        if (!pos && fvar == 2) continue;
                        int occ = 0;
                        if ((pos ? v.pair_pos_occupancy(U, CL, SL, G, use_cluster, &occ)
                                 : v.pair_occupancy(U, CL, SL, G, use_cluster, &occ)) !=
                                cudaSuccess ||
                            occ < 1)
                            continue;
                        Variant vv = v;  // the position-table fold: its op count, no table-build phase
                        if (pos) vv.ops = v.pos_ops;
                        double t = latency ? model_pair_latency(vv, B, M, sms, G, U, occ)
                                           : model_pair(vv, B, M, sms, G, U, occ);
                        if (t < best_t * 0.995) {
                            best_t = t;
                            best.v = &v;
                            best.U = U;
                            best.G = G;
                            best.pos = pos;
                        }
                    }
                }
            }
            continue;
        }
        if (have_pair) continue;  // fp32 shapes with a pair variant use it
        const int umax = v.family == KernelFamily::Path ? (int)std::min<int64_t>(M, v.nt / v.P) : 1;
        for (int U = 1; U <= umax; ++U) {
            if (fU > 0 && v.family == KernelFamily::Path && U != std::min<int64_t>(fU, umax)) continue;
            int occ = 0;
            if (v.occupancy(U, &occ) != cudaSuccess || occ < 1) continue;
            const double t = model_cycles(v, B, M, sms, U, occ, D);
            if (t < best_t * 0.995) {
                best_t = t;
                best.v = &v;
                best.U = U;
                best.G = 1;
            }
        }
    }
    return best;
}

struct PlanKey {
    int d, N, dev;
    bool f64;
    int64_t B, M;
    int fam, q, U, G, mode, fvar;
    bool operator==(const PlanKey& o) const {
        return d == o.d && N == o.N && dev == o.dev && f64 == o.f64 && B == o.B && M == o.M && fam == o.fam &&
               q == o.q && U == o.U && G == o.G && mode == o.mode && fvar == o.fvar;
    }
};

static Plan cached_plan(int d, int N, bool is_f64, int dev, int64_t B, int64_t M, int64_t D, const sigk_tuning* tun) {
    static std::mutex mu;
    static std::vector<std::pair<PlanKey, Plan>> cache;
    const PlanKey key{d, N, dev, is_f64, B, M, tun ? tun->family : 0, tun ? tun->prefix_len : 0,
                      tun ? tun->chunks : 0, tun ? tun->segments : 0, tun ? tun->mode : 0,
                      tun ? tun->fold_variant : 0};
    {
        std::lock_guard<std::mutex> g(mu);
        for (auto& kv : cache)
            if (kv.first == key) return kv.second;
    }
    const Plan p = plan_launch(d, N, is_f64, B, M, device_info(dev).sms, D, tun);
    cudaGetLastError();  // occupancy probes of configurations that do not fit must not leak an error
    std::lock_guard<std::mutex> g(mu);
    if (cache.size() > 256) cache.clear();
    cache.emplace_back(key, p);
    return p;
}

// Programmatic-dependent-launch safety. A fold kernel launched with PDL may
// start while the previous kernel on its stream still runs; it orders only
// its OUTPUT writes after that kernel (griddepcontrol.wait), not its reads of
// X. Only sigk's own fold kernels trigger dependents early, and they write
// nothing but their output rows, so the overlap is safe unless X overlaps the
// output of the previous sigk launch on the same stream (any other kernel in
// between completes before ours can start). Remember each stream's last
// output range and refuse the overlap when X intersects it.
static bool may_overlap_previous(int dev, cudaStream_t s, const void* X, size_t xbytes, const void* out,
                                 size_t obytes) {
    struct Last {
        int dev;
        cudaStream_t s;
        uintptr_t lo, hi;
    };
    static std::mutex mu;
    static std::vector<Last> last;
    const uintptr_t xlo = reinterpret_cast<uintptr_t>(X), xhi = xlo + xbytes;
    const uintptr_t olo = reinterpret_cast<uintptr_t>(out), ohi = olo + obytes;
    std::lock_guard<std::mutex> g(mu);
    for (Last& l : last) {
        if (l.dev == dev && l.s == s) {
            const bool ok = xhi <= l.lo || xlo >= l.hi;
            l.lo = olo;
            l.hi = ohi;
            return ok;
        }
    }
    if (last.size() > 1024) last.clear();
    last.push_back(Last{dev, s, olo, ohi});
    return true;
}

// Per-(device, stream) scratch of the pair family's segmented plans: kind 0 =
// segment rows, kind 1 = per-path arrival counters (zeroed when allocated and
// left at zero by every completed launch); kinds >= 2: stream pieces and
// reverse-mode buffers. A buffer is NEVER freed while the process runs: a
// CUDA graph captured earlier, or a launch another host thread is enqueueing
// with the pointer it got (ctypes releases the GIL), may still reference it.
// Growth (geometric, so rare) allocates a new buffer and retires the old one
// to a list that lives until process exit. During stream capture a missing
// buffer is allocated stream-ordered instead (and freed the same way by the
// caller, inside the captured graph).
static void* segment_scratch(int dev, cudaStream_t s, int kind, size_t bytes, bool capturing, bool* async_alloc) {
    struct Buf {
        int dev;
        cudaStream_t s;
        int kind;
        void* p;
        size_t n;
    };
    static std::mutex mu;
    static std::vector<Buf> bufs;
    static std::vector<void*> retired;  // grown-out buffers: kept alive (see above)
    *async_alloc = false;
    std::lock_guard<std::mutex> g(mu);
    Buf* hit = nullptr;
    for (Buf& b : bufs)
        if (b.dev == dev && b.s == s && b.kind == kind) hit = &b;
    if (hit && hit->n >= bytes) return hit->p;
    if (capturing) {
        void* p = nullptr;
        if (cudaMallocAsync(&p, bytes, s) != cudaSuccess) return nullptr;
        if ((kind == 1 || kind == 12) && cudaMemsetAsync(p, 0, bytes, s) != cudaSuccess) return nullptr;
        *async_alloc = true;
        return p;
    }
    const size_t n = std::max(bytes, hit ? 2 * hit->n : bytes);
    void* p = nullptr;
    if (cudaMalloc(&p, n) != cudaSuccess) return nullptr;
    // counters / flags start at zero, ordered before the launch on this stream
    if ((kind == 1 || kind == 12) && cudaMemsetAsync(p, 0, n, s) != cudaSuccess) return nullptr;
    if (hit) {
        retired.push_back(hit->p);
        hit->p = p;
        hit->n = n;
    } else {
        bufs.push_back(Buf{dev, s, kind, p, n});
    }
    return p;
}

// Increments of one path covered by a launch of G segments x U chunks
// (segment g folds [g*SL, min((g+1)*SL, M)), chunk u of it CL steps):
// sigk_stats.path_steps, counted from the geometry the kernels were given.
static int64_t covered_steps(int64_t M, int64_t G, int64_t U) {
    const int64_t SL = (M + G - 1) / G, CL = (SL + U - 1) / U;
    int64_t n = 0;
    for (int64_t g = 0; g < G; ++g) {  // U chunks of CL steps cover min(segment, U*CL) of each segment
        const int64_t s0 = std::min(M, g * SL), s1 = std::min(M, s0 + SL);
        n += std::min(s1 - s0, U * CL);
    }
    return n;
}

// Chunk paths (reverse mode): run_device's B paths of L = CL + 1 points are the
// chunks of a (B / U, Lsrc, d) batch (PairLaunch::sub_U), read in place by the
// pair family; other plans return kNeedGather without launching.
// reverse mode: the longest chunk one fold-and-passes CTA takes (longer paths chunk
// over more CTAs: chunk signatures in place, then the pass kernel)
constexpr int64_t kPrepMaxChunkSteps = 160;
constexpr int kPrepMaxChunks = 20;  // the passes walk the chunks serially per entry
constexpr int64_t kPrepMinSteps = 750;

struct SubPaths {
    int64_t U = 0, CL = 0, Lsrc = 0;
};
constexpr int kNeedGather = -1000;

template <typename Real>
static int run_device(const Real* X, int64_t B, int64_t L, int d, int N, Real* out, cudaStream_t s,
                      const sigk_tuning* tun, sigk_stats* st, const SubPaths* sub = nullptr) {
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
    cudaEvent_t ev0 = tun ? static_cast<cudaEvent_t>(tun->fold_event_start) : nullptr;
    cudaEvent_t ev1 = tun ? static_cast<cudaEvent_t>(tun->fold_event_stop) : nullptr;
    cudaStreamCaptureStatus cap = cudaStreamCaptureStatusNone;
    if (ev0 || ev1) cudaStreamIsCapturing(s, &cap);
    auto record = [&](cudaEvent_t ev) {  // an event-record node when captured into a graph
        if (!ev) return;
        if (cap == cudaStreamCaptureStatusActive) cudaEventRecordWithFlags(ev, s, cudaEventRecordExternal);
        else cudaEventRecord(ev, s);
    };
    int dev = 0;
    cudaGetDevice(&dev);
    const int64_t plan_rows = (tun && tun->plan_rows > 0) ? tun->plan_rows : B;
    Plan plan;
    if (!(tun && (tun->force_generic || tun->family == SIGK_FAMILY_GENERIC)))
        plan = cached_plan(d, N, is_f64, dev, plan_rows, M, D, tun);
    const Variant* v = plan.v;
    if (sub && (v == nullptr || v->family != KernelFamily::Pair || plan.pos)) return kNeedGather;
    if (v == nullptr) {
        record(ev0);
        e = is_f64 ? launch_generic_f64(X, B, L, d, N, out, s) : launch_generic_f32(X, B, L, d, N, out, s);
        record(ev1);
        if (e != cudaSuccess) return cuda_fail(e, "generic fold launch");
        local.fold_steps = M;
        local.path_steps = M;
        local.chunks = 1;
        local.prefix_len = -1;
        local.threads_per_unit = 0;
        local.launches = 1;
        local.segments = 1;
        local.family = SIGK_FAMILY_GENERIC;
        if (st) *st = local;
        return SIGK_OK;
    }
    const bool overlap = !(tun && tun->no_overlap) &&
                         may_overlap_previous(dev, s, X, sizeof(Real) * B * L * d, out, sizeof(Real) * B * D);
    if (v->family == KernelFamily::Pair) {
        const int G = plan.G, U = plan.U;
        const int64_t SL = (M + G - 1) / G;
        const int CL = (int)((SL + U - 1) / U);
        void* rows = nullptr;
        void* counters = nullptr;
        bool async_rows = false, async_ctr = false;
        const bool cluster = G > 1 && G <= kMaxPairCluster && tun && tun->cluster && !sub;
        if (G > 1 && !cluster) {
            if (cap == cudaStreamCaptureStatusNone) cudaStreamIsCapturing(s, &cap);
            const bool capt = cap == cudaStreamCaptureStatusActive;
            rows = segment_scratch(dev, s, 0, sizeof(float) * B * G * D, capt, &async_rows);
            counters = segment_scratch(dev, s, 1, sizeof(int) * B, capt, &async_ctr);
            if (!rows || !counters) return fail(SIGK_ERESOURCE, "segment scratch allocation failed");
        }
        PairLaunch a{X, B, L, G, SL, U, CL, out, rows, counters, s, overlap, ev0, ev1,
                     cap == cudaStreamCaptureStatusActive, tun ? tun->phase_buf : nullptr, cluster, plan.pos};
        if (sub) {
            a.sub_U = sub->U;
            a.sub_CL = sub->CL;
            a.sub_L = sub->Lsrc;
        }
        e = v->pair_launch(a);
        if (async_rows) cudaFreeAsync(rows, s);
        if (async_ctr) cudaFreeAsync(counters, s);
        if (e != cudaSuccess) return cuda_fail(e, "pair fold launch");
        int rounds = 0;
        while ((1 << rounds) < U) ++rounds;
        int grounds = 0;
        while ((1 << grounds) < G) ++grounds;
        local.fold_steps = CL;
        local.path_steps = covered_steps(M, G, U);
        local.scan_passes = rounds + grounds;
        local.chunks = U;
        local.prefix_len = v->Q;
        local.threads_per_unit = v->P;
        local.launches = 1;
        local.segments = G;
        local.family = SIGK_FAMILY_PAIR;
        if (st) *st = local;
        return SIGK_OK;
    }
    int U = 1;
    if (v->family == KernelFamily::Path) {
        U = (tun && tun->chunks > 0) ? tun->chunks : plan.U;
        U = (int)std::max<int64_t>(1, std::min<int64_t>({(int64_t)U, M, (int64_t)(v->nt / v->P)}));
        int occ = 0;
        for (;;) {  // a forced chunk count may exceed the shared-memory budget: shrink it
            e = v->occupancy(U, &occ);
            if (e != cudaSuccess) return cuda_fail(e, "occupancy query");
            if (occ >= 1 || U == 1) break;
            --U;
        }
        if (occ < 1) return fail(SIGK_ERESOURCE, "fold variant does not fit on this device");
    }
    record(ev0);
    e = v->launch(X, B, L, U, out, s, tun ? tun->phase_buf : nullptr, overlap && !ev0);
    record(ev1);
    if (e != cudaSuccess) return cuda_fail(e, "fold launch");
    const int64_t CL = (M + U - 1) / U;
    int rounds = 0;
    while ((1 << rounds) < U) ++rounds;
    local.fold_steps = CL;
    local.path_steps = v->family == KernelFamily::Path ? covered_steps(M, 1, U) : M;
    local.scan_passes = rounds;
    local.chunks = U;
    local.prefix_len = v->Q;
    local.threads_per_unit = v->P;
    local.launches = 1;
    local.segments = 1;
    local.family = (int)v->family;
    if (st) *st = local;
    return SIGK_OK;
}

// The plan run_device would use (sigk_plan).
static int plan_only(size_t B, size_t L, int d, int N, bool is_f64, const sigk_tuning* tun, sigk_stats* st) {
    sigk_stats local{};
    const int64_t M = (int64_t)L - 1;
    int64_t D = 0, p = 1;
    for (int n = 0; n < N; ++n) {
        p *= d;
        D += p;
    }
    local.segments = 1;
    if (M <= 0) {
        local.chunks = 1;
        if (st) *st = local;
        return SIGK_OK;
    }
    int dev = 0;
    cudaError_t e = cudaGetDevice(&dev);
    if (e != cudaSuccess) return cuda_fail(e, "cudaGetDevice");
    const int64_t plan_rows = (tun && tun->plan_rows > 0) ? tun->plan_rows : (int64_t)B;
    Plan plan;
    if (!(tun && (tun->force_generic || tun->family == SIGK_FAMILY_GENERIC)))
        plan = cached_plan(d, N, is_f64, dev, plan_rows, M, D, tun);
    if (!plan.v) {
        local.family = SIGK_FAMILY_GENERIC;
        local.prefix_len = -1;
        local.chunks = 1;
        local.fold_steps = M;
    } else {
        const int64_t SL = (M + plan.G - 1) / plan.G;
        local.family = (int)plan.v->family;
        local.prefix_len = plan.v->Q;
        local.threads_per_unit = plan.v->P;
        local.chunks = plan.U;
        local.segments = plan.G;
        local.fold_steps = (SL + plan.U - 1) / plan.U;
        local.launches = 1;
    }
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

struct Staging {
    static constexpr int kPieces = 8;
    std::mutex mu;
    void* p = nullptr;
    size_t n = 0;
    cudaStream_t hs = nullptr, ds = nullptr;  // H2D and D2H copy streams
    cudaEvent_t ev[2 * kPieces + 2] = {};
};

// Asynchronous host-buffer calls (SIGK_ASYNC_HOST): a ring of staging slots
// per (device, stream). Slot k serves calls k, k+R, ...; before reusing it a
// call waits (on the device, never the host) for the kernel that read its X
// and the D2H that drained its output. Copies and kernels run on the ring's
// own streams; the caller's stream only waits for each call's D2H, so
// synchronising it covers the results without serialising the next call.
struct AsyncRing {
    static constexpr int R = 3;
    std::mutex mu;
    void* p[R] = {};
    size_t n[R] = {};
    cudaStream_t hs = nullptr, cs = nullptr, ds = nullptr;  // H2D, kernels, D2H
    cudaStream_t hs2 = nullptr;  // second H2D stream: consecutive calls' inputs on both copy engines
    cudaEvent_t h2d[R] = {}, kdone[R] = {}, d2h[R] = {};
    bool used[R] = {};
    unsigned next = 0;
};

static AsyncRing& ring_for(int dev, cudaStream_t s) {
    static std::mutex mu;
    static std::vector<std::pair<std::pair<int, cudaStream_t>, AsyncRing*>> tab;
    std::lock_guard<std::mutex> g(mu);
    for (auto& kv : tab)
        if (kv.first.first == dev && kv.first.second == s) return *kv.second;
    tab.emplace_back(std::make_pair(dev, s), new AsyncRing());
    return *tab.back().second;
}

static bool is_pinned_host(const void* p) {
    cudaPointerAttributes a{};
    if (cudaPointerGetAttributes(&a, p) != cudaSuccess) {
        cudaGetLastError();
        return false;
    }
    return a.type == cudaMemoryTypeHost;
}

// Host-buffer staging per (device, stream); entries live for the process.
static Staging& staging_for(int dev, cudaStream_t s) {
    static std::mutex mu;
    static std::vector<std::pair<std::pair<int, cudaStream_t>, Staging*>> tab;
    std::lock_guard<std::mutex> g(mu);
    for (auto& kv : tab)
        if (kv.first.first == dev && kv.first.second == s) return *kv.second;
    tab.emplace_back(std::make_pair(dev, s), new Staging());
    return *tab.back().second;
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
    cudaError_t e;
    if (xdev && odev) {
        rc = run_device<Real>(Xd, (int64_t)B, (int64_t)L, d, N, Od, s, tun, st);  // asynchronous
        if (rc == SIGK_OK) {
            e = cudaPeekAtLastError();
            if (e != cudaSuccess) rc = cuda_fail(e, "kernel launch");
        }
        return rc;
    }
    if (flags & SIGK_ASYNC_HOST) {
        if (xdev || odev) return fail(SIGK_EDOMAIN, "SIGK_ASYNC_HOST is for host X and out");
        if (!is_pinned_host(X) || !is_pinned_host(out))
            return fail(SIGK_EDOMAIN, "SIGK_ASYNC_HOST needs page-locked X and out (cudaHostAlloc/cudaHostRegister)");
        int dev = 0;
        cudaGetDevice(&dev);
        AsyncRing& rg = ring_for(dev, s);
        std::lock_guard<std::mutex> lock(rg.mu);
        if (!rg.hs) {
            cudaStreamCreateWithFlags(&rg.hs, cudaStreamNonBlocking);
            cudaStreamCreateWithFlags(&rg.hs2, cudaStreamNonBlocking);
            cudaStreamCreateWithFlags(&rg.cs, cudaStreamNonBlocking);
            cudaStreamCreateWithFlags(&rg.ds, cudaStreamNonBlocking);
            for (int k = 0; k < AsyncRing::R; ++k) {
                cudaEventCreateWithFlags(&rg.h2d[k], cudaEventDisableTiming);
                cudaEventCreateWithFlags(&rg.kdone[k], cudaEventDisableTiming);
                cudaEventCreateWithFlags(&rg.d2h[k], cudaEventDisableTiming);
            }
        }
        const int k = (int)(rg.next++ % AsyncRing::R);
        const size_t ooff = (xbytes + 255) / 256 * 256, need = ooff + obytes;
        if (rg.n[k] < need) {
            if (rg.p[k]) {
                cudaEventSynchronize(rg.kdone[k]);  // growth is rare: let the slot drain first
                cudaEventSynchronize(rg.d2h[k]);
                cudaFree(rg.p[k]);
            }
            rg.p[k] = nullptr;
            rg.n[k] = 0;
            e = cudaMalloc(&rg.p[k], need);
            if (e != cudaSuccess) return cuda_fail(e, "async staging allocation");
            rg.n[k] = need;
            rg.used[k] = false;
        }
        Real* xbuf = static_cast<Real*>(rg.p[k]);
        Real* obuf = reinterpret_cast<Real*>(static_cast<char*>(rg.p[k]) + ooff);
        // H2D on the copy stream, ordered only after the slot's last reader: X is
        // host data that is complete at call time, so it need not wait for the
        // caller's queued work (that would serialise consecutive calls)
        // alternate calls between two H2D streams (measured on B200: 48.9 -> 51.2 GB/s
        // aggregate for 2.56 MB copies, tools/h2d_probe.py)
        cudaStream_t hs = (rg.next & 1) ? rg.hs2 : rg.hs;
        if (rg.used[k]) cudaStreamWaitEvent(hs, rg.kdone[k], 0);
        e = cudaMemcpyAsync(xbuf, X, xbytes, cudaMemcpyHostToDevice, hs);
        if (e != cudaSuccess) return cuda_fail(e, "H2D copy");
        cudaEventRecord(rg.h2d[k], hs);
        cudaStreamWaitEvent(rg.cs, rg.h2d[k], 0);
        if (rg.used[k]) cudaStreamWaitEvent(rg.cs, rg.d2h[k], 0);  // obuf drained
        rc = run_device<Real>(xbuf, (int64_t)B, (int64_t)L, d, N, obuf, rg.cs, tun, st);
        if (rc != SIGK_OK) return rc;
        cudaEventRecord(rg.kdone[k], rg.cs);
        cudaStreamWaitEvent(rg.ds, rg.kdone[k], 0);
        e = cudaMemcpyAsync(out, obuf, obytes, cudaMemcpyDeviceToHost, rg.ds);
        if (e != cudaSuccess) return cuda_fail(e, "D2H copy");
        cudaEventRecord(rg.d2h[k], rg.ds);
        cudaStreamWaitEvent(s, rg.d2h[k], 0);  // synchronising the caller's stream covers the result
        rg.used[k] = true;
        e = cudaPeekAtLastError();
        return e == cudaSuccess ? SIGK_OK : cuda_fail(e, "async host call");
    }
    // Host buffers: the call is synchronous. Device staging comes from a
    // per-(device, stream) buffer that persists across calls (a stream-ordered
    // allocation per call would be returned to the OS at every synchronize and
    // re-mapped by the next call), held under its lock for the whole call.
    // The batch is cut into row pieces so PCIe and compute overlap: all H2D
    // copies go back to back on a copy stream, piece i's kernel waits only for
    // its own rows, and its D2H runs on a third stream while later pieces copy
    // in and fold (plan_rows = B keeps the plan, hence the results, identical
    // to a single launch over the whole batch).
    int dev = 0;
    cudaGetDevice(&dev);
    Staging& stg = staging_for(dev, s);
    std::lock_guard<std::mutex> lock(stg.mu);
    const size_t xoff = 0, ooff = xdev ? 0 : (xbytes + 255) / 256 * 256;
    const size_t need = ooff + (odev ? 0 : obytes);
    if (stg.n < need) {
        if (stg.p) cudaFree(stg.p);
        stg.p = nullptr;
        stg.n = 0;
        e = cudaMalloc(&stg.p, need);
        if (e != cudaSuccess) return cuda_fail(e, "staging allocation");
        stg.n = need;
    }
    if (!stg.hs) {
        cudaStreamCreateWithFlags(&stg.hs, cudaStreamNonBlocking);
        cudaStreamCreateWithFlags(&stg.ds, cudaStreamNonBlocking);
        for (auto& ev : stg.ev) cudaEventCreateWithFlags(&ev, cudaEventDisableTiming);
    }
    Real* xbuf = xdev ? const_cast<Real*>(X) : reinterpret_cast<Real*>(static_cast<char*>(stg.p) + xoff);
    Real* obuf = odev ? out : reinterpret_cast<Real*>(static_cast<char*>(stg.p) + ooff);
    // pieces pay off once PCIe time dwarfs the per-piece API cost: one per
    // ~4 MB moved, >= 16 rows each, <= 8 (measured on B200, tools/e2e_ab.py:
    // C2 2.9 MB best whole, C4 30 MB best in 4, C5 415 MB best in 8)
    const size_t moved = (xdev ? 0 : xbytes) + (odev ? 0 : obytes);
    int np = (int)std::max<size_t>(1, std::min<size_t>({(size_t)Staging::kPieces, B / 16, moved >> 22}));
    if (const char* f = getenv("SIGK_HOST_PIECES")) np = std::max(1, std::min(Staging::kPieces, atoi(f)));  // experiments
    const size_t per = (B + np - 1) / np;
    // the copy streams start after everything already queued on the caller's stream
    cudaEventRecord(stg.ev[2 * Staging::kPieces], s);
    cudaStreamWaitEvent(stg.hs, stg.ev[2 * Staging::kPieces], 0);
    cudaStreamWaitEvent(stg.ds, stg.ev[2 * Staging::kPieces], 0);
    sigk_tuning tp = tun ? *tun : sigk_tuning{};
    if (tp.plan_rows <= 0) tp.plan_rows = (int64_t)B;
    // a synchronous host call has no neighbouring launch to overlap: plan for latency
    if (tp.mode == SIGK_MODE_AUTO) tp.mode = SIGK_MODE_LATENCY;
    sigk_stats acc{};
    int launches = 0;
    for (int i = 0; i < np && rc == SIGK_OK; ++i) {
        const size_t r0 = i * per, nr = std::min(per, B - r0);
        if (nr == 0) break;
        if (!xdev) {
            e = cudaMemcpyAsync(xbuf + r0 * L * d, X + r0 * L * d, sizeof(Real) * nr * L * d, cudaMemcpyHostToDevice,
                                stg.hs);
            if (e != cudaSuccess) return cuda_fail(e, "H2D copy");
            cudaEventRecord(stg.ev[i], stg.hs);
            cudaStreamWaitEvent(s, stg.ev[i], 0);
        }
        rc = run_device<Real>(xbuf + r0 * L * d, (int64_t)nr, (int64_t)L, d, N, obuf + r0 * D, s, &tp, &acc);
        launches += acc.launches;
        if (rc == SIGK_OK && !odev) {
            cudaEventRecord(stg.ev[Staging::kPieces + i], s);
            cudaStreamWaitEvent(stg.ds, stg.ev[Staging::kPieces + i], 0);
            e = cudaMemcpyAsync(out + r0 * D, obuf + r0 * D, sizeof(Real) * nr * D, cudaMemcpyDeviceToHost, stg.ds);
            if (e != cudaSuccess) rc = cuda_fail(e, "D2H copy");
        }
    }
    cudaEventRecord(stg.ev[2 * Staging::kPieces + 1], stg.ds);
    cudaStreamWaitEvent(s, stg.ev[2 * Staging::kPieces + 1], 0);
    e = cudaStreamSynchronize(s);
    if (e != cudaSuccess && rc == SIGK_OK) rc = cuda_fail(e, "stream synchronize");
    if (st) {
        *st = acc;
        st->launches = launches;
    }
    return rc;
}

// Elementwise utilities (increments, scaled increments): device buffers run
// asynchronously on `stream`; host buffers go through a stream-ordered
// device copy and the call returns when the result is back.
template <typename Real, typename Launch>
static int elementwise_call(const Real* in, size_t n_in, Real* out, size_t n_out, unsigned flags, void* stream,
                            Launch&& launch) {
    cudaStream_t s = static_cast<cudaStream_t>(stream);
    const bool idev = flags & SIGK_X_ON_DEVICE, odev = flags & SIGK_OUT_ON_DEVICE;
    Real *din = const_cast<Real*>(in), *dout = out;
    cudaError_t e = cudaSuccess;
    if (!idev && n_in) {
        e = cudaMallocAsync(reinterpret_cast<void**>(&din), n_in * sizeof(Real), s);
        if (e == cudaSuccess) e = cudaMemcpyAsync(din, in, n_in * sizeof(Real), cudaMemcpyHostToDevice, s);
    }
    if (e == cudaSuccess && !odev && n_out) e = cudaMallocAsync(reinterpret_cast<void**>(&dout), n_out * sizeof(Real), s);
    if (e == cudaSuccess && n_out) {
        launch(din, dout, s);
        e = cudaPeekAtLastError();
    }
    if (e == cudaSuccess && !odev && n_out) e = cudaMemcpyAsync(out, dout, n_out * sizeof(Real), cudaMemcpyDeviceToHost, s);
    if (!idev && n_in && din) cudaFreeAsync(din, s);
    if (!odev && n_out && dout) cudaFreeAsync(dout, s);
    if (e == cudaSuccess && !(idev && odev)) e = cudaStreamSynchronize(s);
    return e == cudaSuccess ? SIGK_OK : cuda_fail(e, "elementwise kernel");
}

static unsigned elementwise_grid(size_t n) {
    const size_t want = (n + 255) / 256;
    return (unsigned)std::max<size_t>(1, std::min<size_t>(want, 148 * 16));
}

template <typename Real>
static int increments_impl(const Real* X, size_t B, size_t L, int d, Real* out, unsigned flags, void* stream) {
    g_err.clear();
    if (B < 1 || L < 1 || d < 1) return fail(SIGK_EDOMAIN, "paths: batch, len and dim must all be >= 1");
    if (X == nullptr || (out == nullptr && L > 1)) return fail(SIGK_EDOMAIN, "paths/out pointer is null");
    const size_t n_out = B * (L - 1) * (size_t)d;
    return elementwise_call<Real>(X, n_out ? B * L * (size_t)d : 0, out, n_out, flags, stream,
                                  [&](const Real* din, Real* dout, cudaStream_t s) {
                                      increments_kernel<Real><<<elementwise_grid(n_out), 256, 0, s>>>(
                                          din, (int64_t)B, (int64_t)L, d, dout);
                                  });
}

template <typename Real>
static int scaled_increments_impl(const Real* inc, size_t n, int depth, Real* out, unsigned flags, void* stream) {
    g_err.clear();
    if (depth < 1) return fail(SIGK_EDOMAIN, "depth must be >= 1, got " + std::to_string(depth));
    const size_t n_out = n * (size_t)(depth - 1);
    if (n_out && (inc == nullptr || out == nullptr)) return fail(SIGK_EDOMAIN, "increments/out pointer is null");
    return elementwise_call<Real>(inc, n_out ? n : 0, out, n_out, flags, stream,
                                  [&](const Real* din, Real* dout, cudaStream_t s) {
                                      scaled_increments_kernel<Real><<<elementwise_grid(n), 256, 0, s>>>(
                                          din, (int64_t)n, depth, dout);
                                  });
}

// Prefix stream (reference signature_stream, kernels.cpp:156-198): out is
// (B, L-1, D), row t = signature of X[0..t+1]. fp32 shapes with a pair
// variant use the two-pass chunk-pair stream kernel (stream_kernel.cuh); the
// rest use the element-parallel generic stream kernel.
// Per-(device, stream) launch epochs of the look-back stream kernel (flags
// hold the epoch of the launch that set them, so they are never reset).
static int next_stream_epoch(int dev, cudaStream_t s) {
    static std::mutex mu;
    static std::vector<std::pair<std::pair<int, cudaStream_t>, int>> tab;
    std::lock_guard<std::mutex> g(mu);
    for (auto& kv : tab)
        if (kv.first.first == dev && kv.first.second == s) return kv.second = kv.second % 0x7ffffffe + 1;
    tab.emplace_back(std::make_pair(dev, s), 1);
    return 1;
}

template <typename Real>
static int stream_device(const Real* X, int64_t B, int64_t L, int d, int N, Real* out, cudaStream_t s,
                         const sigk_tuning* tun, sigk_stats* st) {
    const bool is_f64 = sizeof(Real) == 8;
    int64_t D = 0, p = 1;
    for (int n = 0; n < N; ++n) {
        p *= d;
        D += p;
    }
    const int64_t M = L - 1;
    int dev = 0;
    cudaGetDevice(&dev);
    sigk_stats local{};
    local.segments = 1;
    local.launches = 1;
    cudaError_t e = cudaErrorInvalidValue;
    bool done = false;
    if (!is_f64 && !(tun && (tun->force_generic || tun->family == SIGK_FAMILY_GENERIC))) {
        sigk_tuning tp = tun ? *tun : sigk_tuning{};
        tp.family = SIGK_FAMILY_PAIR;
        tp.segments = 1;
        const Plan plan = cached_plan(d, N, false, dev, tp.plan_rows > 0 ? tp.plan_rows : B, M, D, &tp);
        if (plan.v && plan.v->stream_launch) {
            const bool overlap = !(tun && tun->no_overlap) &&
                                 may_overlap_previous(dev, s, X, sizeof(Real) * B * L * d, out, sizeof(Real) * B * M * D);
            // one CTA per path: when the batch leaves SMs idle, the widest
            // chunking that fits keeps more warps per SM on the copy-out
            // (C2: U 10 -> 20, 102 -> 88 µs)
            const int sms = device_info(dev).sms;
            // segments per path: one CTA per path leaves SMs idle for small
            // batches, so split each path into G pieces whose CTAs chain their
            // prefixes in-kernel; >= 64 steps per piece
            int G = tun && tun->segments > 0 ? tun->segments : 1;
            if (!(tun && tun->segments > 0)) {
                G = (int)std::max<int64_t>(1, std::min<int64_t>(4, sms / B));  // measured: B*G ~ SMs, <= 4
                while (G > 1 && M / G < 64) --G;
            }
            G = (int)std::max<int64_t>(1, std::min<int64_t>(G, M));
            int64_t SL = (M + G - 1) / G;
            // G > 1: the segment CTAs of a path chain their prefixes in-kernel
            // (decoupled look-back: CTA g waits for the row CTA g-1 publishes)
            void* pub = nullptr;
            int* flags = nullptr;
            int epoch = 0;
            if (G > 1) {
                cudaStreamCaptureStatus cap = cudaStreamCaptureStatusNone;
                cudaStreamIsCapturing(s, &cap);
                if (cap != cudaStreamCaptureStatusNone) {
                    G = 1;  // look-back epochs are host-side state: not capturable
                    SL = M;
                } else {
                    bool a1 = false, a2 = false;
                    pub = segment_scratch(dev, s, 11, sizeof(float) * B * G * D, false, &a1);
                    flags = static_cast<int*>(segment_scratch(dev, s, 12, sizeof(int) * B * G, false, &a2));
                    if (!pub || !flags) return fail(SIGK_ERESOURCE, "stream segment scratch");
                    epoch = next_stream_epoch(dev, s);
                    local.segments = G;
                }
            }
            // chunks per path: each chunk's rows of a tile leave as one bulk copy, so
            // the copy-out wants tiles of >= 4 rows per chunk; take the most chunks
            // (warps) whose double-buffered stage still holds 4-step tiles (measured,
            // C2: U 8 / TS 4 -> 73 us, 0.83 of HBM; U 10 / TS 2 82 us; U 20 / TS 1 93 us)
            int U = plan.U;
            if (!(tun && tun->chunks > 0)) {
                if (B * G <= sms)  // idle SMs: widen the chunking (more warps on the copy-out)
                    U = std::max(U, (int)std::min<int64_t>(2 * plan.v->pair_units_max, std::max<int64_t>(2, SL / 8)));
                for (int u = U / 2 * 2; u >= 2; u -= 2)
                    if (plan.v->stream_tile_steps(L, G, u) >= 4) {
                        U = u;
                        break;
                    }
            }
            for (;;) {
                e = plan.v->stream_launch(X, B, L, U, out, s, overlap, G, pub, flags, epoch);
                if (e != cudaErrorInvalidValue || U <= plan.U) break;
                cudaGetLastError();
                U = std::max(plan.U, U - 2);
            }
            if (e == cudaSuccess) {
                done = true;
                local.family = SIGK_FAMILY_PAIR;
                local.prefix_len = plan.v->Q;
                local.threads_per_unit = plan.v->P;
                local.chunks = std::max(2, U / 2 * 2);
                local.fold_steps = (SL + local.chunks - 1) / local.chunks;
            } else if (e != cudaErrorInvalidValue) {
                return cuda_fail(e, "stream launch");
            }
        }
        cudaGetLastError();
    }
    if (!done) {
        // no pair stream (fp64, large d^N): the element-parallel walk, chunk-parallel
        // along the sequence — chunk signatures by the fold kernels on the gathered
        // chunks, their prefix products at every chunk start (chunk_prefix_kernel),
        // then every (path, chunk) walks its own steps from its prefix
        may_overlap_previous(dev, s, X, 0, out, sizeof(Real) * B * M * D);
        const int sms = device_info(dev).sms;
        int U = (int)std::max<int64_t>(1, std::min<int64_t>((sms * 8 + B - 1) / B, M / 32));
        if (tun && tun->chunks > 0) U = (int)std::max<int64_t>(1, std::min<int64_t>(tun->chunks, M));
        const int64_t CL = (M + U - 1) / U;
        U = (int)((M + CL - 1) / CL);
        const void* starts = nullptr;
        std::vector<void*> tmp;
        cudaStreamCaptureStatus cap = cudaStreamCaptureStatusNone;
        cudaStreamIsCapturing(s, &cap);
        auto alloc = [&](int kind, size_t bytes) -> void* {
            bool async_alloc = false;
            void* p = segment_scratch(dev, s, kind, std::max<size_t>(bytes, 16), cap != cudaStreamCaptureStatusNone,
                                      &async_alloc);
            if (p && async_alloc) tmp.push_back(p);
            return p;
        };
        auto release = [&] {
            for (void* q : tmp) cudaFreeAsync(q, s);
        };
        int launches = 1;
        if (U > 1) {
            Real* Xseg = static_cast<Real*>(alloc(20, sizeof(Real) * B * U * (CL + 1) * d));
            Real* C = static_cast<Real*>(alloc(21, sizeof(Real) * B * U * D));
            Real* P = static_cast<Real*>(alloc(22, sizeof(Real) * B * U * D));
            if (!Xseg || !C || !P) {
                release();
                return fail(SIGK_ERESOURCE, "stream chunk scratch");
            }
            segment_gather_kernel<Real><<<(unsigned)std::min<int64_t>(B * U, (int64_t)sms * 16), 128, 0, s>>>(
                X, B, L, d, U, CL, Xseg);
            sigk_stats cst{};
            sigk_tuning ct{};
            ct.no_overlap = 1;
            const int rc = run_device<Real>(Xseg, B * U, CL + 1, d, N, C, s, &ct, &cst);
            if (rc != SIGK_OK) {
                release();
                return rc;
            }
            chunk_prefix_kernel<Real><<<(unsigned)B, 256, 0, s>>>(C, D, d, N, U, P);
            starts = P;
            launches += 2 + cst.launches;
        }
        e = is_f64 ? launch_generic_stream_f64(X, B, L, d, N, out, s, U, CL, starts)
                   : launch_generic_stream_f32(X, B, L, d, N, out, s, U, CL, starts);
        release();
        if (e != cudaSuccess) return cuda_fail(e, "generic stream launch");
        local.family = SIGK_FAMILY_GENERIC;
        local.prefix_len = -1;
        local.chunks = U;
        local.fold_steps = CL;
        local.launches = launches;
    }
    local.path_steps = M;  // pass 2 folds every step of every path once (pair) / the generic walk does
    if (st) *st = local;
    return SIGK_OK;
}

template <typename Real>
static int stream_impl(const Real* X, size_t B, size_t L, int d, int N, Real* out, unsigned flags, void* stream,
                       const sigk_tuning* tun, sigk_stats* st) {
    g_err.clear();
    int rc = validate(X, B, L, d, N, out);
    if (rc != SIGK_OK) return rc;
    if (L < 2) return fail(SIGK_EDOMAIN, "signature_stream: need at least 2 points, got L = " + std::to_string(L));
    cudaStream_t s = static_cast<cudaStream_t>(stream);
    size_t D = 0;
    sigk_sig_dim(d, N, &D);
    const size_t xbytes = sizeof(Real) * B * L * d, obytes = sizeof(Real) * B * (L - 1) * D;
    const bool xdev = flags & SIGK_X_ON_DEVICE, odev = flags & SIGK_OUT_ON_DEVICE;
    cudaError_t e;
    if (xdev && odev) {
        rc = stream_device<Real>(X, (int64_t)B, (int64_t)L, d, N, out, s, tun, st);
        if (rc == SIGK_OK) {
            e = cudaPeekAtLastError();
            if (e != cudaSuccess) rc = cuda_fail(e, "kernel launch");
        }
        return rc;
    }
    int dev = 0;
    cudaGetDevice(&dev);
    Staging& stg = staging_for(dev, s);
    std::lock_guard<std::mutex> lock(stg.mu);
    const size_t ooff = xdev ? 0 : (xbytes + 255) / 256 * 256;
    const size_t need = ooff + (odev ? 0 : obytes);
    if (stg.n < need) {
        if (stg.p) cudaFree(stg.p);
        stg.p = nullptr;
        stg.n = 0;
        e = cudaMalloc(&stg.p, need);
        if (e != cudaSuccess) return cuda_fail(e, "staging allocation");
        stg.n = need;
    }
    const Real* Xd = X;
    Real* Od = out;
    if (!xdev) {
        Real* xbuf = static_cast<Real*>(stg.p);
        e = cudaMemcpyAsync(xbuf, X, xbytes, cudaMemcpyHostToDevice, s);
        if (e != cudaSuccess) return cuda_fail(e, "H2D copy");
        Xd = xbuf;
    }
    if (!odev) Od = reinterpret_cast<Real*>(static_cast<char*>(stg.p) + ooff);
    rc = stream_device<Real>(Xd, (int64_t)B, (int64_t)L, d, N, Od, s, tun, st);
    if (rc == SIGK_OK && !odev) {
        e = cudaMemcpyAsync(out, Od, obytes, cudaMemcpyDeviceToHost, s);
        if (e != cudaSuccess) rc = cuda_fail(e, "D2H copy");
    }
    e = cudaStreamSynchronize(s);
    if (e != cudaSuccess && rc == SIGK_OK) rc = cuda_fail(e, "stream synchronize");
    return rc;
}

// The paper's parallel formulation (KernelKind::Parallel; reference
// detail::parallel_forward, sig_core.hpp:175-298, scan_kernel.cuh): N degree
// passes over a (B, M, D) workspace of per-position levels. With
// SIGK_PREFIX_ROWS the workspace is the caller's (B, L-1, D) output (the
// reference's signature_stream over the parallel kernel, kernels.cpp:183-197);
// otherwise it is stream-ordered scratch and row M-1 of every path is copied
// out. The reference's memory refusal (check_parallel_memory, :161-173) is
// applied first with the same message.
template <typename Real>
static int parallel_device(const Real* X, int64_t B, int64_t L, int d, int N, Real* out, bool prefix_rows,
                           cudaStream_t s, sigk_stats* st) {
    int64_t D = 0, p = 1;
    for (int n = 0; n < N; ++n) {
        p *= d;
        D += p;
    }
    const int64_t M = L - 1;
    sigk_stats local{};
    local.family = SIGK_FAMILY_SCAN;
    local.chunks = 1;
    local.segments = 1;
    local.prefix_len = -1;
    cudaError_t e;
    if (M == 0) {  // identity; the reference still counts its N (empty) passes (sig_core.hpp:201-206)
        if (!prefix_rows) {
            e = cudaMemsetAsync(out, 0, sizeof(Real) * B * D, s);
            if (e != cudaSuccess) return cuda_fail(e, "memset");
        }
        local.scan_passes = N;
        if (st) *st = local;
        return SIGK_OK;
    }
    ScanGeom<Real> g{};
    Real factorial = 1;
    g.pw[0] = 1;
    for (int j = 1; j <= N; ++j) {
        g.pw[j] = g.pw[j - 1] * d;
        factorial *= Real(j);
        g.inv_fact[j] = Real(1) / factorial;
        g.off[j] = g.off[j - 1] + g.pw[j];  // level j occupies [off[j-1], off[j]) of a D-row
    }
    Real* W = out;
    bool scratch = false;
    if (!prefix_rows) {
        e = cudaMallocAsync(&W, sizeof(Real) * B * M * D, s);
        if (e != cudaSuccess) return cuda_fail(e, "parallel-formulation workspace");
        scratch = true;
    }
    constexpr int NW = 32;  // 32 ranges of the sequence per (path, 32-entry tile): shorter serial walks
    for (int n = 1; n <= N && e == cudaSuccess; ++n) {
        const int64_t grid = B * ((g.pw[n] + 31) / 32);
        if (N <= 8) degree_scan_kernel<Real, NW, 8><<<(unsigned)grid, 32 * NW, 0, s>>>(X, L, d, n, M, W, D, g);
        else degree_scan_kernel<Real, NW, kScanMaxDepth><<<(unsigned)grid, 32 * NW, 0, s>>>(X, L, d, n, M, W, D, g);
        e = cudaGetLastError();
        local.scan_passes += 1;
        local.launches += 1;
    }
    if (e == cudaSuccess && !prefix_rows)  // the last position of every path (gather_position, :300-311)
        e = cudaMemcpy2DAsync(out, sizeof(Real) * D, W + (M - 1) * D, sizeof(Real) * M * D, sizeof(Real) * D, B,
                              cudaMemcpyDeviceToDevice, s);
    if (scratch) cudaFreeAsync(W, s);
    if (e != cudaSuccess) return cuda_fail(e, "parallel formulation");
    if (st) *st = local;
    return SIGK_OK;
}

template <typename Real>
static int parallel_impl(const Real* X, size_t B, size_t L, int d, int N, Real* out, size_t memory_cap,
                         unsigned flags, void* stream, sigk_stats* st) {
    g_err.clear();
    int rc = validate(X, B, L, d, N, out);
    if (rc != SIGK_OK) return rc;
    const bool prefix_rows = flags & SIGK_PREFIX_ROWS;
    if (prefix_rows && L < 2)
        return fail(SIGK_EDOMAIN, "signature_stream: need at least 2 points, got L = " + std::to_string(L));
    {  // check_parallel_memory (sig_core.hpp:161-173), same message
        long double scalars = static_cast<long double>(B) * static_cast<long double>(L);
        for (int n = 0; n < N; ++n) scalars *= static_cast<long double>(d);
        if (scalars > static_cast<long double>(memory_cap))
            return fail(SIGK_ERESOURCE, "parallel kernel: intermediate storage of ~" +
                                            std::to_string(static_cast<double>(scalars)) + " scalars exceeds cap " +
                                            std::to_string(memory_cap) + "; use the sequential kernel for this shape");
    }
    if (N > kScanMaxDepth)
        return fail(SIGK_ERESOURCE, "parallel formulation: depth " + std::to_string(N) + " exceeds " +
                                        std::to_string(kScanMaxDepth));
    cudaStream_t s = static_cast<cudaStream_t>(stream);
    size_t D = 0;
    sigk_sig_dim(d, N, &D);
    const size_t rows = prefix_rows ? B * (L - 1) : B;
    const size_t xbytes = sizeof(Real) * B * L * d, obytes = sizeof(Real) * rows * D;
    const bool xdev = flags & SIGK_X_ON_DEVICE, odev = flags & SIGK_OUT_ON_DEVICE;
    cudaError_t e;
    if (xdev && odev) {
        rc = parallel_device<Real>(X, (int64_t)B, (int64_t)L, d, N, out, prefix_rows, s, st);
        if (rc == SIGK_OK) {
            e = cudaPeekAtLastError();
            if (e != cudaSuccess) rc = cuda_fail(e, "kernel launch");
        }
        return rc;
    }
    // host buffers: synchronous, stream-ordered device copies
    Real* Xd = const_cast<Real*>(X);
    Real* Od = out;
    if (!xdev) {
        e = cudaMallocAsync(&Xd, xbytes, s);
        if (e != cudaSuccess) return cuda_fail(e, "paths allocation");
        e = cudaMemcpyAsync(Xd, X, xbytes, cudaMemcpyHostToDevice, s);
        if (e != cudaSuccess) return cuda_fail(e, "H2D copy");
    }
    if (!odev) {
        e = cudaMallocAsync(&Od, obytes, s);
        if (e != cudaSuccess) return cuda_fail(e, "output allocation");
    }
    rc = parallel_device<Real>(Xd, (int64_t)B, (int64_t)L, d, N, Od, prefix_rows, s, st);
    if (rc == SIGK_OK && !odev) {
        e = cudaMemcpyAsync(out, Od, obytes, cudaMemcpyDeviceToHost, s);
        if (e != cudaSuccess) rc = cuda_fail(e, "D2H copy");
    }
    if (!xdev) cudaFreeAsync(Xd, s);
    if (!odev) cudaFreeAsync(Od, s);
    e = cudaStreamSynchronize(s);
    if (e != cudaSuccess && rc == SIGK_OK) rc = cuda_fail(e, "stream synchronize");
    return rc;
}

// Reverse mode (reference signature_vjp, autodiff.cpp:218-224): the prefix
// states come from the stream kernels into stream-ordered scratch, then
// vjp_kernel walks the steps backwards (vjp_kernel.cuh).
template <typename Real>
static int vjp_device(const Real* X, int64_t B, int64_t L, int d, int N, const Real* cot, Real* grad, cudaStream_t s,
                      const sigk_tuning* tun, sigk_stats* st) {
    int64_t D = 0, p = 1;
    for (int n = 0; n < N; ++n) {
        p *= d;
        D += p;
    }
    const int64_t M = L - 1;
    cudaError_t e;
    int dev = 0;
    cudaGetDevice(&dev);
    if (st) *st = sigk_stats{};  // every field below describes this call only
    const bool pdl = !(tun && tun->no_overlap);  // sigk.h: no_overlap = never a programmatic dependent launch
    cudaStreamCaptureStatus cap = cudaStreamCaptureStatusNone;
    cudaStreamIsCapturing(s, &cap);
    // working buffers persist per (device, stream) across calls (a stream-ordered
    // allocation per call would be unmapped at every synchronize and re-mapped)
    std::vector<void*> tmp;
    int next_kind = 2;
    auto alloc = [&](void** ptr, size_t bytes) {
        bool async_alloc = false;
        *ptr = segment_scratch(dev, s, next_kind++, std::max<size_t>(bytes, 16), cap != cudaStreamCaptureStatusNone,
                               &async_alloc);
        if (*ptr == nullptr) return cudaErrorMemoryAllocation;
        if (async_alloc) tmp.push_back(*ptr);
        return cudaSuccess;
    };
    auto release = [&] {
        for (void* q : tmp) cudaFreeAsync(q, s);
    };
    // slice-parallel adjoint where a prefix length fits a warp: it walks the
    // states back by inverse steps from the chunk ends, so no per-step state is
    // stored; otherwise the element-parallel kernel reads every prefix state
    VjpSlice<Real> sl;
    if constexpr (sizeof(Real) == 4) sl = vjp_slice_for_f32(d, N);
    else sl = vjp_slice_for_f64(d, N);
    if (getenv("SIGK_VJP_ELEMENT")) sl.fn = nullptr;  // experiments: the element-parallel kernel
    Real* states = nullptr;
    if (M > 0 && !sl.fn) {
        e = alloc(reinterpret_cast<void**>(&states), sizeof(Real) * B * M * D);
        if (e != cudaSuccess) return cuda_fail(e, "vjp state allocation");
        const int rc = stream_device<Real>(X, B, L, d, N, states, s, tun, st);
        if (rc != SIGK_OK) {
            release();
            return rc;
        }
    }
    // chunk the steps so B*U CTAs fill the GPU: chunk signatures (the forward
    // kernels on the gathered chunks) give the cotangent at every chunk end
    const int sms = device_info([] { int v = 0; cudaGetDevice(&v); return v; }()).sms;
    int U = 1;
    // (the boundary pass stages 3 rows of D in shared memory, the slice shapes' chunk
    // pass at least 6; wider signatures walk whole paths)
    if (M >= 32 && (tun == nullptr || tun->chunks != 1) && (sl.fn ? 6 : 3) * sizeof(Real) * (size_t)D <= 227 * 1024) {
        // B*U items fill the GPU, and chunks stay <= ~250 steps (the backward walk is
        // latency-bound per item: long paths want more, shorter items)
        const int64_t want = std::max<int64_t>(((int64_t)sms * 8 + B - 1) / B, M / 250);
        U = (int)std::max<int64_t>(1, std::min<int64_t>(want, M / 16));
        if (sl.fn) {
            // the slice walk is issue-bound per SM: its time follows the CTAs the
            // busiest SM runs (4 warps each) times the steps per chunk, so pick U
            // in [want/2, 2 want] minimising that (ties: fewer chunks, cheaper
            // chunk passes). C2: U = 9 (2 CTAs per SM x 111 steps) beats 10 (3 x 100).
            int64_t best = -1;
            // (U = 1 included: when the batch alone fills the GPU one full-path
            // walk per item beats the gather + chunk-signature + chunk passes)
            const int64_t lo = std::max<int64_t>(1, want / 2), hi = std::min<int64_t>(2 * want, M / 16);
            for (int64_t u = lo; u <= hi; ++u) {
                const int64_t cl = (M + u - 1) / u, ctas = (B * u + 4 * sl.slots - 1) / (4 * sl.slots);
                const int64_t cost = (ctas + sms - 1) / sms * cl;
                if (best < 0 || cost < best) {
                    best = cost;
                    U = (int)u;
                }
            }
        }
        if (tun && tun->chunks > 1) U = (int)std::min<int64_t>(tun->chunks, M);
    }
    // fp32 shapes with a pair variant and a slice walk, paths short enough to fold in one
    // CTA: one launch folds every path's U chunks and runs both chunk passes in shared
    // memory (vjp_prep.cuh), replacing the chunk-signature launch, its rows and the pass
    // launch; U is the CTA chunking (<= 2 * units_max) the walk's wave model prefers.
    const Variant* prep = nullptr;
    int prepU = 0;
    int64_t prepCL = 0;
    if constexpr (sizeof(Real) == 4) {
        // one fold-and-passes CTA per path and SM (512 threads x 128 registers): only
        // batches that fit one wave (B = 1024, L = 200 measured 263 vs 80 us otherwise),
        // and paths long enough that the launches it saves outweigh its serial passes
        // (measured: 72 vs 76 us at 128 x 1000, 69 vs 74 at 32 x 2000; 29 vs 25 at
        // 16 x 500 (d 2, N 6), 23 vs 21 at 64 x 300 (d 4, N 4))
        if (sl.fn && M >= kPrepMinSteps && B <= sms && !(tun && tun->chunks > 0) && !getenv("SIGK_VJP_NO_PREP")) {
            const Variant* cands[8];
            const int nc = find_variants(d, N, false, cands, 8);
            for (int i = 0; i < nc; ++i) {
                const Variant* v = cands[i];
                if (v->family != KernelFamily::Pair || !v->vjp_prep_launch) continue;
                // the fold CTA takes up to 2 * units_max chunks; among those chunkings pick the
                // one the walk likes (its CTAs per SM x steps per chunk, the model of the
                // chunk search above; ties: more chunks, a wider fold). C2: U = 18
                // (576 walk CTAs = 4 per SM x 56 steps): 71.4 us vs 78.0 at U = 20 (5 x 50)
                const int umax = std::min(2 * v->pair_units_max, kPrepMaxChunks);
                int64_t best = -1;
                int ub = 0;
                for (int uc = 2; uc <= umax; uc += 2) {
                    const int64_t cl = (M + uc - 1) / uc;
                    if (cl > kPrepMaxChunkSteps || v->vjp_prep_smem(uc, (int)cl, L) > 227 * 1024) continue;
                    const int64_t r = (M + cl - 1) / cl, ctas = (B * r + 4 * sl.slots - 1) / (4 * sl.slots);
                    const int64_t cost = (ctas + sms - 1) / sms * cl;
                    if (best < 0 || cost <= best) {
                        best = cost;
                        ub = uc;
                    }
                }
                if (const char* f = getenv("SIGK_VJP_PREP_U")) ub = std::max(2, std::min(umax, atoi(f) / 2 * 2));  // experiments
                if (ub == 0) continue;
                prep = v;
                prepU = ub;
                prepCL = (M + ub - 1) / ub;
                break;
            }
        }
    }
    if (prep) U = (int)((M + prepCL - 1) / prepCL);
    const int64_t CL = prep ? prepCL : (M > 0 ? (M + U - 1) / U : 1);
    if (M > 0) U = (int)((M + CL - 1) / CL);
    int launches = 0;
    const Real* cbars = cot;
    Real* ends = nullptr;  // slice path: forward prefix at every chunk end
    if (prep) {
        Real* cb = nullptr;
        e = alloc(reinterpret_cast<void**>(&ends), sizeof(Real) * B * U * D);
        if (e == cudaSuccess) e = alloc(reinterpret_cast<void**>(&cb), sizeof(Real) * B * U * D);
        if (e == cudaSuccess) e = prep->vjp_prep_launch(X, B, L, prepU, (int)CL, U, cot, ends, cb, grad, s);
        if (e != cudaSuccess) {
            release();
            return cuda_fail(e, "vjp fold-and-passes launch");
        }
        cbars = cb;
        launches += 1;
    } else if (U == 1 && M > 0 && sl.fn) {
        e = alloc(reinterpret_cast<void**>(&ends), sizeof(Real) * B * D);
        if (e != cudaSuccess) {
            release();
            return cuda_fail(e, "vjp allocation");
        }
        sigk_stats cst{};
        const int rc = run_device<Real>(X, B, L, d, N, ends, s, nullptr, &cst);  // one chunk: the signature
        if (rc != SIGK_OK) {
            release();
            return rc;
        }
        launches += cst.launches;
    }
    if (U > 1 && !prep) {
        Real *Xseg = nullptr, *C = nullptr, *cb = nullptr;
        e = alloc(reinterpret_cast<void**>(&Xseg), sizeof(Real) * B * U * (CL + 1) * d);
        if (e == cudaSuccess) e = alloc(reinterpret_cast<void**>(&C), sizeof(Real) * B * U * D);
        if (e == cudaSuccess) e = alloc(reinterpret_cast<void**>(&cb), sizeof(Real) * B * U * D);
        if (e != cudaSuccess) {
            release();
            return cuda_fail(e, "vjp chunk allocation");
        }
        // chunk signatures: the forward kernels on the chunks as paths of CL + 1 points, read
        // in place where the plan is the pair family, else gathered first
        sigk_stats cst{};
        const SubPaths sub{U, CL, L};
        int rc = getenv("SIGK_VJP_GATHER") ? kNeedGather : run_device<Real>(X, B * U, CL + 1, d, N, C, s, nullptr, &cst, &sub);
        if (rc == kNeedGather) {
            segment_gather_kernel<Real><<<(unsigned)std::min<int64_t>(B * U, (int64_t)sms * 16), 128, 0, s>>>(X, B, L, d, U, CL, Xseg);
            launches += 1;
            rc = run_device<Real>(Xseg, B * U, CL + 1, d, N, C, s, nullptr, &cst);
        }
        if (rc != SIGK_OK) {
            release();
            return rc;
        }
        const size_t bsm = 3 * sizeof(Real) * (size_t)D;
        cbars = cb;
        launches += cst.launches;
        if (sl.fn) {
            if ((e = alloc(reinterpret_cast<void**>(&ends), sizeof(Real) * B * U * D)) != cudaSuccess) {
                release();
                return cuda_fail(e, "vjp allocation");
            }
        }
        const size_t ssm = ((size_t)U * D + (size_t)2 * U * (D - p) + D) * sizeof(Real);  // ScanPasses::smem (p = d^N)
        if (sl.scan && !getenv("SIGK_VJP_SERIAL_PASSES") && ssm <= 220 * 1024) {
            // slice shapes: both passes by degree, every chunk at once
            if (ssm > 48 * 1024)
                cudaFuncSetAttribute(sl.scan, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)ssm);
            sl.scan<<<(unsigned)(2 * B), 512, ssm, s>>>(C, cot, U, 1, cb, ends, L, CL, grad);
            launches += 1;
        } else if (sl.fn) {  // slice shapes: boundary and ends in one compile-time pass per path
            const size_t rsm = (size_t)(U + 4) * D * sizeof(Real);
            const int resident = rsm <= 200 * 1024;
            const size_t psm = resident ? rsm : 6 * D * sizeof(Real);
            if (psm > 48 * 1024)
                cudaFuncSetAttribute(sl.passes, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)std::min<size_t>(psm, 227 * 1024));
            sl.passes<<<(unsigned)B, 256, psm, s>>>(C, cot, U, resident, cb, ends, L, CL, grad);
            launches += 1;
        } else {
            if (bsm > 48 * 1024)
                cudaFuncSetAttribute(vjp_boundary_kernel<Real>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)std::min<size_t>(bsm, 227 * 1024));
            vjp_boundary_kernel<Real><<<(unsigned)B, 256, bsm, s>>>(C, cot, cb, U, d, N, D);
            launches += 1;
        }
    }
    Real* dbar = nullptr;  // element-parallel kernel: δ̄ rows, then vjp_grad_kernel
    if (M > 0 && !sl.fn && (e = alloc(reinterpret_cast<void**>(&dbar), sizeof(Real) * B * M * d)) != cudaSuccess) {
        release();
        return cuda_fail(e, "vjp allocation");
    }
    const size_t work = sizeof(Real) * vjp_work_elems(D, d, N);
    const int use_smem = work <= 160 * 1024;
    Real* gwork = nullptr;
    if (!use_smem) {
        e = alloc(reinterpret_cast<void**>(&gwork), work * B * U);
        if (e != cudaSuccess) {
            release();
            return cuda_fail(e, "vjp work allocation");
        }
    }
    VjpKernelFn<Real> vk;
    if constexpr (sizeof(Real) == 4) vk = vjp_kernel_for_f32(d, N);
    else vk = vjp_kernel_for_f64(d, N);
    if (use_smem && work > 48 * 1024) cudaFuncSetAttribute(vk, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)work);
    if (M > 0 && sl.fn) {
        // slice-parallel adjoint: SLOTS (path, chunk) items per warp, 4 warps per CTA
        const int64_t items = B * U, per_cta = 4 * (int64_t)sl.slots;
        cudaLaunchConfig_t cfg = {};
        cfg.gridDim = dim3((unsigned)((items + per_cta - 1) / per_cta));
        cfg.blockDim = dim3(128);
        cfg.stream = s;
        cudaLaunchAttribute attr[1];
        attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
        attr[0].val.programmaticStreamSerializationAllowed = 1;
        cfg.attrs = attr;
        cfg.numAttrs = pdl ? 1 : 0;
        e = cudaLaunchKernelEx(&cfg, sl.fn, X, L, items, U, CL, static_cast<const Real*>(ends), cbars, grad);
        if (e != cudaSuccess) {
            release();
            return cuda_fail(e, "vjp slice launch");
        }
        launches += 1;
    } else if (M > 0) {
        cudaLaunchConfig_t cfg = {};
        cfg.gridDim = dim3((unsigned)(B * U));
        // most per-step loops are level-sized (d^n items): small blocks keep lanes busy;
        // SIGK_VJP_THREADS overrides (experiments)
        const char* vt = getenv("SIGK_VJP_THREADS");
        cfg.blockDim = dim3(vt ? (unsigned)atoi(vt) : 128u);  // measured: 128 beats 64 and 256 (C2, d=10 N=3)
        cfg.dynamicSmemBytes = use_smem ? work : 0;
        cfg.stream = s;
        cudaLaunchAttribute attr[1];
        attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
        attr[0].val.programmaticStreamSerializationAllowed = 1;
        cfg.attrs = attr;
        cfg.numAttrs = pdl ? 1 : 0;  // the kernel waits for its predecessor before reading anything
        e = cudaLaunchKernelEx(&cfg, vk, X, L, d, N, D, static_cast<const Real*>(states), cbars, U, CL,
                               dbar, gwork, use_smem);
        if (e != cudaSuccess) {
            release();
            return cuda_fail(e, "vjp launch");
        }
        launches += 1;
    }
    if (!(M > 0 && sl.fn)) {  // the slice walk writes ∂/∂X itself
        const int64_t ng = B * L * d;
        vjp_grad_kernel<Real><<<(unsigned)std::max<int64_t>(1, std::min<int64_t>((ng + 255) / 256, sms * 16)), 256, 0, s>>>(
            dbar, B, L, d, grad);
        launches += 1;
    }
    e = cudaPeekAtLastError();
    release();
    if (e != cudaSuccess) return cuda_fail(e, "vjp launch");
    may_overlap_previous(dev, s, X, 0, grad, sizeof(Real) * B * L * d);
    if (st) {
        st->launches += launches;
        st->chunks = U;
        st->fold_steps = CL;
        st->path_steps = covered_steps(std::max<int64_t>(M, 0), 1, U);
        st->scan_passes = 0;
        st->segments = 1;
        st->prefix_len = -1;
        st->threads_per_unit = 0;
        st->family = SIGK_FAMILY_AUTO;  // reverse mode has its own kernels (vjp_slice.cuh / vjp_kernel.cuh)
    }
    return SIGK_OK;
}

// Reverse mode of the parallel formulation (KernelKind::Parallel; the
// reference's vjp_parallel, autodiff.cpp:108-214): the forward scan passes
// materialise every level (scan_kernel.cuh), then per degree n = N..1 a
// suffix scan of the level cotangents and the cross-term distribution, the
// diagonal chain per position and the point gradient (scan_vjp.cuh).
static inline cudaStream_t s_of(void* stream) { return static_cast<cudaStream_t>(stream); }

template <typename Real>
static int vjp_parallel_device(const Real* X, int64_t B, int64_t L, int d, int N, const Real* cot, Real* grad,
                               cudaStream_t s, sigk_stats* st) {
    int64_t D = 0, p = 1;
    for (int n = 0; n < N; ++n) {
        p *= d;
        D += p;
    }
    const int64_t M = L - 1;
    sigk_stats local{};
    local.family = SIGK_FAMILY_SCAN;
    local.chunks = 1;
    local.segments = 1;
    local.prefix_len = -1;
    cudaError_t e;
    if (M == 0) {  // identity signature: zero gradient
        e = cudaMemsetAsync(grad, 0, sizeof(Real) * B * L * d, s);
        if (e != cudaSuccess) return cuda_fail(e, "memset");
        local.scan_passes = N;
        if (st) *st = local;
        return SIGK_OK;
    }
    const size_t big = sizeof(Real) * (size_t)(B * M * D);
    Real *W = nullptr, *Tb = nullptr, *Db = nullptr, *dbar = nullptr;
    e = cudaMallocAsync(&W, big, s);
    if (e == cudaSuccess) e = cudaMallocAsync(&Tb, big, s);
    if (e == cudaSuccess) e = cudaMallocAsync(&Db, big, s);
    if (e == cudaSuccess) e = cudaMallocAsync(&dbar, sizeof(Real) * (size_t)(B * M * d), s);
    auto release = [&] {
        for (Real* q : {W, Tb, Db, dbar})
            if (q) cudaFreeAsync(q, s);
    };
    if (e != cudaSuccess) {
        release();
        return cuda_fail(e, "parallel reverse-mode workspace");
    }
    sigk_stats fst{};
    int rc = parallel_device<Real>(X, B, L, d, N, W, true, s, &fst);  // every level at every position
    if (rc != SIGK_OK) {
        release();
        return rc;
    }
    ScanGeom<Real> g{};
    {
        Real factorial = 1;
        g.pw[0] = 1;
        for (int j = 1; j <= N; ++j) {
            g.pw[j] = g.pw[j - 1] * d;
            factorial *= Real(j);
            g.inv_fact[j] = Real(1) / factorial;
            g.off[j] = g.off[j - 1] + g.pw[j];
        }
    }
    e = cudaMemsetAsync(Tb, 0, big, s);
    if (e == cudaSuccess) e = cudaMemsetAsync(Db, 0, big, s);
    // seed: tbar[b, M-1] = cot[b] (every degree)
    if (e == cudaSuccess)
        e = cudaMemcpy2DAsync(Tb + (M - 1) * D, sizeof(Real) * M * D, cot, sizeof(Real) * D, sizeof(Real) * D, B,
                              cudaMemcpyDeviceToDevice, s);
    const int sms = device_info([] { int v = 0; cudaGetDevice(&v); return v; }()).sms;
    int launches = fst.launches + 1;
    constexpr int NW = 32;  // 32 ranges of the sequence per (path, 32-entry tile): shorter serial walks
    for (int n = N; n >= 1 && e == cudaSuccess; --n) {
        degree_suffix_kernel<Real, NW><<<(unsigned)(B * ((g.pw[n] + 31) / 32)), 32 * NW, 0, s>>>(n, M, Tb, Db, D, g);
        launches += 1;
        if (n >= 2 && M >= 2) {
            const int64_t work = (M - 1) * 2 * g.off[n - 1];
            const unsigned gx = (unsigned)std::max<int64_t>(1, std::min<int64_t>((work + 255) / 256, (int64_t)sms * 8));
            degree_distribute_kernel<Real><<<dim3(gx, (unsigned)B), 256, 0, s>>>(X, L, d, n, M, W, Tb, Db, D, g);
            launches += 1;
        }
        e = cudaGetLastError();
    }
    if (e == cudaSuccess) {
        const int64_t warps = B * M;
        diag_chain_kernel<Real><<<(unsigned)std::max<int64_t>(1, std::min<int64_t>((warps + 3) / 4, (int64_t)sms * 16)), 128, 0, s>>>(
            X, L, d, N, M, B, Db, D, dbar, g);
        const int64_t ng = B * L * d;
        vjp_grad_kernel<Real><<<(unsigned)std::max<int64_t>(1, std::min<int64_t>((ng + 255) / 256, (int64_t)sms * 16)), 256, 0, s>>>(
            dbar, B, L, d, grad);
        launches += 2;
        e = cudaGetLastError();
    }
    release();
    if (e != cudaSuccess) return cuda_fail(e, "parallel reverse mode");
    local.scan_passes = 2 * N;  // the forward degree passes and the reverse ones
    local.launches = launches;
    local.path_steps = M;
    local.fold_steps = 0;
    if (st) *st = local;
    return SIGK_OK;
}

template <typename Real>
static int vjp_impl(const Real* X, size_t B, size_t L, int d, int N, const Real* cot, Real* grad, unsigned flags,
                    void* stream, const sigk_tuning* tun, sigk_stats* st, bool parallel = false,
                    size_t memory_cap = 0) {
    g_err.clear();
    int rc = validate(X, B, L, d, N, grad);
    if (rc != SIGK_OK) return rc;
    if (cot == nullptr) return fail(SIGK_EDOMAIN, "signature_vjp: cotangent pointer is null");
    {
        size_t D = 0;
        sigk_sig_dim(d, N, &D);
        const auto a = reinterpret_cast<uintptr_t>(grad), ae = a + sizeof(Real) * B * L * d;
        const auto x = reinterpret_cast<uintptr_t>(X), xe = x + sizeof(Real) * B * L * d;
        const auto c = reinterpret_cast<uintptr_t>(cot), ce = c + sizeof(Real) * B * D;
        if ((a < xe && x < ae) || (a < ce && c < ae))
            return fail(SIGK_EDOMAIN, "signature_vjp: grad must not overlap the paths or the cotangent");
    }
    if (N > kGenericMaxDepth) return fail(SIGK_ERESOURCE, "signature_vjp: depth above 16 is not supported");
    if (parallel) {  // the forward formulation's storage check (vjp_parallel runs parallel_forward first)
        long double scalars = static_cast<long double>(B) * static_cast<long double>(L);
        for (int n = 0; n < N; ++n) scalars *= static_cast<long double>(d);
        if (scalars > static_cast<long double>(memory_cap))
            return fail(SIGK_ERESOURCE, "parallel kernel: intermediate storage of ~" +
                                            std::to_string(static_cast<double>(scalars)) + " scalars exceeds cap " +
                                            std::to_string(memory_cap) + "; use the sequential kernel for this shape");
    }
    auto run = [&](const Real* x, const Real* c, Real* g_) {
        return parallel ? vjp_parallel_device<Real>(x, (int64_t)B, (int64_t)L, d, N, c, g_, s_of(stream), st)
                        : vjp_device<Real>(x, (int64_t)B, (int64_t)L, d, N, c, g_, s_of(stream), tun, st);
    };
    cudaStream_t s = static_cast<cudaStream_t>(stream);
    size_t D = 0;
    sigk_sig_dim(d, N, &D);
    const size_t xbytes = sizeof(Real) * B * L * d, cbytes = sizeof(Real) * B * D;
    cudaError_t e;
    if (flags & SIGK_X_ON_DEVICE) {
        rc = run(X, cot, grad);
        if (rc == SIGK_OK) {
            e = cudaPeekAtLastError();
            if (e != cudaSuccess) rc = cuda_fail(e, "kernel launch");
        }
        return rc;
    }
    // host buffers: X, cotangent in, gradient out (synchronous)
    int dev = 0;
    cudaGetDevice(&dev);
    Staging& stg = staging_for(dev, s);
    std::lock_guard<std::mutex> lock(stg.mu);
    const size_t coff = (xbytes + 255) / 256 * 256, goff = coff + (cbytes + 255) / 256 * 256;
    const size_t need = goff + xbytes;
    if (stg.n < need) {
        if (stg.p) cudaFree(stg.p);
        stg.p = nullptr;
        stg.n = 0;
        e = cudaMalloc(&stg.p, need);
        if (e != cudaSuccess) return cuda_fail(e, "staging allocation");
        stg.n = need;
    }
    char* base = static_cast<char*>(stg.p);
    Real* xd = reinterpret_cast<Real*>(base);
    Real* cd = reinterpret_cast<Real*>(base + coff);
    Real* gd = reinterpret_cast<Real*>(base + goff);
    if ((e = cudaMemcpyAsync(xd, X, xbytes, cudaMemcpyHostToDevice, s)) != cudaSuccess) return cuda_fail(e, "H2D");
    if ((e = cudaMemcpyAsync(cd, cot, cbytes, cudaMemcpyHostToDevice, s)) != cudaSuccess) return cuda_fail(e, "H2D");
    rc = run(xd, cd, gd);
    if (rc == SIGK_OK && (e = cudaMemcpyAsync(grad, gd, xbytes, cudaMemcpyDeviceToHost, s)) != cudaSuccess)
        rc = cuda_fail(e, "D2H");
    e = cudaStreamSynchronize(s);
    if (e != cudaSuccess && rc == SIGK_OK) rc = cuda_fail(e, "stream synchronize");
    return rc;
}

// One non-blocking stream per device for the sharded entry (created once, so
// its staging buffers are reused across calls).
static cudaStream_t shard_stream(int dev) {
    static std::mutex mu;
    static std::vector<cudaStream_t> streams;
    std::lock_guard<std::mutex> g(mu);
    if ((int)streams.size() <= dev) streams.resize(dev + 1, nullptr);
    if (!streams[dev]) cudaStreamCreateWithFlags(&streams[dev], cudaStreamNonBlocking);
    return streams[dev];
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
            cudaStream_t s = shard_stream(g);
            sigk_tuning tun{};
            tun.plan_rows = (int64_t)B;  // same chunking on every shard -> bitwise equal to G = 1
            rcs[g] = signature_impl<Real>(X + b0 * L * d, nb, L, d, N, out + b0 * D, 0u, s, &tun, &sts[g]);
            errs[g] = g_err;
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

int sigk_signature_bruteforce_f64(const double* path, size_t len, int dim, int depth, int max_segments,
                                  int max_depth, int max_dim, int strict, double* out) {
    sigk::g_err.clear();
    if (len < 1 || dim < 1 || depth < 1)
        return sigk::fail(SIGK_EDOMAIN, "signature_bruteforce: len, dim and depth must be >= 1");
    if (path == nullptr || out == nullptr) return sigk::fail(SIGK_EDOMAIN, "signature_bruteforce: null pointer");
    const int segments = (int)len - 1;
    if (segments > max_segments || depth > max_depth || dim > max_dim || depth > sigk::kBruteMaxDepth)
        return sigk::fail(SIGK_ERESOURCE, "signature_bruteforce: instance exceeds limits (segments " +
                                              std::to_string(segments) + "/" + std::to_string(max_segments) +
                                              ", depth " + std::to_string(depth) + "/" + std::to_string(max_depth) +
                                              ", dim " + std::to_string(dim) + "/" + std::to_string(max_dim) + ")");
    size_t D = 0;
    sigk_sig_dim(dim, depth, &D);
    double *dp = nullptr, *dq = nullptr;
    cudaError_t e = cudaMalloc(&dp, sizeof(double) * len * dim);
    if (e == cudaSuccess) e = cudaMalloc(&dq, sizeof(double) * D);
    if (e == cudaSuccess) e = cudaMemcpy(dp, path, sizeof(double) * len * dim, cudaMemcpyHostToDevice);
    if (e == cudaSuccess) {
        sigk::bruteforce_kernel<<<(unsigned)((D + 127) / 128), 128>>>(dp, segments, dim, depth, strict, dq);
        e = cudaGetLastError();
    }
    if (e == cudaSuccess) e = cudaMemcpy(out, dq, sizeof(double) * D, cudaMemcpyDeviceToHost);
    cudaFree(dp);
    cudaFree(dq);
    return e == cudaSuccess ? SIGK_OK : sigk::cuda_fail(e, "signature_bruteforce");
}

int sigk_increments_f32(const float* X, size_t B, size_t L, int d, float* out, unsigned flags, void* stream) {
    return sigk::increments_impl<float>(X, B, L, d, out, flags, stream);
}
int sigk_increments_f64(const double* X, size_t B, size_t L, int d, double* out, unsigned flags, void* stream) {
    return sigk::increments_impl<double>(X, B, L, d, out, flags, stream);
}
int sigk_scaled_increments_f32(const float* inc, size_t n, int depth, float* out, unsigned flags, void* stream) {
    return sigk::scaled_increments_impl<float>(inc, n, depth, out, flags, stream);
}
int sigk_scaled_increments_f64(const double* inc, size_t n, int depth, double* out, unsigned flags, void* stream) {
    return sigk::scaled_increments_impl<double>(inc, n, depth, out, flags, stream);
}

int sigk_signature_stream_f32(const float* X, size_t B, size_t L, int d, int N, float* out, unsigned flags,
                              void* stream, const sigk_tuning* tuning, sigk_stats* stats) {
    return sigk::stream_impl<float>(X, B, L, d, N, out, flags, stream, tuning, stats);
}

int sigk_signature_stream_f64(const double* X, size_t B, size_t L, int d, int N, double* out, unsigned flags,
                              void* stream, const sigk_tuning* tuning, sigk_stats* stats) {
    return sigk::stream_impl<double>(X, B, L, d, N, out, flags, stream, tuning, stats);
}

int sigk_signature_parallel_f32(const float* X, size_t B, size_t L, int d, int N, float* out, size_t memory_cap,
                                unsigned flags, void* stream, sigk_stats* stats) {
    return sigk::parallel_impl<float>(X, B, L, d, N, out, memory_cap, flags, stream, stats);
}

int sigk_signature_parallel_f64(const double* X, size_t B, size_t L, int d, int N, double* out, size_t memory_cap,
                                unsigned flags, void* stream, sigk_stats* stats) {
    return sigk::parallel_impl<double>(X, B, L, d, N, out, memory_cap, flags, stream, stats);
}

int sigk_signature_vjp_f32(const float* X, size_t B, size_t L, int d, int N, const float* cotangent, float* grad,
                           unsigned flags, void* stream, const sigk_tuning* tuning, sigk_stats* stats) {
    return sigk::vjp_impl<float>(X, B, L, d, N, cotangent, grad, flags, stream, tuning, stats);
}

int sigk_signature_vjp_f64(const double* X, size_t B, size_t L, int d, int N, const double* cotangent, double* grad,
                           unsigned flags, void* stream, const sigk_tuning* tuning, sigk_stats* stats) {
    return sigk::vjp_impl<double>(X, B, L, d, N, cotangent, grad, flags, stream, tuning, stats);
}

int sigk_signature_vjp_parallel_f32(const float* X, size_t B, size_t L, int d, int N, const float* cotangent, float* grad,
                                    size_t memory_cap, unsigned flags, void* stream, sigk_stats* stats) {
    return sigk::vjp_impl<float>(X, B, L, d, N, cotangent, grad, flags, stream, nullptr, stats, true, memory_cap);
}

int sigk_signature_vjp_parallel_f64(const double* X, size_t B, size_t L, int d, int N, const double* cotangent,
                                    double* grad, size_t memory_cap, unsigned flags, void* stream, sigk_stats* stats) {
    return sigk::vjp_impl<double>(X, B, L, d, N, cotangent, grad, flags, stream, nullptr, stats, true, memory_cap);
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

int sigk_plan(size_t B, size_t L, int d, int N, int is_f64, const sigk_tuning* tuning, sigk_stats* plan) {
    sigk::g_err.clear();
    if (B < 1 || L < 1 || d < 1 || N < 1) return sigk::fail(SIGK_EDOMAIN, "plan: bad shape");
    return sigk::plan_only(B, L, d, N, is_f64 != 0, tuning, plan);
}

int sigk_has_fast_variant(int d, int N, int is_f64, int* Q) {
    const sigk::Variant* v = sigk::find_variant(d, N, is_f64 != 0);
    if (Q) *Q = v ? v->Q : -1;
    return v != nullptr;
}

const char* sigk_last_error(void) { return sigk::g_err.c_str(); }

// internal: lets the C++ API units report through sigk_last_error
void sigk_internal_set_error(const char* msg) { sigk::g_err = msg; }

int sigk_version(void) { return 200; }

}  // extern "C"

// Generic / brownian launchers (templates live in generic.cuh).
namespace sigk {
template <typename Real>
static cudaError_t gen(const void* X, int64_t B, int64_t L, int d, int N, void* out, cudaStream_t s) {
    const int64_t D = level_off(d, N);
    if (N > kGenericMaxDepth) return cudaErrorInvalidValue;
    const int64_t M = L - 1;
    int dev = 0;
    cudaGetDevice(&dev);
    const int sms = device_info(dev).sms;
    // small signatures: chunk-parallel one-thread-per-entry walks (each (path, chunk)
    // folds its own steps from the identity, generic_stream_small_kernel in signature
    // mode), then the fixed-order product of the chunk signatures per path
    const bool small = D <= 1024 && N <= 8 && d <= 16;
    if (d <= 16 && M >= 1) {
        int U = (int)std::max<int64_t>(1, std::min<int64_t>((sms * 8 + B - 1) / B, M / 32));
        const int64_t CL = (M + U - 1) / U;
        U = (int)((M + CL - 1) / CL);
        const size_t smem = sizeof(Real) * (16 + 2 * D + (CL + 1) * (int64_t)d);
        if (smem <= (small ? 48 : 200) * 1024) {
            Real* C = static_cast<Real*>(out);
            bool async_alloc = false;
            if (U > 1) {
                cudaStreamCaptureStatus cap = cudaStreamCaptureStatusNone;
                cudaStreamIsCapturing(s, &cap);
                C = static_cast<Real*>(segment_scratch(dev, s, 23, sizeof(Real) * B * U * D,
                                                       cap != cudaStreamCaptureStatusNone, &async_alloc));
                if (!C) return cudaErrorMemoryAllocation;
            }
            cudaLaunchConfig_t cfg = {};
            cfg.gridDim = dim3((unsigned)(B * U));
            cfg.blockDim = dim3(small ? (unsigned)((D + 31) / 32 * 32) : 1024u);
            cfg.dynamicSmemBytes = smem;
            cfg.stream = s;
            cudaError_t e = cudaSuccess;
            if (!small && smem > 48 * 1024)
                e = cudaFuncSetAttribute(generic_walk_kernel<Real>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                         (int)smem);
            if (e == cudaSuccess)
                e = !small ? cudaLaunchKernelEx(&cfg, generic_walk_kernel<Real>, static_cast<const Real*>(X), L, d, N, D,
                                                static_cast<Real*>(nullptr), U, CL, static_cast<const Real*>(nullptr), C)
                    : N <= 4 ? cudaLaunchKernelEx(&cfg, generic_stream_small_kernel<Real, 4>,
                                                  static_cast<const Real*>(X), L, d, N, D, static_cast<Real*>(nullptr),
                                                  U, CL, static_cast<const Real*>(nullptr), C)
                             : cudaLaunchKernelEx(&cfg, generic_stream_small_kernel<Real, 8>,
                                                  static_cast<const Real*>(X), L, d, N, D, static_cast<Real*>(nullptr),
                                                  U, CL, static_cast<const Real*>(nullptr), C);
            if (e == cudaSuccess && U > 1) {
                const size_t psm = 2 * sizeof(Real) * D;
                if (psm > 48 * 1024)
                    e = cudaFuncSetAttribute(chunk_product_kernel<Real>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                             (int)psm);
                if (e == cudaSuccess)
                    chunk_product_kernel<Real><<<(unsigned)B, 256, psm, s>>>(C, D, d, N, U, static_cast<Real*>(out));
            }
            if (async_alloc) cudaFreeAsync(C, s);
            return e == cudaSuccess ? cudaGetLastError() : e;
        }
    }
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
template <typename Real>
static cudaError_t gen_stream(const void* X, int64_t B, int64_t L, int d, int N, void* out, cudaStream_t s, int U,
                              int64_t CL, const void* starts) {
    const int64_t D = level_off(d, N);
    if (N > kGenericMaxDepth) return cudaErrorInvalidValue;
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3((unsigned)(B * U));
    cfg.blockDim = dim3(256);
    cfg.dynamicSmemBytes = sizeof(Real) * d;
    cfg.stream = s;
    const size_t small_smem = sizeof(Real) * (16 + 2 * D + (CL + 1) * (int64_t)d);
    if (D <= 1024 && N <= 8 && d <= 16 && small_smem <= 48 * 1024) {  // one thread per entry, rows + points in smem
        cfg.blockDim = dim3((unsigned)((D + 31) / 32 * 32));
        cfg.dynamicSmemBytes = small_smem;
        if (N <= 4)
            return cudaLaunchKernelEx(&cfg, generic_stream_small_kernel<Real, 4>, static_cast<const Real*>(X), L, d, N,
                                      D, static_cast<Real*>(out), U, CL, static_cast<const Real*>(starts),
                                      static_cast<Real*>(nullptr));
        return cudaLaunchKernelEx(&cfg, generic_stream_small_kernel<Real, 8>, static_cast<const Real*>(X), L, d, N, D,
                                  static_cast<Real*>(out), U, CL, static_cast<const Real*>(starts),
                                  static_cast<Real*>(nullptr));
    }
    if (d <= 16 && small_smem <= 200 * 1024) {  // rows + points in shared memory, entries strided over 1024 threads
        cfg.blockDim = dim3(1024);
        cfg.dynamicSmemBytes = small_smem;
        cudaError_t e = small_smem > 48 * 1024 ? cudaFuncSetAttribute(generic_walk_kernel<Real>,
                                                                      cudaFuncAttributeMaxDynamicSharedMemorySize,
                                                                      (int)small_smem)
                                               : cudaSuccess;
        if (e != cudaSuccess) return e;
        return cudaLaunchKernelEx(&cfg, generic_walk_kernel<Real>, static_cast<const Real*>(X), L, d, N, D,
                                  static_cast<Real*>(out), U, CL, static_cast<const Real*>(starts),
                                  static_cast<Real*>(nullptr));
    }
    return cudaLaunchKernelEx(&cfg, generic_stream_kernel<Real>, static_cast<const Real*>(X), L, d, N, D,
                              static_cast<Real*>(out), U, CL, static_cast<const Real*>(starts));
}
cudaError_t launch_generic_stream_f32(const void* X, int64_t B, int64_t L, int d, int N, void* out, cudaStream_t s,
                                      int U, int64_t CL, const void* starts) {
    return gen_stream<float>(X, B, L, d, N, out, s, U, CL, starts);
}
cudaError_t launch_generic_stream_f64(const void* X, int64_t B, int64_t L, int d, int N, void* out, cudaStream_t s,
                                      int U, int64_t CL, const void* starts) {
    return gen_stream<double>(X, B, L, d, N, out, s, U, CL, starts);
}
cudaError_t launch_brownian_f32(void* X, int64_t B, int64_t L, int d, uint64_t seed, int64_t row0, cudaStream_t s) {
    return brown<float>(X, B, L, d, seed, row0, s);
}
cudaError_t launch_brownian_f64(void* X, int64_t B, int64_t L, int d, uint64_t seed, int64_t row0, cudaStream_t s) {
    return brown<double>(X, B, L, d, seed, row0, s);
}
}  // namespace sigk
