// C++ drop-in API (include/sigkit/*.hpp) over the C ABI (include/sigk.h).
//
// Mirrors the reference public surface (/root/reference/proj/src/kernels.cpp,
// src/tensor_algebra.cpp): same validation messages and exception classes,
// same layouts. Compute goes to the GPU through sigk_signature_f64/_f32.
#include <cstdlib>
#include <string>

#include "sigk.h"
#include "sigkit/autodiff.hpp"
#include "sigkit/kernels.hpp"
#include "sigkit/oracle.hpp"
#include "sigkit/tensor_algebra.hpp"

namespace sigkit {

namespace {

[[noreturn]] void rethrow(int rc) {
    const std::string msg = sigk_last_error();
    if (rc == SIGK_EDOMAIN) throw DomainError(msg);
    if (rc == SIGK_ERESOURCE) throw ResourceError(msg);
    throw DeviceError(msg);
}

void check(int rc) {
    if (rc != SIGK_OK) rethrow(rc);
}

// kernels.cpp:13-26 — identical checks and messages.
void validate_paths(const PathBatch& p) {
    if (p.batch < 1 || p.len < 1 || p.dim < 1) throw DomainError("paths: batch, len and dim must all be >= 1");
    const std::size_t expected = p.batch * p.len * static_cast<std::size_t>(p.dim);
    if (p.values.size() != expected)
        throw DomainError("paths: values has " + std::to_string(p.values.size()) + " entries, shape implies " +
                          std::to_string(expected));
}

void validate_depth(int depth) {
    if (depth < 1) throw DomainError("depth must be >= 1, got " + std::to_string(depth));
}

// KernelStats from what the GPU actually ran (reference meaning,
// kernels.hpp:86-91, kernels.cpp:117-120, 143-146): the sequential kind runs
// the chunked Chen fold, fold_steps = the fold steps its launches applied per
// path (sigk_stats.path_steps, summed over the path's chunk units from the
// launch geometry = L-1), scan_passes = 0; the parallel kind runs the paper's
// per-degree scan formulation, fold_steps = 0, scan_passes = the degree
// passes launched (= depth). The chunk/segment decomposition of the fold is
// in the C ABI's sigk_stats.
void set_counters(const sigk_stats& st, KernelStats* stats) {
    if (!stats) return;
    if (st.family == SIGK_FAMILY_SCAN) {
        stats->fold_steps = 0;
        stats->scan_passes = st.scan_passes;
    } else {
        stats->fold_steps = st.path_steps;
        stats->scan_passes = 0;
    }
}

SignatureBatch run_gpu(const PathBatch& paths, int depth, KernelStats* stats, KernelKind kind,
                       std::size_t memory_cap = kDefaultParallelMemoryCap) {
    validate_paths(paths);
    validate_depth(depth);
    SignatureBatch out;
    out.batch = paths.batch;
    out.dim = paths.dim;
    out.depth = depth;
    out.flat.resize(paths.batch * sig_dim(paths.dim, depth));
    sigk_stats st{};
    if (kind == KernelKind::Parallel)
        check(sigk_signature_parallel_f64(paths.values.data(), paths.batch, paths.len, paths.dim, depth,
                                          out.flat.data(), memory_cap, 0u, nullptr, &st));
    else
        check(sigk_signature_f64(paths.values.data(), paths.batch, paths.len, paths.dim, depth, out.flat.data(), 0u,
                                 nullptr, nullptr, &st));
    set_counters(st, stats);
    return out;
}

}  // namespace

PathGradient signature_vjp(const PathBatch& paths, int depth, const SignatureCotangent& cot, KernelKind kernel,
                           const ExecutionCaps& caps) {
    // same checks and messages as the reference (autodiff.cpp:12-26)
    if (paths.batch < 1 || paths.len < 1 || paths.dim < 1)
        throw DomainError("signature_vjp: batch, len and dim must all be >= 1");
    if (depth < 1) throw DomainError("signature_vjp: depth must be >= 1");
    if (cot.batch != paths.batch || cot.dim != paths.dim || cot.depth != depth)
        throw DomainError("signature_vjp: cotangent shape does not match paths/depth");
    const std::size_t width = sig_dim(paths.dim, depth);
    if (cot.values.size() != cot.batch * width)
        throw DomainError("signature_vjp: cotangent has " + std::to_string(cot.values.size()) + " values, expected " +
                          std::to_string(cot.batch * width));
    validate_paths(paths);
    const KernelKind kind = select_kernel(kernel, caps, paths.len);
    PathGradient g;
    g.batch = paths.batch;
    g.len = paths.len;
    g.dim = paths.dim;
    g.values.assign(paths.values.size(), 0.0);
    // as the reference (autodiff.cpp:218-224): Parallel runs the adjoint of the scan passes
    // (vjp_parallel, with parallel_forward's default storage cap), otherwise the fold adjoint
    if (kind == KernelKind::Parallel)
        check(sigk_signature_vjp_parallel_f64(paths.values.data(), paths.batch, paths.len, paths.dim, depth,
                                              cot.values.data(), g.values.data(), kDefaultParallelMemoryCap, 0u,
                                              nullptr, nullptr));
    else
        check(sigk_signature_vjp_f64(paths.values.data(), paths.batch, paths.len, paths.dim, depth, cot.values.data(),
                                     g.values.data(), 0u, nullptr, nullptr, nullptr));
    return g;
}

PathGradient finite_diff_grad(const PathBatch& paths, int depth, const SignatureCotangent& cot, double h) {
    PathGradient g;
    g.batch = paths.batch;
    g.len = paths.len;
    g.dim = paths.dim;
    g.values.assign(paths.values.size(), 0.0);
    PathBatch p = paths;
    const std::size_t width = sig_dim(paths.dim, depth);
    auto objective = [&](std::size_t b) {
        PathBatch one;
        one.batch = 1;
        one.len = p.len;
        one.dim = p.dim;
        one.values.assign(p.values.begin() + static_cast<std::ptrdiff_t>(b * p.len * p.dim),
                          p.values.begin() + static_cast<std::ptrdiff_t>((b + 1) * p.len * p.dim));
        const SignatureBatch s = signature(one, depth);
        double acc = 0.0;
        for (std::size_t i = 0; i < width; ++i) acc += cot.values[b * width + i] * s.flat[i];
        return acc;
    };
    for (std::size_t b = 0; b < p.batch; ++b)
        for (std::size_t i = 0; i < p.len * static_cast<std::size_t>(p.dim); ++i) {
            double& x = p.values[b * p.len * p.dim + i];
            const double x0 = x;
            x = x0 + h;
            const double fp = objective(b);
            x = x0 - h;
            const double fm = objective(b);
            x = x0;
            g.values[b * p.len * p.dim + i] = (fp - fm) / (2.0 * h);
        }
    return g;
}

PrefixSignatureBatch signature_stream(const PathBatch& paths, int depth, KernelKind kernel, const ExecutionCaps& caps,
                                      KernelStats* stats) {
    validate_paths(paths);
    validate_depth(depth);
    if (paths.len < 2)
        throw DomainError("signature_stream: need at least 2 points, got L = " + std::to_string(paths.len));
    const KernelKind kind = select_kernel(kernel, caps, paths.len);
    PrefixSignatureBatch out;
    out.batch = paths.batch;
    out.prefixes = paths.len - 1;
    out.dim = paths.dim;
    out.depth = depth;
    out.flat.resize(paths.batch * out.prefixes * sig_dim(paths.dim, depth));
    sigk_stats st{};
    if (kind == KernelKind::Parallel)  // kernels.cpp:183-197: every position of the parallel state
        check(sigk_signature_parallel_f64(paths.values.data(), paths.batch, paths.len, paths.dim, depth,
                                          out.flat.data(), kDefaultParallelMemoryCap, SIGK_PREFIX_ROWS, nullptr, &st));
    else
        check(sigk_signature_stream_f64(paths.values.data(), paths.batch, paths.len, paths.dim, depth,
                                        out.flat.data(), 0u, nullptr, nullptr, &st));
    set_counters(st, stats);
    return out;
}

std::vector<double> SignatureBatch::row(std::size_t b) const {
    const std::size_t w = width();
    return std::vector<double>(flat.begin() + static_cast<std::ptrdiff_t>(b * w),
                               flat.begin() + static_cast<std::ptrdiff_t>((b + 1) * w));
}

std::size_t PrefixSignatureBatch::width() const {
    const std::size_t rows = batch * prefixes;
    return rows == 0 ? 0 : flat.size() / rows;
}

std::vector<double> PrefixSignatureBatch::row(std::size_t b, std::size_t k) const {
    const std::size_t w = width();
    const std::size_t s = (b * prefixes + k) * w;
    return std::vector<double>(flat.begin() + static_cast<std::ptrdiff_t>(s),
                               flat.begin() + static_cast<std::ptrdiff_t>(s + w));
}

const char* kernel_name(KernelKind kind) {
    switch (kind) {
        case KernelKind::Sequential: return "sequential";
        case KernelKind::Parallel: return "parallel";
        case KernelKind::Auto: return "auto";
    }
    return "unknown";
}

KernelKind kernel_from_name(const std::string& name) {
    if (name == "sequential") return KernelKind::Sequential;
    if (name == "parallel") return KernelKind::Parallel;
    if (name == "auto") return KernelKind::Auto;
    throw DomainError("unknown kernel '" + name + "', expected sequential, parallel or auto");
}

ExecutionCaps ExecutionCaps::detect() {
    ExecutionCaps caps;
    const char* env = std::getenv("SIGKIT_ACCELERATED");
    caps.accelerated = env != nullptr && std::string(env) != "0" && std::string(env) != "";  // kernels.cpp:64-69
    return caps;
}

KernelKind select_kernel(KernelKind hint, const ExecutionCaps& caps, std::size_t seq_len) {
    if (hint != KernelKind::Auto) return hint;
    return (caps.accelerated && seq_len >= caps.parallel_min_len) ? KernelKind::Parallel : KernelKind::Sequential;
}

FlatSignature signature_bruteforce(const std::vector<double>& path, std::size_t len, int dim, int depth,
                                   const OracleLimits& limits, TupleClass tuples) {
    if (len < 1 || dim < 1 || depth < 1) throw DomainError("signature_bruteforce: len, dim and depth must be >= 1");
    if (path.size() != len * static_cast<std::size_t>(dim))
        throw DomainError("signature_bruteforce: path size does not match (len, dim)");
    FlatSignature out;
    out.dim = dim;
    out.depth = depth;
    out.coeffs.assign(sig_dim(dim, depth), 0.0);
    const int rc = sigk_signature_bruteforce_f64(path.data(), len, dim, depth, limits.max_segments, limits.max_depth,
                                                 limits.max_dim, tuples == TupleClass::StrictlyIncreasing ? 1 : 0,
                                                 out.coeffs.data());
    if (rc != SIGK_OK) rethrow(rc);
    return out;
}

IncrementBatch increments(const PathBatch& paths) {
    validate_paths(paths);
    IncrementBatch inc;
    inc.batch = paths.batch;
    inc.segments = paths.len - 1;
    inc.dim = paths.dim;
    inc.diffs.resize(inc.batch * inc.segments * static_cast<std::size_t>(inc.dim));
    const int rc = sigk_increments_f64(paths.values.data(), paths.batch, paths.len, paths.dim, inc.diffs.data(), 0u,
                                       nullptr);
    if (rc != SIGK_OK) rethrow(rc);
    return inc;
}

ScaledIncrements scaled_increments(const IncrementBatch& inc, int depth) {
    validate_depth(depth);
    ScaledIncrements sc;
    sc.batch = inc.batch;
    sc.segments = inc.segments;
    sc.dim = inc.dim;
    sc.depth = depth;
    const std::size_t n = inc.diffs.size();
    std::vector<double> all(n * static_cast<std::size_t>(depth - 1));
    const int rc = sigk_scaled_increments_f64(inc.diffs.data(), n, depth, all.data(), 0u, nullptr);
    if (rc != SIGK_OK) rethrow(rc);
    for (int m = 2; m <= depth; ++m)
        sc.per_degree.emplace_back(all.begin() + static_cast<std::ptrdiff_t>((m - 2) * n),
                                   all.begin() + static_cast<std::ptrdiff_t>((m - 1) * n));
    return sc;
}

SignatureBatch signature_sequential(const PathBatch& paths, int depth, KernelStats* stats) {
    return run_gpu(paths, depth, stats, KernelKind::Sequential);
}

SignatureBatch signature_parallel(const PathBatch& paths, int depth, KernelStats* stats, std::size_t memory_cap) {
    // the C ABI applies the reference's refusal (sig_core.hpp:161-173) with the same message
    return run_gpu(paths, depth, stats, KernelKind::Parallel, memory_cap);
}

SignatureBatch signature(const PathBatch& paths, int depth, KernelKind kernel, const ExecutionCaps& caps,
                         KernelStats* stats) {
    validate_paths(paths);
    return run_gpu(paths, depth, stats, select_kernel(kernel, caps, paths.len));
}

void signature_f32(const float* paths, std::size_t batch, std::size_t len, int dim, int depth, float* out,
                   KernelStats* stats) {
    sigk_stats st{};
    check(sigk_signature_f32(paths, batch, len, dim, depth, out, 0u, nullptr, nullptr, &st));
    set_counters(st, stats);  // the float core is sequential_forward<float>
}

// ---- tensor algebra (host utilities; semantics of tensor_algebra.cpp:10-127)

std::size_t sig_dim(int dim, int depth) {
    std::size_t D = 0;
    check(sigk_sig_dim(dim, depth, &D));
    return D;
}

std::vector<std::size_t> level_sizes(int dim, int depth) {
    const auto off = level_offsets(dim, depth);
    std::vector<std::size_t> s(static_cast<std::size_t>(depth));
    for (int n = 0; n < depth; ++n) s[static_cast<std::size_t>(n)] = off[n + 1] - off[n];
    return s;
}

std::vector<std::size_t> level_offsets(int dim, int depth) {
    std::vector<std::size_t> off(static_cast<std::size_t>(depth > 0 ? depth + 1 : 1));
    check(sigk_level_offsets(dim, depth, off.data()));
    return off;
}

TruncatedTensor TruncatedTensor::zero(int dim, int depth) {
    TruncatedTensor t;
    t.dim = dim;
    t.depth = depth;
    for (std::size_t sz : level_sizes(dim, depth)) t.levels.emplace_back(sz, 0.0);
    return t;
}

std::vector<double> tensor_product(const std::vector<double>& a, const std::vector<double>& b) {
    std::vector<double> out;
    out.reserve(a.size() * b.size());
    for (double x : a)
        for (double y : b) out.push_back(x * y);
    return out;
}

TruncatedTensor restricted_exp(const std::vector<double>& v, int depth) {
    if (v.empty()) throw DomainError("restricted_exp: empty increment");
    TruncatedTensor t = TruncatedTensor::zero(static_cast<int>(v.size()), depth);
    t.level(1) = v;
    for (int n = 2; n <= depth; ++n) {
        std::vector<double>& cur = t.level(n);
        const std::vector<double>& prev = t.level(n - 1);
        const double inv = 1.0 / n;
        std::size_t w = 0;
        for (double p : prev)
            for (double x : v) cur[w++] = p * x * inv;
    }
    return t;
}

TruncatedTensor chen_product(const TruncatedTensor& a, const TruncatedTensor& b) {
    if (a.dim != b.dim || a.depth != b.depth) throw DomainError("chen_product: operands must share dim and depth");
    TruncatedTensor c = TruncatedTensor::zero(a.dim, a.depth);
    for (int n = 1; n <= a.depth; ++n) {
        std::vector<double>& cn = c.level(n);
        for (std::size_t i = 0; i < cn.size(); ++i) cn[i] = a.level(n)[i] + b.level(n)[i];
        for (int i = 1; i < n; ++i) {
            const std::vector<double>& ai = a.level(i);
            const std::vector<double>& bj = b.level(n - i);
            std::size_t w = 0;
            for (double x : ai)
                for (double y : bj) cn[w++] += x * y;
        }
    }
    return c;
}

FlatSignature flatten(const TruncatedTensor& t) {
    FlatSignature f{t.dim, t.depth, {}};
    for (const auto& l : t.levels) f.coeffs.insert(f.coeffs.end(), l.begin(), l.end());
    return f;
}

TruncatedTensor unflatten(const FlatSignature& f) {
    if (f.coeffs.size() != sig_dim(f.dim, f.depth))
        throw DomainError("unflatten: coeffs length " + std::to_string(f.coeffs.size()) + " does not match sig_dim(" +
                          std::to_string(f.dim) + ", " + std::to_string(f.depth) + ")");
    TruncatedTensor t = TruncatedTensor::zero(f.dim, f.depth);
    std::size_t w = 0;
    for (auto& l : t.levels)
        for (double& x : l) x = f.coeffs[w++];
    return t;
}

}  // namespace sigkit
