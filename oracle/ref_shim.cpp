// TEST INFRASTRUCTURE ONLY — never linked into the product library.
//
// extern "C" shim over the UNMODIFIED reference sources in
// /root/reference/proj/src (compiled by oracle/Makefile with
// -Dsigkit=sigkit_ref so every reference symbol lives in sigkit_ref::).
// Used (a) to pin the C restatement in oracle/sig_oracle.c bit-for-bit,
// (b) to generate the golden fixtures under tests/golden/, and (c) as the
// "reference" CPU arm of bench.py (cpu_baseline.kind == "reference").
//
// Return codes mirror include/sigk.h: 0 OK, 1 DomainError, 2 ResourceError,
// 4 other exception.

#include <cstddef>
#include <cstdint>
#include <cstring>
#include <exception>
#include <string>
#include <thread>
#include <vector>

#include "sigkit/autodiff.hpp"
#include "sigkit/model.hpp"
#include "helpers.hpp"  // testutil::random_paths (reference tests/helpers.hpp:16-36)
#include "sigkit/bench.hpp"
#include "sigkit/detail/sig_core.hpp"
#include "sigkit/errors.hpp"
#include "sigkit/kernels.hpp"
#include "sigkit/oracle.hpp"
#include "sigkit/tensor_algebra.hpp"

namespace {

thread_local std::string g_err;

template <class F>
int guarded(F&& f) {
    try {
        f();
        return 0;
    } catch (const sigkit::DomainError& e) {
        g_err = e.what();
        return 1;
    } catch (const sigkit::ResourceError& e) {
        g_err = e.what();
        return 2;
    } catch (const std::exception& e) {
        g_err = e.what();
        return 4;
    }
}

sigkit::PathBatch make_batch(const double* x, std::size_t B, std::size_t L, int d) {
    sigkit::PathBatch p;
    p.batch = B;
    p.len = L;
    p.dim = d;
    p.values.assign(x, x + B * L * static_cast<std::size_t>(d));
    return p;
}

// Row-split driver: the reference core is pure per row and
// batch rows are bitwise independent (tests/test_kernels.cpp:252-263), so
// contiguous row blocks per std::thread give identical results.
template <typename Real>
void run_rows(const Real* x, std::size_t B, std::size_t L, int d, int N, Real* out, int threads) {
    const std::size_t D = sigkit::sig_dim(d, N);
    if (threads < 1) threads = 1;
    if (static_cast<std::size_t>(threads) > B) threads = static_cast<int>(B);
    if (threads == 1) {
        sigkit::detail::sequential_forward<Real>(x, B, L, d, N, out, nullptr);
        return;
    }
    std::vector<std::thread> pool;
    const std::size_t per = (B + static_cast<std::size_t>(threads) - 1) / static_cast<std::size_t>(threads);
    for (int t = 0; t < threads; ++t) {
        const std::size_t b0 = static_cast<std::size_t>(t) * per;
        if (b0 >= B) break;
        const std::size_t nb = (b0 + per <= B) ? per : B - b0;
        pool.emplace_back([=] {
            sigkit::detail::sequential_forward<Real>(x + b0 * L * static_cast<std::size_t>(d), nb, L, d, N,
                                                     out + b0 * D, nullptr);
        });
    }
    for (auto& th : pool) th.join();
}

}  // namespace

extern "C" {

const char* ref_last_error(void) { return g_err.c_str(); }

int ref_sig_dim(int d, int N, std::size_t* D) {
    return guarded([&] { *D = sigkit::sig_dim(d, N); });
}

// sigkit::signature_sequential (kernels.cpp:106-122) — the public double API.
int ref_signature_sequential(const double* x, std::size_t B, std::size_t L, int d, int N,
                             double* out, std::int64_t* fold_steps) {
    return guarded([&] {
        sigkit::KernelStats st;
        auto r = sigkit::signature_sequential(make_batch(x, B, L, d), N, &st);
        std::memcpy(out, r.flat.data(), r.flat.size() * sizeof(double));
        if (fold_steps) *fold_steps = st.fold_steps;
    });
}

// sigkit::signature_parallel (kernels.cpp:124-148) — the paper formulation.
int ref_signature_parallel(const double* x, std::size_t B, std::size_t L, int d, int N,
                           double* out, std::int64_t* scan_passes) {
    return guarded([&] {
        sigkit::KernelStats st;
        auto r = sigkit::signature_parallel(make_batch(x, B, L, d), N, &st);
        std::memcpy(out, r.flat.data(), r.flat.size() * sizeof(double));
        if (scan_passes) *scan_passes = st.scan_passes;
    });
}

// sigkit::signature_stream (kernels.cpp:156-198), sequential route.
int ref_signature_stream(const double* x, std::size_t B, std::size_t L, int d, int N, double* out) {
    return guarded([&] {
        auto r = sigkit::signature_stream(make_batch(x, B, L, d), N, sigkit::KernelKind::Sequential);
        std::memcpy(out, r.flat.data(), r.flat.size() * sizeof(double));
    });
}

// detail::sequential_forward<Real> (sig_core.hpp:120-147) on `threads`
// std::threads — the CPU baseline timed by bench.py.
int ref_sequential_forward_f64(const double* x, std::size_t B, std::size_t L, int d, int N,
                               double* out, int threads) {
    return guarded([&] { run_rows<double>(x, B, L, d, N, out, threads); });
}

int ref_sequential_forward_f32(const float* x, std::size_t B, std::size_t L, int d, int N,
                               float* out, int threads) {
    return guarded([&] { run_rows<float>(x, B, L, d, N, out, threads); });
}

// signature_bruteforce (oracle.cpp:28-96) with default OracleLimits.
int ref_bruteforce(const double* path, std::size_t L, int d, int N, double* out) {
    return guarded([&] {
        std::vector<double> p(path, path + L * static_cast<std::size_t>(d));
        auto f = sigkit::signature_bruteforce(p, L, d, N);
        std::memcpy(out, f.coeffs.data(), f.coeffs.size() * sizeof(double));
    });
}

// signature_bruteforce with the strict tuple class (oracle.cpp:28-96)
int ref_bruteforce_strict(const double* path, std::size_t L, int d, int N, double* out) {
    return guarded([&] {
        std::vector<double> p(path, path + L * static_cast<std::size_t>(d));
        auto f = sigkit::signature_bruteforce(p, L, d, N, sigkit::OracleLimits{}, sigkit::TupleClass::StrictlyIncreasing);
        std::memcpy(out, f.coeffs.data(), f.coeffs.size() * sizeof(double));
    });
}

// flatten(chen_product(unflatten(a), unflatten(b))) (tensor_algebra.cpp:80-127).
int ref_chen_product(int d, int N, const double* a, const double* b, double* c) {
    return guarded([&] {
        const std::size_t D = sigkit::sig_dim(d, N);
        sigkit::FlatSignature fa{d, N, std::vector<double>(a, a + D)};
        sigkit::FlatSignature fb{d, N, std::vector<double>(b, b + D)};
        auto r = sigkit::flatten(sigkit::chen_product(sigkit::unflatten(fa), sigkit::unflatten(fb)));
        std::memcpy(c, r.coeffs.data(), D * sizeof(double));
    });
}

// flatten(restricted_exp(v, N)) (tensor_algebra.cpp:63-78).
int ref_restricted_exp(int d, int N, const double* v, double* out) {
    return guarded([&] {
        auto r = sigkit::flatten(sigkit::restricted_exp(std::vector<double>(v, v + d), N));
        std::memcpy(out, r.coeffs.data(), r.coeffs.size() * sizeof(double));
    });
}

// make_bench_paths (bench.cpp:134-161): the reference's bench input.
int ref_make_bench_paths(std::uint64_t seed, std::size_t B, std::size_t L, int d, double* out) {
    return guarded([&] {
        auto p = sigkit::make_bench_paths(seed, B, L, d);
        std::memcpy(out, p.values.data(), p.values.size() * sizeof(double));
    });
}

// testutil::random_paths (tests/helpers.hpp:16-36): the reference tests' input.
int ref_random_paths(std::uint64_t seed, std::size_t B, std::size_t L, int d, double step_scale,
                     double* out) {
    return guarded([&] {
        auto p = testutil::random_paths(seed, B, L, d, step_scale);
        std::memcpy(out, p.values.data(), p.values.size() * sizeof(double));
    });
}

// signature_vjp (autodiff.cpp:218-224): kernel 0 = sequential (fold adjoint,
// :31-107), 1 = parallel (scan adjoint, :114-214).
int ref_signature_vjp(const double* x, std::size_t B, std::size_t L, int d, int N, const double* cot, int kernel,
                      double* grad) {
    return guarded([&] {
        sigkit::SignatureCotangent c;
        c.batch = B;
        c.dim = d;
        c.depth = N;
        c.values.assign(cot, cot + B * sigkit::sig_dim(d, N));
        auto g = sigkit::signature_vjp(make_batch(x, B, L, d), N, c,
                                       kernel == 1 ? sigkit::KernelKind::Parallel : sigkit::KernelKind::Sequential);
        std::memcpy(grad, g.values.data(), g.values.size() * sizeof(double));
    });
}

// finite_diff_grad (autodiff.cpp:226-266): central differences, step h.
int ref_finite_diff_grad(const double* x, std::size_t B, std::size_t L, int d, int N, const double* cot, double h,
                         double* grad) {
    return guarded([&] {
        sigkit::SignatureCotangent c;
        c.batch = B;
        c.dim = d;
        c.depth = N;
        c.values.assign(cot, cot + B * sigkit::sig_dim(d, N));
        auto g = sigkit::finite_diff_grad(make_batch(x, B, L, d), N, c, h);
        std::memcpy(grad, g.values.data(), g.values.size() * sizeof(double));
    });
}

// increments / scaled_increments (kernels.cpp:71-104)
int ref_increments(const double* x, std::size_t B, std::size_t L, int d, double* out) {
    return guarded([&] {
        auto inc = sigkit::increments(make_batch(x, B, L, d));
        std::memcpy(out, inc.diffs.data(), inc.diffs.size() * sizeof(double));
    });
}
int ref_scaled_increments(const double* diffs, std::size_t B, std::size_t S, int d, int depth, double* out) {
    return guarded([&] {
        sigkit::IncrementBatch inc;
        inc.batch = B;
        inc.segments = S;
        inc.dim = d;
        inc.diffs.assign(diffs, diffs + B * S * static_cast<std::size_t>(d));
        auto sc = sigkit::scaled_increments(inc, depth);
        for (std::size_t m = 0; m < sc.per_degree.size(); ++m)
            std::memcpy(out + m * inc.diffs.size(), sc.per_degree[m].data(), inc.diffs.size() * sizeof(double));
    });
}

// train (model.cpp:222-263): the reference's training loop; writes the
// per-epoch mean losses. kernel 0 sequential, 1 parallel, 2 auto; activation 0 tanh, 1 identity.
int ref_train(std::size_t n_samples, std::size_t seq_len, int sig_input_size, int depth, std::size_t batch_size,
              int epochs, double lr, std::uint64_t seed, int kernel, int activation, double* losses) {
    return guarded([&] {
        sigkit::TrainConfig c;
        c.n_samples = n_samples;
        c.seq_len = seq_len;
        c.sig_input_size = sig_input_size;
        c.depth = depth;
        c.batch_size = batch_size;
        c.epochs = epochs;
        c.learning_rate = lr;
        c.seed = seed;
        c.kernel = kernel == 0 ? sigkit::KernelKind::Sequential
                               : kernel == 1 ? sigkit::KernelKind::Parallel : sigkit::KernelKind::Auto;
        c.activation = activation == 1 ? sigkit::Activation::Identity : sigkit::Activation::Tanh;
        auto rep = sigkit::train(c);
        for (std::size_t i = 0; i < rep.epoch_losses.size(); ++i) losses[i] = rep.epoch_losses[i];
    });
}

}  // extern "C"
