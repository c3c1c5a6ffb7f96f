// The reference's own kernel tests (proj/tests/test_kernels.cpp,
// proj/tests/acceptance/acceptance.cpp), restated against the drop-in C++ API
// (include/sigkit/*.hpp) backed by the B200 kernels. Built by
// tests/test_cpp_dropin.py; exits non-zero on the first failure.
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <random>
#include <string>
#include <vector>

#include "sigkit/errors.hpp"
#include "sigkit/kernels.hpp"
#include "sigkit/oracle.hpp"
#include "sigkit/tensor_algebra.hpp"

using namespace sigkit;

static int failures = 0;
#define CHECK(cond)                                                          \
    do {                                                                     \
        if (!(cond)) {                                                       \
            std::fprintf(stderr, "FAIL %s:%d: %s\n", __FILE__, __LINE__, #cond); \
            ++failures;                                                      \
        }                                                                    \
    } while (0)

static PathBatch random_paths(unsigned seed, std::size_t B, std::size_t L, int d, double step) {
    PathBatch p;
    p.batch = B;
    p.len = L;
    p.dim = d;
    p.values.assign(B * L * d, 0.0);
    std::mt19937_64 rng(seed);
    std::normal_distribution<double> nd(0.0, 1.0);
    for (std::size_t b = 0; b < B; ++b)
        for (std::size_t t = 0; t < L; ++t)
            for (int c = 0; c < d; ++c)
                p.at(b, t, c) = (t ? p.at(b, t - 1, c) : 0.0) + step * nd(rng);
    return p;
}

static double max_abs_diff(const std::vector<double>& a, const std::vector<double>& b) {
    double m = 0;
    for (std::size_t i = 0; i < a.size(); ++i) m = std::fmax(m, std::fabs(a[i] - b[i]));
    return m;
}

// test_kernels.cpp:299-315 — dispatch follows hint, capability and length;
// detect() reads SIGKIT_ACCELERATED (host logic only: runs without a GPU)
static void host_dispatch_cases() {
    ExecutionCaps plain;  // accelerated = false
    ExecutionCaps accel;
    accel.accelerated = true;
    CHECK(!plain.accelerated && plain.parallel_min_len == 64);
    CHECK(select_kernel(KernelKind::Sequential, accel, 1000) == KernelKind::Sequential);
    CHECK(select_kernel(KernelKind::Parallel, plain, 2) == KernelKind::Parallel);
    CHECK(select_kernel(KernelKind::Auto, accel, 64) == KernelKind::Parallel);
    CHECK(select_kernel(KernelKind::Auto, accel, 63) == KernelKind::Sequential);
    CHECK(select_kernel(KernelKind::Auto, plain, 1000) == KernelKind::Sequential);
    accel.parallel_min_len = 10;
    CHECK(select_kernel(KernelKind::Auto, accel, 10) == KernelKind::Parallel);

    const char* old = std::getenv("SIGKIT_ACCELERATED");
    const std::string saved = old ? old : "";
    unsetenv("SIGKIT_ACCELERATED");
    CHECK(!ExecutionCaps::detect().accelerated);
    setenv("SIGKIT_ACCELERATED", "1", 1);
    CHECK(ExecutionCaps::detect().accelerated);
    setenv("SIGKIT_ACCELERATED", "0", 1);
    CHECK(!ExecutionCaps::detect().accelerated);
    setenv("SIGKIT_ACCELERATED", "", 1);
    CHECK(!ExecutionCaps::detect().accelerated);
    if (old) setenv("SIGKIT_ACCELERATED", saved.c_str(), 1);
    else unsetenv("SIGKIT_ACCELERATED");
    CHECK(std::string(kernel_name(KernelKind::Parallel)) == "parallel");
    CHECK(kernel_from_name("sequential") == KernelKind::Sequential);
}

int main(int argc, char** argv) {
    host_dispatch_cases();
    if (argc > 1 && std::string(argv[1]) == "--host-only") {
        std::printf("%s: %d failure(s)\n", failures ? "FAILED" : "ok", failures);
        return failures ? 1 : 0;
    }

    // test_kernels.cpp:102-117 — structural counters from what the GPU ran:
    // the fold's steps per path, the scan formulation's degree passes
    {
        const PathBatch paths = random_paths(24, 2, 17, 2, 0.5);
        KernelStats stats;
        signature_sequential(paths, 3, &stats);
        CHECK(stats.fold_steps == 16 && stats.scan_passes == 0);
        signature_parallel(paths, 3, &stats);
        CHECK(stats.fold_steps == 0 && stats.scan_passes == 3);
        const PathBatch longer = random_paths(25, 1, 200, 2, 0.1);
        signature_sequential(longer, 3, &stats);
        CHECK(stats.fold_steps == 199);
        signature_parallel(longer, 3, &stats);
        CHECK(stats.scan_passes == 3);
        // the memory refusal (sig_core.hpp:161-173), before any device work
        bool threw = false;
        try { signature_parallel(longer, 3, &stats, 100); } catch (const ResourceError&) { threw = true; }
        CHECK(threw);
    }

    // acceptance.cpp:87-107 — the two GPU algorithms (chunked fold vs per-degree
    // scans) agree on a grid of shapes, including L = 1 and L = 2
    {
        double worst = 0;
        for (std::size_t L : {1, 2, 3, 17, 64, 130})
            for (int d : {1, 2, 3, 5})
                for (int N : {1, 2, 3, 4}) {
                    const PathBatch p = random_paths(static_cast<unsigned>(L * 100 + d * 10 + N), 3, L, d, 0.4);
                    const SignatureBatch a = signature(p, N, KernelKind::Sequential);
                    const SignatureBatch b = signature(p, N, KernelKind::Parallel);
                    double mx = 0;
                    for (double v : a.flat) mx = std::fmax(mx, std::fabs(v));
                    worst = std::fmax(worst, max_abs_diff(a.flat, b.flat) / (1 + mx));
                }
        CHECK(worst <= 1e-9);
        const PathBatch p = random_paths(5, 2, 40, 3, 0.3);
        ExecutionCaps accel;
        accel.accelerated = true;
        KernelStats sa, sb;
        const PrefixSignatureBatch s0 = signature_stream(p, 3, KernelKind::Sequential, accel, &sa);
        const PrefixSignatureBatch s1 = signature_stream(p, 3, KernelKind::Auto, accel, &sb);  // 40 < 64: sequential
        CHECK(max_abs_diff(s0.flat, s1.flat) == 0.0 && sa.fold_steps == 39);
        const PrefixSignatureBatch s2 = signature_stream(p, 3, KernelKind::Parallel, accel, &sb);
        CHECK(max_abs_diff(s0.flat, s2.flat) <= 1e-10 && sb.scan_passes == 3 && sb.fold_steps == 0);
    }

    // acceptance.cpp:54-58
    CHECK(sig_dim(10, 4) == 11110 && sig_dim(2, 2) == 6 && sig_dim(6, 3) == 258);

    // acceptance.cpp:195-209 — the corner path
    {
        PathBatch p;
        p.batch = 1;
        p.len = 3;
        p.dim = 2;
        p.values = {0, 0, 1, 0, 1, 1};
        const std::vector<double> expected{1, 1, 0.5, 1, 0, 0.5};
        for (KernelKind k : {KernelKind::Sequential, KernelKind::Parallel, KernelKind::Auto})
            CHECK(max_abs_diff(signature(p, 2, k).flat, expected) < 1e-12);
    }

    // test_kernels.cpp:65-74 — a single point is the identity
    {
        const SignatureBatch s = signature(random_paths(21, 2, 1, 3, 1.0), 3);
        CHECK(s.flat.size() == 2 * sig_dim(3, 3));
        for (double x : s.flat) CHECK(x == 0.0);
    }

    // test_kernels.cpp:89-100 — two points give the restricted exponential
    {
        const PathBatch p = random_paths(23, 1, 2, 3, 1.0);
        std::vector<double> v(3);
        for (int c = 0; c < 3; ++c) v[c] = p.at(0, 1, c) - p.at(0, 0, c);
        CHECK(max_abs_diff(signature_sequential(p, 4).flat, flatten(restricted_exp(v, 4)).coeffs) < 1e-14);
    }

    // test_kernels.cpp:148-171 — concatenation composes through the Chen product
    for (unsigned seed = 40; seed < 45; ++seed) {
        const PathBatch p = random_paths(seed, 1, 11, 3, 0.5);
        PathBatch head, tail;
        head.batch = tail.batch = 1;
        head.dim = tail.dim = 3;
        head.len = 5;
        tail.len = 7;
        head.values.assign(p.values.begin(), p.values.begin() + 15);
        tail.values.assign(p.values.begin() + 12, p.values.end());
        const FlatSignature a{3, 4, signature(head, 4).flat}, b{3, 4, signature(tail, 4).flat};
        CHECK(max_abs_diff(signature(p, 4).flat, flatten(chen_product(unflatten(a), unflatten(b))).coeffs) < 1e-10);
    }

    // test_kernels.cpp:207-228 — scaling by lambda scales degree n by lambda^n
    {
        const PathBatch p = random_paths(100, 1, 6, 2, 1.0);
        PathBatch s = p;
        for (double& x : s.values) x *= 2.0;
        const auto off = level_offsets(2, 4);
        const SignatureBatch a = signature(p, 4), b = signature(s, 4);
        double f = 1;
        for (int n = 1; n <= 4; ++n) {
            f *= 2.0;
            for (std::size_t i = off[n - 1]; i < off[n]; ++i) CHECK(std::fabs(b.flat[i] - f * a.flat[i]) <= 1e-10 * (1 + std::fabs(f * a.flat[i])));
        }
    }

    // test_kernels.cpp:119-126 and a long batch against the f32 entry
    {
        const SignatureBatch s = signature(random_paths(26, 1, 3, 10, 1.0), 4);
        CHECK(s.width() == 11110);
        const PathBatch p = random_paths(7, 32, 1000, 5, 1.0 / std::sqrt(999.0));
        const SignatureBatch ref = signature(p, 4);
        std::vector<float> x(p.values.begin(), p.values.end()), out(32 * 780);
        KernelStats st;
        signature_f32(x.data(), 32, 1000, 5, 4, out.data(), &st);
        double scale = 0;
        for (double v : ref.flat) scale = std::fmax(scale, std::fabs(v));
        std::vector<double> o(out.begin(), out.end());
        CHECK(max_abs_diff(o, ref.flat) <= 1e-5 * scale);
        CHECK(st.fold_steps == 999 && st.scan_passes == 0);  // reference counters (kernels.cpp:106-122)
        KernelStats sp, ss;
        signature_parallel(random_paths(8, 2, 50, 2, 0.3), 3, &sp);
        signature_sequential(random_paths(8, 2, 50, 2, 0.3), 3, &ss);
        CHECK(sp.fold_steps == 0 && sp.scan_passes == 3 && ss.fold_steps == 49 && ss.scan_passes == 0);
    }

    // test_kernels.cpp:334-346 — invalid shapes and depths, exception classes
    {
        PathBatch p;
        p.batch = 1;
        p.len = 3;
        p.dim = 2;
        p.values.assign(5, 0.0);
        bool threw = false;
        try { signature_sequential(p, 2); } catch (const DomainError&) { threw = true; }
        CHECK(threw);
        p.values.assign(6, 0.0);
        threw = false;
        try { signature(p, 0); } catch (const DomainError&) { threw = true; }
        CHECK(threw);
        threw = false;
        try { signature_parallel(random_paths(140, 4, 32, 3, 1.0), 3, nullptr, 1000); } catch (const ResourceError&) { threw = true; }
        CHECK(threw);
        threw = false;
        try { kernel_from_name("gpu"); } catch (const DomainError&) { threw = true; }
        CHECK(threw);
    }

    // increments / scaled_increments (kernels.cpp:71-104; test_kernels.cpp increment cases)
    {
        const PathBatch p = random_paths(77, 3, 9, 2, 0.5);
        const IncrementBatch inc = increments(p);
        CHECK(inc.batch == 3 && inc.segments == 8 && inc.dim == 2 && inc.diffs.size() == 48);
        bool exact = true;
        for (std::size_t b = 0; b < 3; ++b)
            for (std::size_t k = 0; k < 8; ++k)
                for (int c = 0; c < 2; ++c)
                    exact &= inc.diffs[(b * 8 + k) * 2 + c] == p.at(b, k + 1, c) - p.at(b, k, c);
        CHECK(exact);
        const ScaledIncrements sc = scaled_increments(inc, 4);
        CHECK(sc.per_degree.size() == 3 && sc.depth == 4);
        CHECK(sc.per_degree[2][5] == inc.diffs[5] / 24.0);
        PathBatch one = random_paths(78, 2, 1, 3, 1.0);
        CHECK(increments(one).diffs.empty());
        CHECK(scaled_increments(increments(p), 1).per_degree.empty());
    }

    // signature_bruteforce (oracle.hpp; test_oracle.cpp:27-45): corner path and limits
    {
        const std::vector<double> corner = {0, 0, 1, 0, 1, 1};
        const FlatSignature f = signature_bruteforce(corner, 3, 2, 2);
        const double want[6] = {1, 1, 0.5, 1, 0, 0.5};
        bool ok = f.coeffs.size() == 6;
        for (int i = 0; ok && i < 6; ++i) ok = std::abs(f.coeffs[i] - want[i]) <= 1e-12;
        CHECK(ok);
        bool threw = false;
        try { signature_bruteforce(std::vector<double>(20, 0.0), 10, 2, 2); } catch (const ResourceError&) { threw = true; }
        CHECK(threw);
    }

    std::printf("%s: %d failure(s)\n", failures ? "FAILED" : "ok", failures);
    return failures ? 1 : 0;
}
