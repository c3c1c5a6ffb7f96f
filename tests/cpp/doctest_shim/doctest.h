// Minimal doctest-compatible test harness (written for this repository; the
// reference's vendor/doctest.h is not shipped with it). Supports what the
// reference's unit suites use (proj/tests/test_*.cpp): TEST_SUITE, TEST_CASE,
// CHECK / CHECK_FALSE / CHECK_NOTHROW / CHECK_THROWS_AS, REQUIRE, CAPTURE,
// doctest::Approx, and a main() with --test-suite=NAME / --test-case=NAME
// filters (DOCTEST_CONFIG_IMPLEMENT_WITH_MAIN). Test infrastructure only.
#pragma once

#include <algorithm>
#include <cmath>
#include <cstdio>
#include <cstring>
#include <exception>
#include <string>
#include <vector>

#define DOCTEST_CAT_(a, b) a##b
#define DOCTEST_CAT(a, b) DOCTEST_CAT_(a, b)

namespace doctest {

class Approx {
public:
    explicit Approx(double v) : value_(v) {}
    Approx& epsilon(double e) {
        eps_ = e;
        return *this;
    }
    Approx& scale(double s) {
        scale_ = s;
        return *this;
    }
    bool matches(double x) const {
        return std::fabs(x - value_) < eps_ * (scale_ + std::max(std::fabs(x), std::fabs(value_)));
    }
    double value() const { return value_; }

private:
    double value_;
    double eps_ = 1.1920928955078125e-05;  // 100 x float epsilon
    double scale_ = 1.0;
};
inline bool operator==(double x, const Approx& a) { return a.matches(x); }
inline bool operator==(const Approx& a, double x) { return a.matches(x); }
inline bool operator!=(double x, const Approx& a) { return !a.matches(x); }
inline bool operator!=(const Approx& a, double x) { return !a.matches(x); }

namespace detail {

struct TestCase {
    const char* name;
    const char* suite;
    void (*fn)();
    const char* file;
    int line;
};

inline std::vector<TestCase>& registry() {
    static std::vector<TestCase> r;
    return r;
}

struct State {
    int failed_checks = 0;
    int checks = 0;
};
inline State& state() {
    static State s;
    return s;
}

struct RequireFailure {};

inline int reg(const char* name, const char* suite, void (*fn)(), const char* file, int line) {
    registry().push_back(TestCase{name, suite, fn, file, line});
    return 0;
}

inline bool check(bool ok, const char* expr, const char* file, int line, bool require) {
    ++state().checks;
    if (!ok) {
        ++state().failed_checks;
        std::fprintf(stderr, "%s:%d: FAILED: %s\n", file, line, expr);
        if (require) throw RequireFailure{};
    }
    return ok;
}

}  // namespace detail
}  // namespace doctest

// the suite a TEST_CASE belongs to: TEST_SUITE opens a namespace that shadows this
inline const char* doctest_current_suite() { return ""; }

#define TEST_SUITE(name) DOCTEST_SUITE_IMPL(name, DOCTEST_CAT(doctest_suite_, __COUNTER__))
#define DOCTEST_SUITE_IMPL(name, ns)                                \
    namespace ns {                                                  \
    inline const char* doctest_current_suite() { return name; }     \
    }                                                               \
    namespace ns

#define TEST_CASE(name) DOCTEST_CASE_IMPL(name, DOCTEST_CAT(doctest_case_, __COUNTER__))
#define DOCTEST_CASE_IMPL(name, fn)                                                                      \
    static void fn();                                                                                    \
    [[maybe_unused]] static const int DOCTEST_CAT(fn, _registered) =                                     \
        doctest::detail::reg(name, doctest_current_suite(), fn, __FILE__, __LINE__);                    \
    static void fn()

#define CHECK(...) doctest::detail::check(static_cast<bool>(__VA_ARGS__), #__VA_ARGS__, __FILE__, __LINE__, false)
#define CHECK_FALSE(...) doctest::detail::check(!static_cast<bool>(__VA_ARGS__), "!(" #__VA_ARGS__ ")", __FILE__, __LINE__, false)
#define REQUIRE(...) doctest::detail::check(static_cast<bool>(__VA_ARGS__), #__VA_ARGS__, __FILE__, __LINE__, true)
#define REQUIRE_FALSE(...) doctest::detail::check(!static_cast<bool>(__VA_ARGS__), "!(" #__VA_ARGS__ ")", __FILE__, __LINE__, true)
#define CAPTURE(x) ((void)0)
#define INFO(...) ((void)0)

#define CHECK_THROWS_AS(expr, ...)                                                                    \
    do {                                                                                              \
        bool doctest_ok_ = false;                                                                     \
        try {                                                                                         \
            (void)(expr);                                                                             \
        } catch (const __VA_ARGS__&) {                                                                \
            doctest_ok_ = true;                                                                       \
        } catch (...) {                                                                               \
        }                                                                                             \
        doctest::detail::check(doctest_ok_, "CHECK_THROWS_AS(" #expr ", " #__VA_ARGS__ ")", __FILE__, \
                               __LINE__, false);                                                      \
    } while (0)
#define REQUIRE_THROWS_AS(expr, ...) CHECK_THROWS_AS(expr, __VA_ARGS__)

#define CHECK_NOTHROW(...)                                                                          \
    do {                                                                                            \
        bool doctest_ok_ = true;                                                                    \
        try {                                                                                       \
            (void)(__VA_ARGS__);                                                                    \
        } catch (...) {                                                                             \
            doctest_ok_ = false;                                                                    \
        }                                                                                           \
        doctest::detail::check(doctest_ok_, "CHECK_NOTHROW(" #__VA_ARGS__ ")", __FILE__, __LINE__, false); \
    } while (0)

#ifdef DOCTEST_CONFIG_IMPLEMENT_WITH_MAIN
int main(int argc, char** argv) {
    std::string suite, name;
    for (int i = 1; i < argc; ++i) {
        const std::string a = argv[i];
        if (a.rfind("--test-suite=", 0) == 0) suite = a.substr(13);
        if (a.rfind("--test-case=", 0) == 0) name = a.substr(12);
    }
    int run = 0, failed = 0;
    for (const auto& tc : doctest::detail::registry()) {
        if (!suite.empty() && suite != tc.suite) continue;
        if (!name.empty() && name != tc.name) continue;
        ++run;
        const int before = doctest::detail::state().failed_checks;
        bool threw = false;
        try {
            tc.fn();
        } catch (const doctest::detail::RequireFailure&) {
            threw = true;
        } catch (const std::exception& e) {
            std::fprintf(stderr, "%s:%d: test case threw: %s\n", tc.file, tc.line, e.what());
            threw = true;
        } catch (...) {
            std::fprintf(stderr, "%s:%d: test case threw an unknown exception\n", tc.file, tc.line);
            threw = true;
        }
        if (threw || doctest::detail::state().failed_checks != before) {
            ++failed;
            std::fprintf(stderr, "TEST CASE FAILED: [%s] %s\n", tc.suite, tc.name);
        }
    }
    std::printf("[doctest] test cases: %d | %d passed | %d failed | checks: %d | %d failed\n", run, run - failed,
                failed, doctest::detail::state().checks, doctest::detail::state().failed_checks);
    return failed ? 1 : 0;
}
#endif
