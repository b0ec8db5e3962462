// integration/doctest_shim/doctest.h — a minimal doctest-compatible harness
// (doctest itself is not vendored in the reference, proj/.gitignore:2) so the
// reference's own unit suites compile unchanged against the B200 facade.
// Supports what those suites use: TEST_CASE, CHECK, REQUIRE, CHECK_THROWS_AS,
// CHECK_NOTHROW, doctest::Approx(...).epsilon(...), and
// DOCTEST_CONFIG_IMPLEMENT_WITH_MAIN. Prints one line per test case.
#pragma once
#include <chrono>
#include <cmath>
#include <cstdio>
#include <cstring>
#include <exception>
#include <functional>
#include <limits>
#include <string>
#include <vector>

namespace doctest {

class Approx {
public:
    explicit Approx(double v) : v_(v) {}
    Approx& epsilon(double e) { eps_ = e; return *this; }
    friend bool operator==(double a, const Approx& b) { return b.eq(a); }
    friend bool operator==(const Approx& b, double a) { return b.eq(a); }
    friend bool operator!=(double a, const Approx& b) { return !b.eq(a); }
    friend bool operator!=(const Approx& b, double a) { return !b.eq(a); }

private:
    bool eq(double a) const {  // doctest's rule: |a-b| < eps * (scale + max(|a|,|b|))
        return std::fabs(a - v_) < eps_ * (1.0 + std::max(std::fabs(a), std::fabs(v_)));
    }
    double v_;
    double eps_ = std::numeric_limits<float>::epsilon() * 100;
};

namespace detail {
struct Case {
    const char* name;
    const char* file;
    int line;
    void (*fn)();
};
inline std::vector<Case>& registry() {
    static std::vector<Case> r;
    return r;
}
struct Reg {
    Reg(const char* n, const char* f, int l, void (*fn)()) { registry().push_back({n, f, l, fn}); }
};
struct RequireFailed {};
inline int& failures() {
    static int f = 0;
    return f;
}
inline void fail(const char* kind, const char* expr, const char* file, int line) {
    ++failures();
    std::fprintf(stderr, "  %s:%d: %s( %s ) FAILED\n", file, line, kind, expr);
}
}  // namespace detail
}  // namespace doctest

#define DOCTEST_CAT_(a, b) a##b
#define DOCTEST_CAT(a, b) DOCTEST_CAT_(a, b)
#define TEST_CASE(name)                                                                          \
    static void DOCTEST_CAT(dt_case_, __LINE__)();                                               \
    static doctest::detail::Reg DOCTEST_CAT(dt_reg_, __LINE__)(name, __FILE__, __LINE__,         \
                                                               &DOCTEST_CAT(dt_case_, __LINE__)); \
    static void DOCTEST_CAT(dt_case_, __LINE__)()
#define CHECK(...)                                                                  \
    do {                                                                            \
        if (!(__VA_ARGS__)) doctest::detail::fail("CHECK", #__VA_ARGS__, __FILE__, __LINE__); \
    } while (0)
#define REQUIRE(...)                                                                  \
    do {                                                                              \
        if (!(__VA_ARGS__)) {                                                         \
            doctest::detail::fail("REQUIRE", #__VA_ARGS__, __FILE__, __LINE__);       \
            throw doctest::detail::RequireFailed{};                                   \
        }                                                                             \
    } while (0)
#define CHECK_THROWS_AS(expr, T)                                                     \
    do {                                                                             \
        bool dt_ok = false;                                                          \
        try {                                                                        \
            (void)(expr);                                                            \
        } catch (const T&) {                                                         \
            dt_ok = true;                                                            \
        } catch (...) {                                                              \
        }                                                                            \
        if (!dt_ok) doctest::detail::fail("CHECK_THROWS_AS", #expr ", " #T, __FILE__, __LINE__); \
    } while (0)
#define FAIL(msg)                                                                    \
    do {                                                                             \
        doctest::detail::fail("FAIL", msg, __FILE__, __LINE__);                      \
        throw doctest::detail::RequireFailed{};                                      \
    } while (0)
#define CHECK_NOTHROW(expr)                                                          \
    do {                                                                             \
        try {                                                                        \
            (void)(expr);                                                            \
        } catch (...) {                                                              \
            doctest::detail::fail("CHECK_NOTHROW", #expr, __FILE__, __LINE__);       \
        }                                                                            \
    } while (0)

#ifdef DOCTEST_CONFIG_IMPLEMENT_WITH_MAIN
int main(int argc, char** argv) {
    const char* filter = argc > 1 ? argv[1] : nullptr;
    int failed_cases = 0, run = 0;
    for (const auto& c : doctest::detail::registry()) {
        if (filter && !std::strstr(c.name, filter)) continue;
        const int before = doctest::detail::failures();
        const auto t0 = std::chrono::steady_clock::now();
        bool threw = false;
        try {
            c.fn();
        } catch (const doctest::detail::RequireFailed&) {
        } catch (const std::exception& e) {
            threw = true;
            std::fprintf(stderr, "  unexpected exception: %s\n", e.what());
        }
        const double s = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
        const bool ok = !threw && doctest::detail::failures() == before;
        failed_cases += !ok;
        ++run;
        std::printf("[%s] %s (%.2fs)\n", ok ? "PASS" : "FAIL", c.name, s);
        std::fflush(stdout);
    }
    std::printf("test cases: %d | passed: %d | failed: %d\n", run, run - failed_cases, failed_cases);
    return failed_cases ? 1 : 0;
}
#endif
