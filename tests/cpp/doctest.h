// tests/cpp/doctest.h -- a minimal doctest-compatible runner (TEST
// INFRASTRUCTURE).  The reference's unit tests (proj/tests/test_*.cpp) include
// <doctest.h>, which is vendored under the reference's git-ignored proj/vendor/
// and absent here; this shim implements the subset they use (TEST_CASE, flat
// SUBCASE re-entry, CHECK/REQUIRE family, CHECK_THROWS_AS, doctest::Approx) so
// the reference's own tests can be compiled, unmodified, against the B200
// drop-in headers (tests/cpp/Makefile).
#pragma once

#include <algorithm>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <exception>
#include <functional>
#include <limits>
#include <string>
#include <vector>

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
    friend bool operator==(double lhs, const Approx& rhs) {
        return std::fabs(lhs - rhs.value_) <
               rhs.eps_ * (rhs.scale_ + std::max(std::fabs(lhs), std::fabs(rhs.value_)));
    }
    friend bool operator==(const Approx& lhs, double rhs) { return rhs == lhs; }
    friend bool operator!=(double lhs, const Approx& rhs) { return !(lhs == rhs); }
    friend bool operator!=(const Approx& lhs, double rhs) { return !(rhs == lhs); }
    friend bool operator<=(double lhs, const Approx& rhs) { return lhs < rhs.value_ || lhs == rhs; }
    friend bool operator>=(double lhs, const Approx& rhs) { return lhs > rhs.value_ || lhs == rhs; }
    friend bool operator<(double lhs, const Approx& rhs) { return lhs < rhs.value_ && lhs != rhs; }
    friend bool operator>(double lhs, const Approx& rhs) { return lhs > rhs.value_ && lhs != rhs; }

private:
    double value_;
    double eps_ = static_cast<double>(std::numeric_limits<float>::epsilon()) * 100;
    double scale_ = 1.0;
};

namespace detail {

struct TestCase {
    const char* name;
    const char* file;
    int line;
    void (*fn)();
};

inline std::vector<TestCase>& registry() {
    static std::vector<TestCase> r;
    return r;
}

struct Registrar {
    Registrar(const char* name, const char* file, int line, void (*fn)()) {
        registry().push_back({name, file, line, fn});
    }
};

struct State {
    int failed_checks = 0, passed_checks = 0;
    bool case_failed = false;
    // flat SUBCASE re-entry: run k enters only the k-th subcase met
    int subcase_target = 0, subcase_seen = 0;
};

inline State& state() {
    static State s;
    return s;
}

struct RequireFailed {};

inline bool enter_subcase() { return state().subcase_seen++ == state().subcase_target; }

inline void report(bool ok, const char* kind, const char* expr, const char* file, int line) {
    if (ok) {
        ++state().passed_checks;
        return;
    }
    ++state().failed_checks;
    state().case_failed = true;
    std::printf("%s:%d: %s( %s ) FAILED\n", file, line, kind, expr);
}

inline int run_all() {
    int failed_cases = 0, cases = 0;
    for (const TestCase& tc : registry()) {
        ++cases;
        state().case_failed = false;
        state().subcase_target = 0;
        for (;;) {
            state().subcase_seen = 0;
            try {
                tc.fn();
            } catch (const RequireFailed&) {
            } catch (const std::exception& e) {
                state().case_failed = true;
                ++state().failed_checks;
                std::printf("%s:%d: TEST CASE \"%s\" threw: %s\n", tc.file, tc.line, tc.name, e.what());
            }
            if (state().subcase_target + 1 < state().subcase_seen) {
                ++state().subcase_target;
                continue;
            }
            break;
        }
        if (state().case_failed) {
            ++failed_cases;
            std::printf("[FAILED] %s\n", tc.name);
        } else {
            std::printf("[ ok ] %s\n", tc.name);
        }
    }
    std::printf("[doctest-shim] test cases: %d | passed: %d | failed: %d | assertions passed: %d | failed: %d\n",
                cases, cases - failed_cases, failed_cases, state().passed_checks, state().failed_checks);
    return failed_cases ? 1 : 0;
}

}  // namespace detail
}  // namespace doctest

#define DOCTEST_CAT_(a, b) a##b
#define DOCTEST_CAT(a, b) DOCTEST_CAT_(a, b)
#define DOCTEST_TEST_CASE_IMPL(fn, name)                                                             \
    static void fn();                                                                                \
    static ::doctest::detail::Registrar DOCTEST_CAT(fn, _reg)(name, __FILE__, __LINE__, &fn);        \
    static void fn()
#define TEST_CASE(name) DOCTEST_TEST_CASE_IMPL(DOCTEST_CAT(doctest_case_, __COUNTER__), name)
#define SUBCASE(name) if (::doctest::detail::enter_subcase())
#define CHECK(...) ::doctest::detail::report(static_cast<bool>(__VA_ARGS__), "CHECK", #__VA_ARGS__, __FILE__, __LINE__)
#define CHECK_FALSE(...) \
    ::doctest::detail::report(!static_cast<bool>(__VA_ARGS__), "CHECK_FALSE", #__VA_ARGS__, __FILE__, __LINE__)
#define REQUIRE(...)                                                                                  \
    do {                                                                                              \
        const bool ok_ = static_cast<bool>(__VA_ARGS__);                                              \
        ::doctest::detail::report(ok_, "REQUIRE", #__VA_ARGS__, __FILE__, __LINE__);                  \
        if (!ok_) throw ::doctest::detail::RequireFailed{};                                           \
    } while (0)
#define FAIL(msg)                                                                                     \
    do {                                                                                              \
        ::doctest::detail::report(false, "FAIL", "", __FILE__, __LINE__);                             \
        throw ::doctest::detail::RequireFailed{};                                                     \
    } while (0)
#define CHECK_THROWS_AS(expr, type)                                                                   \
    do {                                                                                              \
        bool ok_ = false;                                                                             \
        try {                                                                                         \
            (void)(expr);                                                                             \
        } catch (const type&) {                                                                       \
            ok_ = true;                                                                               \
        } catch (...) {                                                                               \
        }                                                                                             \
        ::doctest::detail::report(ok_, "CHECK_THROWS_AS", #expr ", " #type, __FILE__, __LINE__);      \
    } while (0)
#define CHECK_NOTHROW(expr)                                                                           \
    do {                                                                                              \
        bool ok_ = true;                                                                              \
        try {                                                                                         \
            (void)(expr);                                                                             \
        } catch (...) {                                                                               \
            ok_ = false;                                                                              \
        }                                                                                             \
        ::doctest::detail::report(ok_, "CHECK_NOTHROW", #expr, __FILE__, __LINE__);                   \
    } while (0)

#ifdef DOCTEST_CONFIG_IMPLEMENT_WITH_MAIN
int main() { return ::doctest::detail::run_all(); }
#endif
