// doctest.h -- a minimal stand-in for the doctest test framework (TEST INFRASTRUCTURE ONLY).
//
// The reference vendors doctest but does not ship it (proj/.gitignore:2), so its unit tests
// (proj/tests/test_*.cpp) cannot be built as-is in this image.  This header implements just the
// subset of the doctest interface those files use -- TEST_SUITE, TEST_CASE, CHECK, CHECK_FALSE,
// REQUIRE, REQUIRE_MESSAGE, CHECK_THROWS_AS, CHECK_THROWS_WITH_AS, FAIL, doctest::Approx -- so
// the reference's own unit tests compile unmodified against this repo's C++ API (oracle/Makefile
// target `unit`) and run on the B200 library.  Written from the documented behaviour of those
// macros; no doctest source is used.
#pragma once

#include <cmath>
#include <cstdio>
#include <exception>
#include <limits>
#include <string>
#include <vector>

namespace dtshim {

struct TestCase {
    void (*fn)();
    const char* name;
    const char* file;
    int line;
};

inline std::vector<TestCase>& registry() {
    static std::vector<TestCase> r;
    return r;
}
inline int add(void (*fn)(), const char* name, const char* file, int line) {
    registry().push_back({fn, name, file, line});
    return 0;
}

struct State {
    long long checks = 0, failed_checks = 0;
    bool case_failed = false;
};
inline State& state() {
    static State s;
    return s;
}
struct Abort {};  // thrown by a failed REQUIRE / FAIL to leave the test case

inline void report(bool ok, const char* kind, const char* expr, const char* file, int line, const std::string& extra = "") {
    ++state().checks;
    if (ok) return;
    ++state().failed_checks;
    state().case_failed = true;
    std::fprintf(stderr, "%s:%d: %s( %s ) failed%s%s\n", file, line, kind, expr, extra.empty() ? "" : ": ",
                 extra.c_str());
}

}  // namespace dtshim

namespace doctest {
// Approx: |a - b| < eps * (scale + max(|a|, |b|)), eps defaulting to 100 float epsilons.
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
    bool matches(double other) const {
        return std::fabs(other - value_) < eps_ * (scale_ + std::fmax(std::fabs(other), std::fabs(value_)));
    }
    friend bool operator==(double a, const Approx& b) { return b.matches(a); }
    friend bool operator==(const Approx& a, double b) { return a.matches(b); }
    friend bool operator!=(double a, const Approx& b) { return !b.matches(a); }
    friend bool operator!=(const Approx& a, double b) { return !a.matches(b); }
    friend bool operator<=(double a, const Approx& b) { return a < b.value_ || b.matches(a); }
    friend bool operator>=(double a, const Approx& b) { return a > b.value_ || b.matches(a); }
    friend bool operator<=(const Approx& a, double b) { return a.value_ < b || a.matches(b); }
    friend bool operator>=(const Approx& a, double b) { return a.value_ > b || a.matches(b); }

  private:
    double value_;
    double eps_ = static_cast<double>(std::numeric_limits<float>::epsilon()) * 100.0;
    double scale_ = 1.0;
};
}  // namespace doctest

#define DTSHIM_CAT_(a, b) a##b
#define DTSHIM_CAT(a, b) DTSHIM_CAT_(a, b)

// TEST_SUITE(name) { ... } opens a uniquely named namespace (suite names are not used)
#define TEST_SUITE(name) namespace DTSHIM_CAT(dtshim_suite_, __COUNTER__)

#define DTSHIM_TEST_CASE(fn, name)                                                             \
    static void fn();                                                                          \
    [[maybe_unused]] static const int DTSHIM_CAT(fn, _reg) = ::dtshim::add(fn, name, __FILE__, __LINE__); \
    static void fn()
#define TEST_CASE(name) DTSHIM_TEST_CASE(DTSHIM_CAT(dtshim_case_, __COUNTER__), name)

#define CHECK(...) ::dtshim::report(static_cast<bool>(__VA_ARGS__), "CHECK", #__VA_ARGS__, __FILE__, __LINE__)
#define CHECK_FALSE(...) ::dtshim::report(!static_cast<bool>(__VA_ARGS__), "CHECK_FALSE", #__VA_ARGS__, __FILE__, __LINE__)
#define REQUIRE(...)                                                                            \
    do {                                                                                        \
        const bool dtshim_ok = static_cast<bool>(__VA_ARGS__);                                  \
        ::dtshim::report(dtshim_ok, "REQUIRE", #__VA_ARGS__, __FILE__, __LINE__);               \
        if (!dtshim_ok) throw ::dtshim::Abort{};                                                \
    } while (0)
#define REQUIRE_MESSAGE(cond, msg)                                                              \
    do {                                                                                        \
        const bool dtshim_ok = static_cast<bool>(cond);                                         \
        ::dtshim::report(dtshim_ok, "REQUIRE_MESSAGE", #cond, __FILE__, __LINE__, std::string(msg)); \
        if (!dtshim_ok) throw ::dtshim::Abort{};                                                \
    } while (0)
#define FAIL(msg)                                                                               \
    do {                                                                                        \
        ::dtshim::report(false, "FAIL", "", __FILE__, __LINE__, std::string(msg));              \
        throw ::dtshim::Abort{};                                                                \
    } while (0)
#define CHECK_THROWS_AS(expr, ...)                                                              \
    do {                                                                                        \
        bool dtshim_ok = false;                                                                 \
        try {                                                                                   \
            static_cast<void>(expr);                                                            \
        } catch (const __VA_ARGS__&) {                                                          \
            dtshim_ok = true;                                                                   \
        } catch (...) {                                                                         \
        }                                                                                       \
        ::dtshim::report(dtshim_ok, "CHECK_THROWS_AS", #expr ", " #__VA_ARGS__, __FILE__, __LINE__); \
    } while (0)
#define CHECK_THROWS_WITH_AS(expr, msg, ...)                                                    \
    do {                                                                                        \
        bool dtshim_ok = false;                                                                 \
        std::string dtshim_what = "no exception";                                               \
        try {                                                                                   \
            static_cast<void>(expr);                                                            \
        } catch (const __VA_ARGS__& e) {                                                        \
            dtshim_what = e.what();                                                             \
            dtshim_ok = dtshim_what == std::string(msg);                                        \
        } catch (...) {                                                                         \
            dtshim_what = "other exception type";                                               \
        }                                                                                       \
        ::dtshim::report(dtshim_ok, "CHECK_THROWS_WITH_AS", #expr, __FILE__, __LINE__, dtshim_what); \
    } while (0)

#ifdef DOCTEST_CONFIG_IMPLEMENT_WITH_MAIN
int main() {
    int failed_cases = 0, total = 0;
    for (const auto& tc : ::dtshim::registry()) {
        ++total;
        ::dtshim::state().case_failed = false;
        try {
            tc.fn();
        } catch (const ::dtshim::Abort&) {
        } catch (const std::exception& e) {
            ::dtshim::report(false, "TEST_CASE", tc.name, tc.file, tc.line, std::string("unexpected exception: ") + e.what());
        } catch (...) {
            ::dtshim::report(false, "TEST_CASE", tc.name, tc.file, tc.line, "unexpected exception");
        }
        if (::dtshim::state().case_failed) {
            ++failed_cases;
            std::fprintf(stderr, "FAILED test case: %s (%s:%d)\n", tc.name, tc.file, tc.line);
        }
    }
    std::printf("[doctest shim] test cases: %d | %d passed | %d failed\n", total, total - failed_cases, failed_cases);
    std::printf("[doctest shim] assertions: %lld | %lld passed | %lld failed\n", ::dtshim::state().checks,
                ::dtshim::state().checks - ::dtshim::state().failed_checks, ::dtshim::state().failed_checks);
    return failed_cases == 0 ? 0 : 1;
}
#endif
