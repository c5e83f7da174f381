// ORACLE — TEST INFRASTRUCTURE ONLY.
//
// Minimal doctest-compatible harness so the reference's own unit tests
// (/root/reference/proj/tests/*.cpp, which #include <doctest.h>; the vendored
// doctest is absent, proj/.gitignore:2) compile unmodified.  Supports exactly
// the subset those suites use: TEST_CASE, CHECK, CHECK_FALSE,
// REQUIRE, FAIL, CHECK_THROWS_AS, CHECK_NOTHROW, doctest::Approx.
//
// Environment: DOCTEST_FILTER=<substring> runs only matching test cases.
#pragma once

#include <algorithm>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <exception>
#include <limits>
#include <sstream>
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
    bool matches(double other) const {
        return std::fabs(other - value_) <
               eps_ * (scale_ + std::max(std::fabs(other), std::fabs(value_)));
    }

private:
    double value_;
    double eps_ = static_cast<double>(std::numeric_limits<float>::epsilon()) * 100.0;
    double scale_ = 1.0;
};

template <typename T>
bool operator==(const T& lhs, const Approx& rhs) {
    return rhs.matches(static_cast<double>(lhs));
}
template <typename T>
bool operator==(const Approx& lhs, const T& rhs) {
    return lhs.matches(static_cast<double>(rhs));
}
template <typename T>
bool operator!=(const T& lhs, const Approx& rhs) {
    return !rhs.matches(static_cast<double>(lhs));
}

namespace detail {

struct Case {
    const char* name;
    const char* file;
    int line;
    void (*fn)();
};

inline std::vector<Case>& registry() {
    static std::vector<Case> cases;
    return cases;
}

struct State {
    long checks = 0;
    long failed_checks = 0;
    bool case_failed = false;
};

inline State& state() {
    static State s;
    return s;
}

struct Abort {};  // unwinds a failed REQUIRE / FAIL out of its test case

inline int add_case(const char* name, const char* file, int line, void (*fn)()) {
    registry().push_back({name, file, line, fn});
    return 0;
}

inline void record(bool ok, const char* kind, const char* expr, const char* file, int line) {
    State& s = state();
    ++s.checks;
    if (!ok) {
        ++s.failed_checks;
        s.case_failed = true;
        std::fprintf(stderr, "%s:%d: %s( %s ) FAILED\n", file, line, kind, expr);
    }
}

inline void stream_all(std::ostringstream&) {}
template <typename T, typename... Rest>
void stream_all(std::ostringstream& os, const T& first, const Rest&... rest) {
    os << first;
    stream_all(os, rest...);
}

template <typename... Args>
[[noreturn]] void fail(const char* file, int line, const Args&... args) {
    std::ostringstream os;
    stream_all(os, args...);
    record(false, "FAIL", os.str().c_str(), file, line);
    throw Abort{};
}

inline int run_all() {
    const char* filter = std::getenv("DOCTEST_FILTER");
    int cases = 0, failed_cases = 0;
    for (const Case& c : registry()) {
        if (filter && *filter && std::strstr(c.name, filter) == nullptr) continue;
        ++cases;
        state().case_failed = false;
        try {
            c.fn();
        } catch (const Abort&) {
        } catch (const std::exception& e) {
            std::fprintf(stderr, "%s:%d: test case '%s' threw: %s\n", c.file, c.line, c.name,
                         e.what());
            state().case_failed = true;
            ++state().failed_checks;
        } catch (...) {
            std::fprintf(stderr, "%s:%d: test case '%s' threw a non-std exception\n", c.file,
                         c.line, c.name);
            state().case_failed = true;
            ++state().failed_checks;
        }
        if (state().case_failed) {
            ++failed_cases;
            std::fprintf(stderr, "  -> test case FAILED: %s\n", c.name);
        }
    }
    std::printf("[doctest-shim] test cases: %d | %d passed | %d failed | checks: %ld | %ld failed\n",
                cases, cases - failed_cases, failed_cases, state().checks,
                state().failed_checks);
    return failed_cases == 0 ? 0 : 1;
}

}  // namespace detail
}  // namespace doctest

#define DOCTEST_CAT_IMPL(a, b) a##b
#define DOCTEST_CAT(a, b) DOCTEST_CAT_IMPL(a, b)
#define DOCTEST_ANON(prefix) DOCTEST_CAT(prefix, __LINE__)

#define TEST_CASE(name)                                                               \
    static void DOCTEST_ANON(doctest_fn_)();                                          \
    [[maybe_unused]] static const int DOCTEST_ANON(doctest_reg_) =                    \
        ::doctest::detail::add_case(name, __FILE__, __LINE__, &DOCTEST_ANON(doctest_fn_)); \
    static void DOCTEST_ANON(doctest_fn_)()

#define CHECK(...) ::doctest::detail::record(static_cast<bool>(__VA_ARGS__), "CHECK", #__VA_ARGS__, __FILE__, __LINE__)
#define CHECK_FALSE(...) ::doctest::detail::record(!static_cast<bool>(__VA_ARGS__), "CHECK_FALSE", #__VA_ARGS__, __FILE__, __LINE__)
#define REQUIRE(...)                                                                     \
    do {                                                                                 \
        const bool doctest_ok_ = static_cast<bool>(__VA_ARGS__);                         \
        ::doctest::detail::record(doctest_ok_, "REQUIRE", #__VA_ARGS__, __FILE__, __LINE__); \
        if (!doctest_ok_) throw ::doctest::detail::Abort{};                              \
    } while (0)
#define FAIL(...) ::doctest::detail::fail(__FILE__, __LINE__, __VA_ARGS__)
#define CHECK_THROWS_AS(expr, ...)                                                       \
    do {                                                                                 \
        bool doctest_ok_ = false;                                                        \
        try {                                                                            \
            static_cast<void>(expr);                                                     \
        } catch (const __VA_ARGS__&) {                                                   \
            doctest_ok_ = true;                                                          \
        } catch (...) {                                                                  \
        }                                                                                \
        ::doctest::detail::record(doctest_ok_, "CHECK_THROWS_AS", #expr, __FILE__, __LINE__); \
    } while (0)
#define CHECK_NOTHROW(...)                                                               \
    do {                                                                                 \
        bool doctest_ok_ = true;                                                         \
        try {                                                                            \
            static_cast<void>(__VA_ARGS__);                                              \
        } catch (...) {                                                                  \
            doctest_ok_ = false;                                                         \
        }                                                                                \
        ::doctest::detail::record(doctest_ok_, "CHECK_NOTHROW", #__VA_ARGS__, __FILE__, __LINE__); \
    } while (0)

#ifdef DOCTEST_CONFIG_IMPLEMENT_WITH_MAIN
int main() { return ::doctest::detail::run_all(); }
#endif
