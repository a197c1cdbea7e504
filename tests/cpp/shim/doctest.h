// Minimal doctest-compatible test harness (the real doctest single header is
// not available offline).  Implements exactly the subset the reference's
// unit suites use: TEST_SUITE, TEST_CASE, CHECK, CHECK_FALSE, CHECK_NOTHROW,
// CHECK_THROWS_AS, REQUIRE, FAIL, doctest::Approx(...).epsilon(...), and a
// main() honouring --test-suite=<name> when DOCTEST_CONFIG_IMPLEMENT_WITH_MAIN
// is defined.  Written for this repo; only the macro names follow doctest.
#pragma once

#include <cmath>
#include <cstdio>
#include <cstring>
#include <exception>
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

private:
    double value_;
    double eps_ = std::numeric_limits<float>::epsilon() * 100;
    double scale_ = 1.0;
};

}  // namespace doctest

namespace dtshim {

struct Case {
    const char* name;
    const char* suite;
    void (*fn)();
};

inline std::vector<Case>& registry() {
    static std::vector<Case> r;
    return r;
}

struct Reg {
    Reg(const char* name, const char* suite, void (*fn)()) { registry().push_back({name, suite, fn}); }
};

struct Abort {};  // REQUIRE / FAIL stop the current test case

inline int& failures() {
    static int f = 0;
    return f;
}

inline int& asserts() {
    static int a = 0;
    return a;
}

inline void report(const char* file, int line, const char* what, const char* expr) {
    ++failures();
    std::fprintf(stderr, "%s:%d: %s( %s ) FAILED\n", file, line, what, expr);
}

inline void check(bool ok, const char* what, const char* expr, const char* file, int line, bool fatal) {
    ++asserts();
    if (ok) return;
    report(file, line, what, expr);
    if (fatal) throw Abort{};
}

}  // namespace dtshim

inline const char* dtshim_suite() { return ""; }

#define DTSHIM_CAT_(a, b) a##b
#define DTSHIM_CAT(a, b) DTSHIM_CAT_(a, b)

#define TEST_SUITE(name) DTSHIM_SUITE_(name, DTSHIM_CAT(dtshim_suite_ns_, __COUNTER__))
#define DTSHIM_SUITE_(name, ns)                       \
    namespace ns {                                    \
    inline const char* dtshim_suite() { return name; } \
    }                                                 \
    namespace ns

#define TEST_CASE(name) DTSHIM_CASE_(name, DTSHIM_CAT(dtshim_case_, __COUNTER__))
#define DTSHIM_CASE_(name, f)                                                  \
    static void f();                                                           \
    static const ::dtshim::Reg DTSHIM_CAT(f, _reg){name, dtshim_suite(), &f}; \
    static void f()

#define CHECK(...) ::dtshim::check(static_cast<bool>(__VA_ARGS__), "CHECK", #__VA_ARGS__, __FILE__, __LINE__, false)
#define CHECK_FALSE(...) \
    ::dtshim::check(!static_cast<bool>(__VA_ARGS__), "CHECK_FALSE", #__VA_ARGS__, __FILE__, __LINE__, false)
#define REQUIRE(...) ::dtshim::check(static_cast<bool>(__VA_ARGS__), "REQUIRE", #__VA_ARGS__, __FILE__, __LINE__, true)
#define FAIL(msg) ::dtshim::check(false, "FAIL", msg, __FILE__, __LINE__, true)
#define CHECK_NOTHROW(...)                                                                       \
    do {                                                                                         \
        bool dtshim_ok = true;                                                                   \
        try {                                                                                    \
            (void)(__VA_ARGS__);                                                                 \
        } catch (...) {                                                                          \
            dtshim_ok = false;                                                                   \
        }                                                                                        \
        ::dtshim::check(dtshim_ok, "CHECK_NOTHROW", #__VA_ARGS__, __FILE__, __LINE__, false);    \
    } while (0)
#define CHECK_THROWS_AS(expr, ...)                                                               \
    do {                                                                                         \
        bool dtshim_ok = false;                                                                  \
        try {                                                                                    \
            (void)(expr);                                                                        \
        } catch (const __VA_ARGS__&) {                                                           \
            dtshim_ok = true;                                                                    \
        } catch (...) {                                                                          \
        }                                                                                        \
        ::dtshim::check(dtshim_ok, "CHECK_THROWS_AS", #expr ", " #__VA_ARGS__, __FILE__, __LINE__, false); \
    } while (0)

#ifdef DOCTEST_CONFIG_IMPLEMENT_WITH_MAIN
int main(int argc, char** argv) {
    std::string suite;
    for (int i = 1; i < argc; ++i)
        if (std::strncmp(argv[i], "--test-suite=", 13) == 0) suite = argv[i] + 13;
    int ran = 0, failed_cases = 0;
    for (const auto& c : ::dtshim::registry()) {
        if (!suite.empty() && suite != c.suite) continue;
        ++ran;
        const int before = ::dtshim::failures();
        try {
            c.fn();
        } catch (const ::dtshim::Abort&) {
        } catch (const std::exception& e) {
            ++::dtshim::failures();
            std::fprintf(stderr, "[%s] %s: unexpected exception: %s\n", c.suite, c.name, e.what());
        } catch (...) {
            ++::dtshim::failures();
            std::fprintf(stderr, "[%s] %s: unexpected exception\n", c.suite, c.name);
        }
        if (::dtshim::failures() != before) {
            ++failed_cases;
            std::fprintf(stderr, "[%s] %s: FAILED\n", c.suite, c.name);
        }
    }
    std::printf("[dtshim] test cases: %d | %d passed | %d failed | assertions: %d | %d failed\n", ran,
                ran - failed_cases, failed_cases, ::dtshim::asserts(), ::dtshim::failures());
    return failed_cases ? 1 : 0;
}
#endif
