// Test infrastructure (never linked into the product). A minimal stand-in
// for doctest 2.x — the reference's test framework, named by its suites
// (proj/tests/*.cpp `#include "doctest.h"`) but not vendored — written for
// this repo so the reference's OWN test suites compile unchanged against the
// reference's own headers (oracle/Makefile target `ref-suites`). Passing them
// here pins oracle/_ref, which in turn pins the CPU restatement and the
// golden fixtures.
//
// Covers the macro surface those suites use: TEST_CASE, CHECK,
// CHECK_MESSAGE, CHECK_NOTHROW, CHECK_THROWS_AS, REQUIRE, FAIL and
// doctest::Approx (with .epsilon()), plus DOCTEST_CONFIG_IMPLEMENT_WITH_MAIN.
#pragma once

#include <algorithm>
#include <cmath>
#include <cstdio>
#include <exception>
#include <limits>
#include <sstream>
#include <string>
#include <vector>

namespace doctest {

class Approx {
public:
    Approx(double v) : value_(v) {}  // NOLINT: implicit like doctest's
    Approx& epsilon(double e) {
        eps_ = e;
        return *this;
    }
    Approx& scale(double s) {
        scale_ = s;
        return *this;
    }
    // doctest's comparison: |lhs - v| < eps * (scale + max(|lhs|, |v|))
    friend bool operator==(double lhs, const Approx& a) {
        return std::fabs(lhs - a.value_) < a.eps_ * (a.scale_ + std::max(std::fabs(lhs), std::fabs(a.value_)));
    }
    friend bool operator==(const Approx& a, double rhs) { return rhs == a; }
    friend bool operator!=(double lhs, const Approx& a) { return !(lhs == a); }
    friend bool operator!=(const Approx& a, double rhs) { return !(rhs == a); }

private:
    double value_;
    double eps_ = static_cast<double>(std::numeric_limits<float>::epsilon()) * 100;
    double scale_ = 1.0;
};

namespace detail {

struct Case {
    const char* name;
    void (*fn)();
    const char* file;
    int line;
};
inline std::vector<Case>& cases() {
    static std::vector<Case> c;
    return c;
}
struct Counters {
    long checks = 0, failed_checks = 0;
    bool case_failed = false;
};
inline Counters& counters() {
    static Counters c;
    return c;
}
struct Register {
    Register(const char* name, void (*fn)(), const char* file, int line) { cases().push_back({name, fn, file, line}); }
};
struct Abort {};  // REQUIRE / FAIL end the current test case

inline void report(bool ok, const std::string& what, const char* file, int line) {
    Counters& c = counters();
    ++c.checks;
    if (ok) return;
    ++c.failed_checks;
    c.case_failed = true;
    std::fprintf(stderr, "%s:%d: ERROR: %s\n", file, line, what.c_str());
}

// doctest's -tce / --test-case-exclude=<filters>: comma-separated names,
// '*' matching any run of characters.
inline bool glob_match(const char* p, const char* s) {
    if (*p == 0) return *s == 0;
    if (*p == '*') return glob_match(p + 1, s) || (*s && glob_match(p, s + 1));
    return *s == *p && glob_match(p + 1, s + 1);
}
inline std::vector<std::string>& excluded() {
    static std::vector<std::string> v;
    return v;
}
inline void parse_args(int argc, char** argv) {
    for (int a = 1; a < argc; ++a) {
        std::string arg = argv[a];
        for (const char* pre : {"-tce=", "--test-case-exclude="}) {
            const std::string p = pre;
            if (arg.rfind(p, 0) != 0) continue;
            std::string rest = arg.substr(p.size());
            size_t pos;
            while ((pos = rest.find(',')) != std::string::npos) {
                excluded().push_back(rest.substr(0, pos));
                rest = rest.substr(pos + 1);
            }
            if (!rest.empty()) excluded().push_back(rest);
        }
    }
}

inline int run_all() {
    int passed = 0, failed = 0, skipped = 0;
    for (const Case& tc : cases()) {
        bool skip = false;
        for (const std::string& f : excluded()) skip = skip || glob_match(f.c_str(), tc.name);
        if (skip) {
            ++skipped;
            std::printf("[doctest-shim] excluded: %s\n", tc.name);
            continue;
        }
        counters().case_failed = false;
        try {
            tc.fn();
        } catch (const Abort&) {
        } catch (const std::exception& e) {
            report(false, std::string("test case threw: ") + e.what(), tc.file, tc.line);
        } catch (...) {
            report(false, "test case threw a non-std exception", tc.file, tc.line);
        }
        if (counters().case_failed) {
            ++failed;
            std::fprintf(stderr, "  in TEST_CASE(\"%s\")\n", tc.name);
        } else {
            ++passed;
        }
    }
    std::printf("[doctest-shim] test cases: %d | %d passed | %d failed | %d skipped\n", passed + failed, passed, failed,
                skipped);
    std::printf("[doctest-shim] assertions: %ld | %ld passed | %ld failed\n", counters().checks,
                counters().checks - counters().failed_checks, counters().failed_checks);
    return failed == 0 ? 0 : 1;
}

}  // namespace detail
}  // namespace doctest

#define DOCTEST_SHIM_CAT_(a, b) a##b
#define DOCTEST_SHIM_CAT(a, b) DOCTEST_SHIM_CAT_(a, b)
#define DOCTEST_SHIM_TC(f, name)                                                                      \
    static void f();                                                                                  \
    static const ::doctest::detail::Register DOCTEST_SHIM_CAT(f, _reg)(name, &f, __FILE__, __LINE__); \
    static void f()
#define TEST_CASE(name) DOCTEST_SHIM_TC(DOCTEST_SHIM_CAT(doctest_shim_tc_, __COUNTER__), name)

#define CHECK(...) ::doctest::detail::report(static_cast<bool>(__VA_ARGS__), "CHECK( " #__VA_ARGS__ " )", __FILE__, __LINE__)
// the message is a stream expression (`a << " at " << x`), expanded textually as doctest does
#define CHECK_MESSAGE(cond, ...)                                                                     \
    do {                                                                                             \
        std::ostringstream doctest_shim_os_;                                                         \
        doctest_shim_os_ << "CHECK_MESSAGE( " #cond " ) with message: " << __VA_ARGS__;              \
        ::doctest::detail::report(static_cast<bool>(cond), doctest_shim_os_.str(), __FILE__, __LINE__); \
    } while (0)
#define REQUIRE(...)                                                                                         \
    do {                                                                                                     \
        const bool doctest_shim_ok_ = static_cast<bool>(__VA_ARGS__);                                       \
        ::doctest::detail::report(doctest_shim_ok_, "REQUIRE( " #__VA_ARGS__ " )", __FILE__, __LINE__);     \
        if (!doctest_shim_ok_) throw ::doctest::detail::Abort{};                                            \
    } while (0)
#define FAIL(msg)                                                                                   \
    do {                                                                                            \
        std::ostringstream doctest_shim_os_;                                                        \
        doctest_shim_os_ << "FAIL: " << msg;                                                        \
        ::doctest::detail::report(false, doctest_shim_os_.str(), __FILE__, __LINE__);               \
        throw ::doctest::detail::Abort{};                                                           \
    } while (0)
#define CHECK_NOTHROW(...)                                                                          \
    do {                                                                                            \
        bool doctest_shim_ok_ = true;                                                               \
        try {                                                                                       \
            __VA_ARGS__;                                                                            \
        } catch (...) {                                                                             \
            doctest_shim_ok_ = false;                                                               \
        }                                                                                           \
        ::doctest::detail::report(doctest_shim_ok_, "CHECK_NOTHROW( " #__VA_ARGS__ " )", __FILE__, __LINE__); \
    } while (0)
#define CHECK_THROWS_AS(expr, ...)                                                                  \
    do {                                                                                            \
        bool doctest_shim_ok_ = false;                                                              \
        try {                                                                                       \
            expr;                                                                                   \
        } catch (const __VA_ARGS__&) {                                                              \
            doctest_shim_ok_ = true;                                                                \
        } catch (...) {                                                                             \
        }                                                                                           \
        ::doctest::detail::report(doctest_shim_ok_, "CHECK_THROWS_AS( " #expr ", " #__VA_ARGS__ " )", __FILE__, \
                                  __LINE__);                                                        \
    } while (0)

#ifdef DOCTEST_CONFIG_IMPLEMENT_WITH_MAIN
int main(int argc, char** argv) {
    ::doctest::detail::parse_args(argc, argv);
    return ::doctest::detail::run_all();
}
#endif
