// Minimal doctest-style harness (TEST_CASE / CHECK / REQUIRE /
// CHECK_THROWS_AS) so the C++ drop-in tests read like the reference's own
// doctest suites (proj/tests/*.cpp). One binary per suite; exit code 0 iff
// every check passed.
#pragma once

#include <cmath>
#include <cstdio>
#include <functional>
#include <string>
#include <vector>

namespace mini {

struct Case {
    const char* name;
    std::function<void()> fn;
};

inline std::vector<Case>& cases() {
    static std::vector<Case> c;
    return c;
}
inline int& failures() {
    static int f = 0;
    return f;
}
inline int& checks() {
    static int c = 0;
    return c;
}

struct Register {
    Register(const char* n, std::function<void()> f) { cases().push_back({n, std::move(f)}); }
};

struct RequireFailed {};

inline bool close(double a, double b, double rtol, double atol = 0.0) {
    const double scale = std::fabs(a) > std::fabs(b) ? std::fabs(a) : std::fabs(b);
    return std::fabs(a - b) <= atol + rtol * scale;
}

inline int run_all() {
    int failed_cases = 0;
    for (const Case& c : cases()) {
        const int before = failures();
        try {
            c.fn();
        } catch (const RequireFailed&) {
        } catch (const std::exception& e) {
            std::printf("  [%s] unexpected exception: %s\n", c.name, e.what());
            ++failures();
        }
        const bool ok = failures() == before;
        failed_cases += ok ? 0 : 1;
        std::printf("%s %s\n", ok ? "PASS" : "FAIL", c.name);
    }
    std::printf("%zu cases, %d failed; %d checks, %d failed\n", cases().size(), failed_cases, checks(), failures());
    return failures() == 0 ? 0 : 1;
}

}  // namespace mini

#define MINI_CAT2(a, b) a##b
#define MINI_CAT(a, b) MINI_CAT2(a, b)
#define TEST_CASE(name)                                                            \
    static void MINI_CAT(mini_case_, __LINE__)();                                  \
    static mini::Register MINI_CAT(mini_reg_, __LINE__)(name, &MINI_CAT(mini_case_, __LINE__)); \
    static void MINI_CAT(mini_case_, __LINE__)()

#define CHECK(expr)                                                                        \
    do {                                                                                   \
        ++mini::checks();                                                                  \
        if (!(expr)) {                                                                     \
            ++mini::failures();                                                            \
            std::printf("  %s:%d CHECK(%s) failed\n", __FILE__, __LINE__, #expr);          \
        }                                                                                  \
    } while (0)

#define REQUIRE(expr)                                                                      \
    do {                                                                                   \
        ++mini::checks();                                                                  \
        if (!(expr)) {                                                                     \
            ++mini::failures();                                                            \
            std::printf("  %s:%d REQUIRE(%s) failed\n", __FILE__, __LINE__, #expr);        \
            throw mini::RequireFailed{};                                                   \
        }                                                                                  \
    } while (0)

#define CHECK_THROWS_AS(expr, type)                                                        \
    do {                                                                                   \
        ++mini::checks();                                                                  \
        bool caught_ = false;                                                              \
        try {                                                                              \
            (void)(expr);                                                                  \
        } catch (const type&) {                                                            \
            caught_ = true;                                                                \
        } catch (...) {                                                                    \
        }                                                                                  \
        if (!caught_) {                                                                    \
            ++mini::failures();                                                            \
            std::printf("  %s:%d CHECK_THROWS_AS(%s, %s) failed\n", __FILE__, __LINE__, #expr, #type); \
        }                                                                                  \
    } while (0)

#define MINI_MAIN \
    int main() { return mini::run_all(); }
