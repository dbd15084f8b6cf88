// Portable seeded generator (reference proj/include/bcad/rng.hpp:11-31):
// mt19937_64 with hand-rolled distributions, so inputs generated here are
// bit-identical to the reference's for the same seed.
#pragma once

#include <cstdint>
#include <random>

namespace bcad {

class Rng {
public:
    explicit Rng(std::uint64_t seed) : gen_(seed) {}
    std::uint64_t raw() { return gen_(); }
    double uniform01() { return static_cast<double>(gen_() >> 11) * 0x1.0p-53; }
    double uniform_pm1() { return 2.0 * uniform01() - 1.0; }
    double binary(double p_one = 0.5) { return uniform01() < p_one ? 1.0 : 0.0; }
    std::uint64_t below(std::uint64_t n) { return gen_() % n; }
    // Skip n draws (every distribution above consumes exactly one draw), so a
    // row block of a tensor can be generated without its predecessors.
    void discard(std::uint64_t n) { gen_.discard(n); }

private:
    std::mt19937_64 gen_;
};

// Distinct deterministic stream per (seed, salt) (proj/src/bench.cpp:31-37).
inline std::uint64_t mix_seed(std::uint64_t seed, std::uint64_t salt) {
    std::uint64_t x = seed ^ (salt * 0x9e3779b97f4a7c15ULL);
    x ^= x >> 30;
    x *= 0xbf58476d1ce4e5b9ULL;
    x ^= x >> 27;
    return x;
}

}  // namespace bcad
