// Evaluation counters of the drop-in API (reference proj/include/bcad/
// counters.hpp:10-33, src/counters.cpp).
//
// Element visits are counted like the reference counts them, once per
// broadcast with the output volume (broadcast.hpp:123, forward.hpp:148): each
// device forward, and each RecomputeReverse pullback (which re-derives every
// cell's diagonals), visits every output cell exactly once.
// Transcendental evaluations are counted for HOST scalar evaluations only:
// BroadcastKernel::eval on reals or duals (the finite-difference / Jacobian
// oracles and the body check at kernel construction) calls the counting
// wrappers of bcad/dual.hpp exactly as the reference's bodies do. On the
// device a per-evaluation counter would sit in the hot loop: the device's
// transcendental census is measured with ncu instead
// (smsp__inst_executed_pipe_xu, profiles/r02/census.md).
#pragma once

#include <cstdint>
#include <memory>
#include <mutex>
#include <vector>

namespace bcad {

struct EvalCounters {
    std::uint64_t transcendental_evals = 0;
    std::uint64_t kernel_element_visits = 0;
};

namespace detail {

// Every thread's slot stays registered after the thread exits, so totals
// keep the work of finished threads (as the reference's leaked slots do).
struct CounterRegistry {
    std::mutex mu;
    std::vector<std::unique_ptr<EvalCounters>> slots;
};
inline CounterRegistry& counter_registry() {
    static CounterRegistry* r = new CounterRegistry();  // never destroyed: threads may outlive statics
    return *r;
}
inline EvalCounters& local_counters() {
    thread_local EvalCounters* mine = [] {
        CounterRegistry& r = counter_registry();
        std::lock_guard<std::mutex> lock(r.mu);
        r.slots.push_back(std::make_unique<EvalCounters>());
        return r.slots.back().get();
    }();
    return *mine;
}

}  // namespace detail

inline void count_transcendental(std::uint64_t n = 1) { detail::local_counters().transcendental_evals += n; }
inline void count_element_visits(std::uint64_t n) { detail::local_counters().kernel_element_visits += n; }

inline EvalCounters counter_totals() {
    detail::CounterRegistry& r = detail::counter_registry();
    std::lock_guard<std::mutex> lock(r.mu);
    EvalCounters t;
    for (const auto& s : r.slots) {
        t.transcendental_evals += s->transcendental_evals;
        t.kernel_element_visits += s->kernel_element_visits;
    }
    return t;
}

}  // namespace bcad
