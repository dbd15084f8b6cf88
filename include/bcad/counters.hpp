// Evaluation counters of the drop-in API (reference proj/include/bcad/
// counters.hpp:10-33, src/counters.cpp).
//
// Element visits are counted like the reference counts them, once per
// broadcast with the output volume (broadcast.hpp:123, forward.hpp:148): each
// device forward, and each RecomputeReverse pullback (which re-derives every
// cell's diagonals), visits every output cell exactly once.
// Transcendental evaluations (exp, log, sin, cos, tanh, sigmoid on reals and
// duals) are counted where they execute: host scalar evaluations
// (BroadcastKernel::eval with a host body, the finite-difference / Jacobian
// oracles) through the counting wrappers of bcad/dual.hpp, and device kernels
// through a census launch that follows each body-evaluating launch and re-runs
// the body per cell on counting scalars (bcad_cu_eval_counters). The device
// census is armed by the first counter_totals() call, so programs that never
// read the counters never pay for it; launches before that first read are not
// counted (the reference's tests read before and after).
#pragma once

#include <cstdint>
#include <memory>
#include <mutex>
#include <vector>

#include "bcad_cu.h"

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

namespace detail {
inline int& count_pause_depth() {
    static thread_local int d = 0;
    return d;
}
}  // namespace detail

inline void count_transcendental(std::uint64_t n = 1) {
    if (detail::count_pause_depth() == 0) detail::local_counters().transcendental_evals += n;
}
inline void count_element_visits(std::uint64_t n) {
    if (detail::count_pause_depth() == 0) detail::local_counters().kernel_element_visits += n;
}

// Pauses both censuses on this thread (host wrappers and the device launches
// this thread makes): the library's own probe evaluations, which the
// reference never performs, stay out of the totals.
class CountPause {
public:
    CountPause() {
        ++detail::count_pause_depth();
        bcad_cu_count_pause(1);
    }
    ~CountPause() {
        bcad_cu_count_pause(0);
        --detail::count_pause_depth();
    }
    CountPause(const CountPause&) = delete;
    CountPause& operator=(const CountPause&) = delete;
};

inline EvalCounters counter_totals() {
    unsigned long long dev = 0;  // the device census (arms it on first use; synchronises)
    const bool have_dev = bcad_cu_eval_counters(&dev) == BCAD_CU_OK;
    detail::CounterRegistry& r = detail::counter_registry();
    std::lock_guard<std::mutex> lock(r.mu);
    EvalCounters t;
    for (const auto& s : r.slots) {
        t.transcendental_evals += s->transcendental_evals;
        t.kernel_element_visits += s->kernel_element_visits;
    }
    if (have_dev) t.transcendental_evals += dev;
    return t;
}

}  // namespace bcad
