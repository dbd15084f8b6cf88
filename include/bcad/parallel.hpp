// Broadcast thread-count knob of the reference (proj/include/bcad/parallel.hpp:
// 15-16, src/parallel.cpp). The reference chunks broadcast cells over OpenMP
// threads; here every broadcast is a CUDA grid sized from the device's SM
// count (csrc/plan.hpp), so the value is recorded and reported but does not
// change how the device runs. Results are bit-identical for any setting, as
// the reference guarantees for any thread count (README.md:59-60).
#pragma once

#include <atomic>

namespace bcad {

namespace detail {
inline std::atomic<int>& broadcast_threads_setting() {
    static std::atomic<int> v{0};
    return v;
}
}  // namespace detail

// 0 = library default, 1 = serial in the reference; accepted and recorded.
inline void set_broadcast_threads(int threads) { detail::broadcast_threads_setting().store(threads < 0 ? 0 : threads); }
inline int broadcast_threads() { return detail::broadcast_threads_setting().load(); }

}  // namespace bcad
