// Registering a user's own kernel body on the device (the B200 replacement for
// the reference's body capture, proj/include/bcad/kernel.hpp:26-43).
//
// The reference type-erases any generic lambda into std::function and runs it
// on the CPU. A body that runs on the GPU must be compiled for sm_100a, so a
// user writes it once as a generic expression in an nvcc translation unit:
//
//   // my_kernels.cu   (nvcc -std=c++20 --fmad=false -gencode arch=compute_100a,code=sm_100a
//   //                  -I<repo>/include -I<repo>/paper_1810_08297_b200/csrc ...)
//   #include "bcad/device_kernel.cuh"
//   BCAD_DEVICE_KERNEL(SoftGate, "soft_gate", 2, 1,
//                      out[0] = sigmoid(in[0]) * tanh(in[1]) + in[0] * in[0])
//
// and links the object with libbcad_cu.so. At load time the macro's static
// object registers the forward (K1) and pullback (K2 / K2r / K2f) launchers,
// instantiated on that body in the user's own object, under "soft_gate"
// (bcad_cu_register_kernel); from then on reference-style host code binds it
// by name exactly like a library body:
//
//   BroadcastKernel<float> k(2, 1, "soft_gate", [](auto in, auto out) {
//       out[0] = sigmoid(in[0]) * tanh(in[1]) + in[0] * in[0]; });   // checked against the device body
//   auto y = mixed_broadcast(tape, k, {x, b}, MixedPolicy::CacheForward);
//
// The expression is instantiated on plain reals (primal-only forward) and on
// the device duals of csrc/dual.cuh (every other path); it may use + - * /,
// comparisons, the ternary operator and sigmoid / tanh / exp / log / sin / cos
// / sqrt / abs / pow(x, c), with `S` naming the scalar type and `in` / `out`
// the argument / result arrays. Names are unique: registering a name that is
// already taken (by the library or another user object) aborts at load with
// the reason, so a body can never silently replace another.
//
// BCAD_DEVICE_KERNEL bodies are treated as possibly raising (domain errors of
// log / division / sqrt / abs / pow are detected and reported with the output
// index, which costs a stream synchronisation per forward);
// BCAD_DEVICE_KERNEL_NOTHROW declares a body free of those operations (no
// check, fully asynchronous, graph-capturable). Both evaluate every cell on
// its own (no lane-vector evaluation across cells), which is correct for any
// branch structure; BCAD_DEVICE_KERNEL_NOTHROW_P declares which arguments
// the branches read, enabling the lane-vector evaluation (below).
#pragma once

#include <cstdio>
#include <cstdlib>

#if __has_include("launch.cuh")
#include "launch.cuh"
#else
#include "../../paper_1810_08297_b200/csrc/launch.cuh"
#endif

namespace bcad_dev {

// Static registration object: one per BCAD_DEVICE_KERNEL.
template <class Body>
struct DeviceKernelRegistration {
    static bcad_cu_kernel_entry make_entry() {
        // a body declaring its branch arguments (..._P) also gets the layout
        // in which exactly those are (B)-shaped, the lane-vector fast path
        if constexpr (Body::kPredicateArgs != ~0u && Body::kPredicateArgs != 0u)
            return BCAD_ENTRY(Body, bcad_cu_impl::SigAllFull<Body::kIn>,
                              bcad_cu_impl::SigPredRow<Body::kIn, Body::kPredicateArgs>);
        else
            return BCAD_ENTRY(Body, bcad_cu_impl::SigAllFull<Body::kIn>);
    }
    DeviceKernelRegistration() {
        // runtime argument classes, plus the all-full-shape signature for
        // elementwise calls (no per-argument class branches; measured 10-30%
        // faster on the library's wide bodies, csrc/reg_arity.cu)
        static const bcad_cu_kernel_entry entry = make_entry();
        if (bcad_cu_register_kernel(&entry) != BCAD_CU_OK) {
            std::fprintf(stderr, "bcad: cannot register device kernel '%s': %s\n", Body::kName, bcad_cu_last_error());
            std::abort();
        }
    }
};

}  // namespace bcad_dev

#define BCAD_DEVICE_KERNEL_IMPL_(ID, NAME, NIN, NOUT, RAISES, PRED, ...)                        \
    namespace bcad_dev {                                                                       \
    namespace user_bodies {                                                                    \
    struct ID {                                                                                \
        static constexpr const char* kName = NAME;                                             \
        static constexpr int kIn = NIN, kOut = NOUT;                                           \
        static constexpr bool kMayRaise = RAISES;                                              \
        static constexpr uint32_t kPredicateArgs = PRED;                                       \
        static constexpr bool kSelectForm = false;                                             \
        template <class S>                                                                     \
        BCAD_HD static void body(const S* in, S* out) { __VA_ARGS__; }                        \
        template <class S>                                                                     \
        BCAD_HD static void body_select(const S* in, S* out) { __VA_ARGS__; }                 \
    };                                                                                         \
    }                                                                                          \
    }                                                                                          \
    static const ::bcad_dev::DeviceKernelRegistration<::bcad_dev::user_bodies::ID> bcad_user_kernel_##ID;

#define BCAD_DEVICE_KERNEL(ID, NAME, NIN, NOUT, ...) \
    BCAD_DEVICE_KERNEL_IMPL_(ID, NAME, NIN, NOUT, true, ~0u, __VA_ARGS__)
#define BCAD_DEVICE_KERNEL_NOTHROW(ID, NAME, NIN, NOUT, ...) \
    BCAD_DEVICE_KERNEL_IMPL_(ID, NAME, NIN, NOUT, false, ~0u, __VA_ARGS__)
// PRED: bitmask of the arguments the body's comparisons read (0 for a
// branch-free body). When every one of them is constant along the output's
// last axis for a call (broadcast (B)-shaped or scalar), each thread
// evaluates its 4 (fp32) / 2 (fp64) cells as ONE lane-vector dual, taking
// the branch once — the HM-LSTM bodies' fast path. ~0u (the default above)
// is always correct.
#define BCAD_DEVICE_KERNEL_NOTHROW_P(ID, NAME, NIN, NOUT, PRED, ...) \
    BCAD_DEVICE_KERNEL_IMPL_(ID, NAME, NIN, NOUT, false, PRED, __VA_ARGS__)
