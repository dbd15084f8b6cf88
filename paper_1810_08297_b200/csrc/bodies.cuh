// Device kernel bodies: the registry's named pure scalar functions.
//
// A reference BroadcastKernel holds one generic body instantiated on reals
// and on duals behind std::function (proj/include/bcad/kernel.hpp:21-51);
// std::function cannot cross to the device, so here each body is a
// compile-time functor whose `body<S>` is instantiated on T (primal-only
// path) and on Dual<T, N> (forward / recompute-pullback paths) inside the
// broadcast kernels, and registered under the reference kernel's name.
//
// Sources of the bodies (file:line in /root/reference/proj):
//   hmlstm_update        include/bcad/hmlstm.hpp:49-61
//   hmlstm_update_bias   SURVEY §8(d) config 3/5: cell_update(c, f+bf, i+bi, g+bg, z1, z2)
//   tanh_product_<A>     include/bcad/arity_workload.hpp:12-28
//   identity             include/bcad/kernel.hpp:72-76
//   pool kernels         tests/support/kernel_pool.hpp:19-102
//   mul/gate/square_gate/two  tests/test_mixed.cpp:21-25, 160-163, 197-200, 137-140
//   plus / sig_tanh      tests/test_broadcast.cpp (plus, gate)
//   log/div/sqrt/abs/pow_half/recip/exp  dual.hpp:280-342 error-path probes
#pragma once

#include "dual.cuh"

namespace bcad_dev {

template <class S>
BCAD_HD S reflect_below_half(S x) {  // arity_workload.hpp:12-15
    return x > 0.5 ? x : -x;
}

// Ordered cases; everything that is not UPDATE or COPY flushes, including
// (z1=1, z2=0) (hmlstm.hpp:45-54). The boundary values are exact binaries.
template <class S>
BCAD_HD S cell_update_scalar(S c, S f, S i, S g, S z1, S z2) {
    if (z1 == 0.0 && z2 == 1.0) return sigmoid(f) * c + sigmoid(i) * tanh(g);  // UPDATE
    if (z1 == 0.0 && z2 == 0.0) return c;                                       // COPY
    return sigmoid(i) * tanh(g);                                                // FLUSH
}

// Branch-free form of cell_update_scalar for cells whose boundary bits
// differ across a warp (per-cell z, SURVEY §8(d) config 4 divergence): every
// lane evaluates sigmoid(f), sigmoid(i) and tanh(g) once and the ordered
// cases select among the results, so a warp runs three transcendental
// sequences per cell instead of the five a divergent UPDATE + FLUSH pair
// costs. Per cell the value and every partial are the branchy form's bit for
// bit (the same operations in the same order; the selected one is kept).
template <class S>
BCAD_HD S cell_update_select(S c, S f, S i, S g, S z1, S z2) {
    const S flush = sigmoid(i) * tanh(g);
    const S update = sigmoid(f) * c + flush;
    const bool upd = z1 == 0.0 && z2 == 1.0, cpy = z1 == 0.0 && z2 == 0.0;
    return upd ? update : cpy ? c : flush;
}

// kPredicateArgs: bit j set when argument j feeds a branch predicate of
// the body (a comparison). The lane-vector evaluation (VDual) is used only
// when all of them are uniform across a thread's V cells. kSelectForm: the
// body also provides body_select, a branch-free equivalent used when they
// are not.
#define BCAD_BODY_P(NAME, STR, NIN, NOUT, RAISES, PRED, ...)                 \
    struct NAME {                                                            \
        static constexpr const char* kName = STR;                            \
        static constexpr int kIn = NIN, kOut = NOUT;                         \
        static constexpr bool kMayRaise = RAISES;                            \
        static constexpr uint32_t kPredicateArgs = PRED;                     \
        static constexpr bool kSelectForm = false;                           \
        template <class S>                                                   \
        BCAD_HD static void body(const S* in, S* out) { __VA_ARGS__; }       \
        template <class S>                                                   \
        BCAD_HD static void body_select(const S* in, S* out) { __VA_ARGS__; } \
    };
#define BCAD_BODY(NAME, STR, NIN, NOUT, RAISES, ...) BCAD_BODY_P(NAME, STR, NIN, NOUT, RAISES, 0u, __VA_ARGS__)

struct KHmlstm {  // hmlstm.hpp:56-61
    static constexpr const char* kName = "hmlstm_update";
    static constexpr int kIn = 6, kOut = 1;
    static constexpr bool kMayRaise = false;
    static constexpr uint32_t kPredicateArgs = 0x30u;      // z1, z2
    static constexpr uint32_t kPredicateOnlyArgs = 0x30u;  // ... and nothing else reads them
    static constexpr bool kSelectForm = true;
    template <class S>
    BCAD_HD static void body(const S* in, S* out) {
        out[0] = cell_update_scalar(in[0], in[1], in[2], in[3], in[4], in[5]);
    }
    template <class S>
    BCAD_HD static void body_select(const S* in, S* out) {
        out[0] = cell_update_select(in[0], in[1], in[2], in[3], in[4], in[5]);
    }
};
struct KHmlstmBias {  // cell_update(c, f + bf, i + bi, g + bg, z1, z2), SURVEY §8(d) configs 3/5
    static constexpr const char* kName = "hmlstm_update_bias";
    static constexpr int kIn = 9, kOut = 1;
    static constexpr bool kMayRaise = false;
    static constexpr uint32_t kPredicateArgs = 0x180u;      // z1, z2
    static constexpr uint32_t kPredicateOnlyArgs = 0x180u;  // ... and nothing else reads them
    static constexpr bool kSelectForm = true;
    template <class S>
    BCAD_HD static void body(const S* in, S* out) {
        out[0] = cell_update_scalar(in[0], in[1] + in[4], in[2] + in[5], in[3] + in[6], in[7], in[8]);
    }
    template <class S>
    BCAD_HD static void body_select(const S* in, S* out) {
        out[0] = cell_update_select(in[0], in[1] + in[4], in[2] + in[5], in[3] + in[6], in[7], in[8]);
    }
};
BCAD_BODY(KIdentity, "identity", 1, 1, false, out[0] = in[0])
BCAD_BODY_P(KReflect, "reflect", 1, 1, false, 0x1u, out[0] = reflect_below_half(in[0]))
BCAD_BODY(KTanhSigmoid, "tanh_sigmoid", 1, 1, false, out[0] = tanh(in[0]) * sigmoid(in[0]))
BCAD_BODY(KProduct, "product", 2, 1, false, out[0] = in[0] * in[1])
BCAD_BODY(KMul, "mul", 2, 1, false, out[0] = in[0] * in[1])
BCAD_BODY(KPlus, "plus", 2, 1, false, out[0] = in[0] + in[1])
BCAD_BODY(KGated, "gated", 2, 1, false, out[0] = in[0] + sigmoid(in[1]) * tanh(in[0]))
BCAD_BODY(KProdDiff, "prod_diff", 2, 2, false, out[0] = in[0] * in[1]; out[1] = in[0] - in[1])
BCAD_BODY(KBlend, "blend", 3, 1, false, S w = sigmoid(in[0]); out[0] = w * in[1] + (1.0 - w) * in[2])
BCAD_BODY(KCurl, "curl", 3, 2, false, out[0] = in[0] * in[1] + cos(in[2]); out[1] = in[2] * tanh(in[0]))
BCAD_BODY(KFanout, "fanout", 2, 3, false, out[0] = in[0] + in[1]; out[1] = in[0] * in[1];
          out[2] = sigmoid(in[0]) - tanh(in[1]))
BCAD_BODY(KFiveway, "fiveway", 5, 1, false, out[0] = in[0] * in[1] + in[2] * in[3] * in[4])
BCAD_BODY(KWave, "wave", 3, 1, false, out[0] = sin(in[0]) * exp(-(in[1] * in[1])) + cos(in[2]))
BCAD_BODY(KGate, "gate", 2, 1, false, out[0] = sigmoid(in[0]) * tanh(in[1]) + in[0])
BCAD_BODY(KSigTanh, "sig_tanh", 2, 1, false, out[0] = sigmoid(in[0]) * tanh(in[1]))
BCAD_BODY(KSquareGate, "square_gate", 2, 1, false, out[0] = sigmoid(in[0]) * in[1])
BCAD_BODY(KTwo, "two", 2, 2, false, out[0] = in[0] * in[1]; out[1] = sigmoid(in[0]) + tanh(in[1]))
BCAD_BODY(KLog, "log", 1, 1, true, out[0] = log(in[0]))
BCAD_BODY(KDiv, "div", 2, 1, true, out[0] = in[0] / in[1])
BCAD_BODY(KSqrt, "sqrt", 1, 1, true, out[0] = sqrt(in[0]))
BCAD_BODY(KAbs, "abs", 1, 1, true, out[0] = abs(in[0]))
BCAD_BODY(KPowHalf, "pow_half", 1, 1, true, out[0] = pow(in[0], 0.5))
BCAD_BODY(KRecip, "recip", 1, 1, true, out[0] = 1.0 / in[0])
BCAD_BODY(KExp, "exp", 1, 1, false, out[0] = exp(in[0]))
// Tensor-level primitives of the reverse tape (tape.hpp:84-129, 284-330),
// evaluated with their real bodies: forward values and the exact backward
// element rules of the reference's unfused baseline.
BCAD_BODY(KMinus, "minus", 2, 1, false, out[0] = in[0] - in[1])
BCAD_BODY(KNeg, "neg", 1, 1, false, out[0] = -in[0])
BCAD_BODY(KSigmoid, "sigmoid", 1, 1, false, out[0] = sigmoid(in[0]))
BCAD_BODY(KTanh, "tanh", 1, 1, false, out[0] = tanh(in[0]))
BCAD_BODY_P(KSelect, "select", 3, 1, false, 0x1u, out[0] = in[0] != 0.0 ? in[1] : in[2])
BCAD_BODY(KSigmoidBwd, "sigmoid_bwd", 2, 1, false, out[0] = in[0] * in[1] * (S(1.0) - in[1]))
BCAD_BODY(KTanhBwd, "tanh_bwd", 2, 1, false, out[0] = in[0] * (S(1.0) - in[1] * in[1]))
BCAD_BODY_P(KSelectTrueBwd, "select_true_bwd", 2, 1, false, 0x2u, out[0] = in[1] != 0.0 ? in[0] : S(0.0))
BCAD_BODY_P(KSelectFalseBwd, "select_false_bwd", 2, 1, false, 0x2u, out[0] = in[1] != 0.0 ? S(0.0) : in[0])
#undef BCAD_BODY
#undef BCAD_BODY_P

template <int A>
struct KTanhProduct {  // arity_workload.hpp:19-28
    static constexpr const char* kName =
        A == 1 ? "tanh_product_1" : A == 2 ? "tanh_product_2" : A == 3 ? "tanh_product_3"
      : A == 4 ? "tanh_product_4" : A == 5 ? "tanh_product_5" : A == 8 ? "tanh_product_8"
      : A == 16 ? "tanh_product_16" : A == 18 ? "tanh_product_18" : A == 32 ? "tanh_product_32" : nullptr;
    static_assert(A == 1 || A == 2 || A == 3 || A == 4 || A == 5 || A == 8 || A == 16 || A == 18 || A == 32,
                  "add the arity's name to KTanhProduct::kName");
    static constexpr int kIn = A, kOut = 1;
    static constexpr bool kMayRaise = false;
    static constexpr uint32_t kPredicateArgs = A >= 32 ? ~0u : (1u << A) - 1u;  // reflect_below_half on every arg
    static constexpr bool kSelectForm = false;
    // cells per K1 thread: the product's dual keeps all A partials live, so
    // wide arities evaluate fewer cells at once (register study, paper Fig. 3)
    static constexpr int kMaxVec = A >= 16 ? 1 : A >= 8 ? 2 : 4;
    // K1 rows per thread on large problems, measured with the all-full-shape
    // signature (reg_arity.cu) at 4096^2 fp32 (scripts/lab "arity",
    // "arity32", means; profiles/r02/lab_arity_static.jsonl): A <= 8 best at
    // 2 rows (A4 0.96, A8 0.99 of the copy peak), A = 16 / 18 at 4 (0.93 /
    // 0.92), A = 32 at 16 (0.795; 8 rows 0.787, 32 rows 0.777 — lab "arity32").
    static constexpr int kFwdRows = A >= 32 ? 16 : A >= 16 ? 4 : 2;
    // lab A/B of the K1 register pipeline for wide bodies: 0 = next-row
    // pipeline (default; with the static signature A = 32 runs 0.793 with it
    // against 0.778 without it at >= 3 CTAs per SM); 1 = no pipeline for
    // A >= 32; 2 = no pipeline and >= 3 CTAs per SM for A >= 32
#ifndef BCAD_ARITY_VARIANT
#define BCAD_ARITY_VARIANT 0
#endif
    static constexpr bool kFwdPipeline = !(BCAD_ARITY_VARIANT >= 1 && A >= 32);
    static constexpr int kFwdMinBlocks = (BCAD_ARITY_VARIANT >= 2 && A >= 32) ? 3 : 0;
    template <class S>
    BCAD_HD static void body_select(const S* in, S* out) { body(in, out); }
    template <class S>
    BCAD_HD static void body(const S* in, S* out) {
        S acc = tanh(reflect_below_half(in[0]));
#pragma unroll
        for (int j = 1; j < A; ++j) acc = acc * tanh(reflect_below_half(in[j]));
        out[0] = acc;
    }
};

}  // namespace bcad_dev
