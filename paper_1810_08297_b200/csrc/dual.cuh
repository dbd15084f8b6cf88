// Register-resident forward-mode dual numbers for sm_100a.
//
// Device counterpart of bcad::Dual (reference proj/include/bcad/dual.hpp:68-244):
// a primal plus N perturbation coefficients, N fixed at compile time to the
// kernel's input arity so the whole vector lives in registers. One
// differentiation per output cell means every live dual shares one tag, so
// tags (dual.hpp:18-34, 218-226) stay a host-side concept; constants carry
// zero partials, arithmetically identical to the reference's width-0
// constants. Every rule mirrors the reference's operation order so that,
// compiled with --fmad=false (one rounding per source operation, like the
// reference's -ffp-contract=off), only the transcendental ulps differ.
#pragma once

#include <cstdint>
#include <cuda_runtime.h>

#define BCAD_HD __host__ __device__ __forceinline__

namespace bcad_dev {

// ------------------------------------------------------------ error flags
// Status codes (include/bcad_cu.h) raised by dual rules. The reference throws
// at the offending operation (dual.hpp:130, 163, 286, 322, 331, 340); a
// device thread cannot, so the rule records the code in a per-thread shared
// slot that the launching kernel inspects after each cell and turns into the
// first failing flat index (forward.hpp:137-146).
enum DevStatus : uint32_t {
    kDevOk = 0,
    kDevDivisionByZero = 2,
    kDevDomainError = 3,
    kDevNonDifferentiable = 4,
};

constexpr int kMaxThreadsPerCta = 256;
__shared__ uint8_t s_err_flag[kMaxThreadsPerCta];

// Transcendental-evaluation census (the reference's EvalCounters,
// counters.hpp:20-22, bumped by dual.hpp:55-60 and 280-320 for exp, log, sin,
// cos, tanh and sigmoid): the production kernels carry no counting code. When
// the census is armed, each forward / RecomputeReverse pullback launch is
// followed by one census launch that re-runs the body per cell on CountReal
// scalars (census.cuh), which tally into this per-thread slot.
__shared__ uint32_t s_tcount[kMaxThreadsPerCta];

BCAD_HD void raise_status(uint32_t code) {
#ifdef __CUDA_ARCH__
    uint8_t& f = s_err_flag[threadIdx.x];
    if (f == 0) f = uint8_t(code);
#else
    (void)code;
#endif
}

// ------------------------------------------------------------ real math
// Non-fast-math libdevice calls; the two-branch sigmoid never exponentiates
// a positive argument (dual.hpp:38-48).
BCAD_HD float d_exp(float x) { return ::expf(x); }
BCAD_HD double d_exp(double x) { return ::exp(x); }
BCAD_HD float d_log(float x) { return ::logf(x); }
BCAD_HD double d_log(double x) { return ::log(x); }
BCAD_HD float d_sin(float x) { return ::sinf(x); }
BCAD_HD double d_sin(double x) { return ::sin(x); }
BCAD_HD float d_cos(float x) { return ::cosf(x); }
BCAD_HD double d_cos(double x) { return ::cos(x); }
BCAD_HD float d_tanh(float x) { return ::tanhf(x); }
BCAD_HD double d_tanh(double x) { return ::tanh(x); }
BCAD_HD float d_sqrt(float x) { return ::sqrtf(x); }
BCAD_HD double d_sqrt(double x) { return ::sqrt(x); }
BCAD_HD float d_pow(float x, float c) { return ::powf(x, c); }
BCAD_HD double d_pow(double x, double c) { return ::pow(x, c); }
BCAD_HD float d_floor(float x) { return ::floorf(x); }
BCAD_HD double d_floor(double x) { return ::floor(x); }

// Branch-free form of the same arithmetic: x >= 0 gives e = exp(-x) and
// 1 / (1 + e); x < 0 gives e = exp(x) and e / (1 + e) — one exp and one
// correctly rounded division either way, so the result is bit-identical to
// the two-branch source while lanes never diverge.
template <class F>
BCAD_HD F raw_sigmoid(F x) {
    const bool pos = x >= F(0);
    const F e = d_exp(pos ? -x : x);
    return (pos ? F(1) : e) / (F(1) + e);
}

// Real-body primitives (dual.hpp:55-63): what the generic kernel bodies call
// when instantiated on plain reals (the primal-only / broadcast_apply path).
BCAD_HD float sigmoid(float x) { return raw_sigmoid(x); }
BCAD_HD double sigmoid(double x) { return raw_sigmoid(x); }
BCAD_HD float tanh(float x) { return d_tanh(x); }
BCAD_HD double tanh(double x) { return d_tanh(x); }
BCAD_HD float exp(float x) { return d_exp(x); }
BCAD_HD double exp(double x) { return d_exp(x); }
BCAD_HD float log(float x) { return d_log(x); }
BCAD_HD double log(double x) { return d_log(x); }
BCAD_HD float sin(float x) { return d_sin(x); }
BCAD_HD double sin(double x) { return d_sin(x); }
BCAD_HD float cos(float x) { return d_cos(x); }
BCAD_HD double cos(double x) { return d_cos(x); }
BCAD_HD float sqrt(float x) { return d_sqrt(x); }
BCAD_HD double sqrt(double x) { return d_sqrt(x); }
BCAD_HD float abs(float x) { return ::fabsf(x); }
BCAD_HD double abs(double x) { return ::fabs(x); }
// A float base with a double literal exponent is ::pow(double, double) in the
// reference's generic lambdas (bcad::pow<F> cannot deduce mixed types).
BCAD_HD double pow(float x, double c) { return ::pow(double(x), c); }
BCAD_HD double pow(double x, double c) { return ::pow(x, c); }

// ------------------------------------------------------------ duals
// Structural sparsity. Each dual carries `nz`, a bit per partial slot that
// may be nonzero; a seeded input x_j has only bit j. Every rule below skips
// the terms whose operand slot is a structural zero. Because the seeds are
// compile-time constants once the body is inlined, the masks are integer
// constants the compiler folds away: a product of two seeded duals costs two
// multiplies instead of 3N flops. On every finite operand the nonzero
// partials are bit-identical to the reference's dense rule (x + 0 == x and
// x - 0 == x exactly, and the skipped products are of an exact zero); only
// the sign of a zero partial and NaN propagation out of a non-finite primal
// into structurally-zero slots can differ. kDenseDuals = true restores the
// dense evaluation (every slot computed) for A/B checks.
#ifndef BCAD_DENSE_DUALS
#define BCAD_DENSE_DUALS 0
#endif
constexpr bool kDenseDuals = BCAD_DENSE_DUALS != 0;

template <class T, int N>
struct Dual {
    T v;
    T d[N];
    uint32_t nz;

    Dual() = default;
    BCAD_HD Dual(T x) : v(x), nz(kDenseDuals ? ~0u : 0u) {  // NOLINT constant embedding (dual.hpp:78)
#pragma unroll
        for (int k = 0; k < N; ++k) d[k] = T(0);
    }
    // x_j + e_j (forward.hpp:121-126)
    BCAD_HD static Dual seeded(T x, int j) {
        Dual r(x);
        r.d[j] = T(1);
        r.nz = kDenseDuals ? ~0u : (1u << j);
        return r;
    }
    BCAD_HD bool has(int k) const { return (nz >> k) & 1u; }
};

template <class T, int N>
BCAD_HD Dual<T, N> operator-(const Dual<T, N>& a) {
    Dual<T, N> r;
    r.v = -a.v;
    r.nz = a.nz;
#pragma unroll
    for (int k = 0; k < N; ++k) r.d[k] = a.has(k) ? -a.d[k] : T(0);
    return r;
}
template <class T, int N>
BCAD_HD Dual<T, N> operator+(const Dual<T, N>& a, const Dual<T, N>& b) {  // dual.hpp:107-112
    Dual<T, N> r;
    r.v = a.v + b.v;
    r.nz = a.nz | b.nz;
#pragma unroll
    for (int k = 0; k < N; ++k)
        r.d[k] = a.has(k) && b.has(k) ? a.d[k] + b.d[k] : a.has(k) ? a.d[k] : b.has(k) ? b.d[k] : T(0);
    return r;
}
template <class T, int N>
BCAD_HD Dual<T, N> operator-(const Dual<T, N>& a, const Dual<T, N>& b) {  // dual.hpp:114-119
    Dual<T, N> r;
    r.v = a.v - b.v;
    r.nz = a.nz | b.nz;
#pragma unroll
    for (int k = 0; k < N; ++k)
        r.d[k] = a.has(k) && b.has(k) ? a.d[k] - b.d[k] : a.has(k) ? a.d[k] : b.has(k) ? -b.d[k] : T(0);
    return r;
}
template <class T, int N>
BCAD_HD Dual<T, N> operator*(const Dual<T, N>& a, const Dual<T, N>& b) {  // dual.hpp:121-127
    Dual<T, N> r;
    r.v = a.v * b.v;
    r.nz = a.nz | b.nz;
#pragma unroll
    for (int k = 0; k < N; ++k)
        r.d[k] = a.has(k) && b.has(k) ? a.d[k] * b.v + a.v * b.d[k]
                 : a.has(k)            ? a.d[k] * b.v
                 : b.has(k)            ? a.v * b.d[k]
                                       : T(0);
    return r;
}
template <class T, int N>
BCAD_HD Dual<T, N> operator/(const Dual<T, N>& a, const Dual<T, N>& b) {  // dual.hpp:129-137
    if (b.v == T(0)) raise_status(kDevDivisionByZero);
    Dual<T, N> r;
    r.v = a.v / b.v;
    r.nz = a.nz | b.nz;
    const T denom = b.v * b.v;
#pragma unroll
    for (int k = 0; k < N; ++k)
        r.d[k] = a.has(k) && b.has(k) ? (a.d[k] * b.v - a.v * b.d[k]) / denom
                 : a.has(k)            ? (a.d[k] * b.v) / denom
                 : b.has(k)            ? (-(a.v * b.d[k])) / denom
                                       : T(0);
    return r;
}

// Scalar forms (dual.hpp:139-166, 229-240).
template <class T, int N>
BCAD_HD Dual<T, N> shifted(const Dual<T, N>& a, T s) {
    Dual<T, N> r = a;
    r.v = a.v + s;
    return r;
}
template <class T, int N>
BCAD_HD Dual<T, N> scaled(const Dual<T, N>& a, T s) {
    Dual<T, N> r;
    r.v = a.v * s;
    r.nz = a.nz;
#pragma unroll
    for (int k = 0; k < N; ++k) r.d[k] = a.has(k) ? a.d[k] * s : T(0);
    return r;
}
template <class T, int N> BCAD_HD Dual<T, N> operator+(const Dual<T, N>& a, double s) { return shifted(a, T(s)); }
template <class T, int N> BCAD_HD Dual<T, N> operator+(double s, const Dual<T, N>& a) { return shifted(a, T(s)); }
template <class T, int N> BCAD_HD Dual<T, N> operator-(const Dual<T, N>& a, double s) { return shifted(a, -T(s)); }
template <class T, int N> BCAD_HD Dual<T, N> operator-(double s, const Dual<T, N>& a) { return shifted(-a, T(s)); }
template <class T, int N> BCAD_HD Dual<T, N> operator*(const Dual<T, N>& a, double s) { return scaled(a, T(s)); }
template <class T, int N> BCAD_HD Dual<T, N> operator*(double s, const Dual<T, N>& a) { return scaled(a, T(s)); }
template <class T, int N>
BCAD_HD Dual<T, N> operator/(const Dual<T, N>& a, double s) {
    const T rs = T(s);
    if (rs == T(0)) raise_status(kDevDivisionByZero);
    return scaled(a, T(1) / rs);
}
template <class T, int N>
BCAD_HD Dual<T, N> operator/(double s, const Dual<T, N>& b) {
    if (b.v == T(0)) raise_status(kDevDivisionByZero);
    const T rs = T(s);
    Dual<T, N> r;
    r.v = rs / b.v;
    r.nz = b.nz;
    const T scale = -rs / (b.v * b.v);
#pragma unroll
    for (int k = 0; k < N; ++k) r.d[k] = b.has(k) ? scale * b.d[k] : T(0);
    return r;
}

// Comparisons read primals only: the differentiated kernel takes the branch
// the undifferentiated one would (dual.hpp:175-208).
template <class T, int N> BCAD_HD bool operator<(const Dual<T, N>& a, const Dual<T, N>& b) { return a.v < b.v; }
template <class T, int N> BCAD_HD bool operator>(const Dual<T, N>& a, const Dual<T, N>& b) { return a.v > b.v; }
template <class T, int N> BCAD_HD bool operator<=(const Dual<T, N>& a, const Dual<T, N>& b) { return a.v <= b.v; }
template <class T, int N> BCAD_HD bool operator>=(const Dual<T, N>& a, const Dual<T, N>& b) { return a.v >= b.v; }
template <class T, int N> BCAD_HD bool operator==(const Dual<T, N>& a, const Dual<T, N>& b) { return a.v == b.v; }
template <class T, int N> BCAD_HD bool operator!=(const Dual<T, N>& a, const Dual<T, N>& b) { return a.v != b.v; }
template <class T, int N> BCAD_HD bool operator<(const Dual<T, N>& a, double s) { return a.v < T(s); }
template <class T, int N> BCAD_HD bool operator>(const Dual<T, N>& a, double s) { return a.v > T(s); }
template <class T, int N> BCAD_HD bool operator<=(const Dual<T, N>& a, double s) { return a.v <= T(s); }
template <class T, int N> BCAD_HD bool operator>=(const Dual<T, N>& a, double s) { return a.v >= T(s); }
template <class T, int N> BCAD_HD bool operator==(const Dual<T, N>& a, double s) { return a.v == T(s); }
template <class T, int N> BCAD_HD bool operator!=(const Dual<T, N>& a, double s) { return a.v != T(s); }

// f(x + y e) = f(x) + f'(x) y e, coefficient-wise (dual.hpp:211-215).
template <class T, int N>
BCAD_HD Dual<T, N> chain(const Dual<T, N>& a, T p, T scale) {
    Dual<T, N> r;
    r.v = p;
    r.nz = a.nz;
#pragma unroll
    for (int k = 0; k < N; ++k) r.d[k] = a.has(k) ? scale * a.d[k] : T(0);
    return r;
}

// Unary rules (dual.hpp:280-342).
template <class T, int N> BCAD_HD Dual<T, N> exp(const Dual<T, N>& a) {
    const T p = d_exp(a.v);
    return chain(a, p, p);
}
template <class T, int N> BCAD_HD Dual<T, N> log(const Dual<T, N>& a) {
    if (!(a.v > T(0))) raise_status(kDevDomainError);
    return chain(a, d_log(a.v), T(1) / a.v);
}
template <class T, int N> BCAD_HD Dual<T, N> sin(const Dual<T, N>& a) {
    return chain(a, d_sin(a.v), d_cos(a.v));
}
template <class T, int N> BCAD_HD Dual<T, N> cos(const Dual<T, N>& a) {
    return chain(a, d_cos(a.v), -d_sin(a.v));
}
template <class T, int N> BCAD_HD Dual<T, N> tanh(const Dual<T, N>& a) {
    const T t = d_tanh(a.v);
    return chain(a, t, T(1) - t * t);
}
template <class T, int N> BCAD_HD Dual<T, N> sigmoid(const Dual<T, N>& a) {
    const T s = raw_sigmoid(a.v);
    return chain(a, s, s * (T(1) - s));
}
template <class T, int N> BCAD_HD Dual<T, N> sqrt(const Dual<T, N>& a) {
    if (a.v < T(0)) raise_status(kDevDomainError);
    const T s = d_sqrt(a.v);
    return chain(a, s, T(1) / (T(2) * s));
}
template <class T, int N> BCAD_HD Dual<T, N> abs(const Dual<T, N>& a) {
    if (a.v == T(0)) raise_status(kDevNonDifferentiable);
    return a.v > T(0) ? a : -a;
}
template <class T, int N> BCAD_HD Dual<T, N> pow(const Dual<T, N>& a, double exponent) {
    const T c = T(exponent);
    if (a.v < T(0) && c != d_floor(c)) raise_status(kDevDomainError);
    const T p = d_pow(a.v, c);
    return chain(a, p, c * d_pow(a.v, c - T(1)));
}

// Scalar selector used by kernel bodies that need the arithmetic type.
template <class S> struct scalar_of { using type = S; };
template <class T, int N> struct scalar_of<Dual<T, N>> { using type = T; };

// ------------------------------------------------------- lane-vector duals
// VDual<T, N, V>: the V cells one thread owns (its 128-bit vector), evaluated
// together. Every rule is the Dual rule applied lane by lane, in the same
// operation order, so each lane's result is bit-identical to evaluating that
// cell alone. The point is control flow: a body's branch is taken ONCE for
// all V lanes and their arithmetic interleaves (ILP V instead of V serial
// branch regions). Comparisons read lane 0, so a VDual evaluation is only
// valid when every branch predicate of the body depends on arguments that
// are uniform across the V lanes (ROW / SCALAR stride class). The kernels use
// it only under such a signature (Body::kPredicateArgs).
template <class T, int N, int V>
struct VDual {
    T v[V];
    T d[N][V];
    uint32_t nz;

    VDual() = default;
    BCAD_HD VDual(T x) : nz(kDenseDuals ? ~0u : 0u) {  // NOLINT constant embedding
#pragma unroll
        for (int l = 0; l < V; ++l) {
            v[l] = x;
#pragma unroll
            for (int k = 0; k < N; ++k) d[k][l] = T(0);
        }
    }
    BCAD_HD bool has(int k) const { return (nz >> k) & 1u; }
};

#define BCAD_VLANES _Pragma("unroll") for (int l = 0; l < V; ++l)

template <class T, int N, int V>
BCAD_HD VDual<T, N, V> operator-(const VDual<T, N, V>& a) {
    VDual<T, N, V> r;
    r.nz = a.nz;
    BCAD_VLANES {
        r.v[l] = -a.v[l];
#pragma unroll
        for (int k = 0; k < N; ++k) r.d[k][l] = a.has(k) ? -a.d[k][l] : T(0);
    }
    return r;
}
template <class T, int N, int V>
BCAD_HD VDual<T, N, V> operator+(const VDual<T, N, V>& a, const VDual<T, N, V>& b) {
    VDual<T, N, V> r;
    r.nz = a.nz | b.nz;
    BCAD_VLANES {
        r.v[l] = a.v[l] + b.v[l];
#pragma unroll
        for (int k = 0; k < N; ++k)
            r.d[k][l] = a.has(k) && b.has(k) ? a.d[k][l] + b.d[k][l] : a.has(k) ? a.d[k][l] : b.has(k) ? b.d[k][l] : T(0);
    }
    return r;
}
template <class T, int N, int V>
BCAD_HD VDual<T, N, V> operator-(const VDual<T, N, V>& a, const VDual<T, N, V>& b) {
    VDual<T, N, V> r;
    r.nz = a.nz | b.nz;
    BCAD_VLANES {
        r.v[l] = a.v[l] - b.v[l];
#pragma unroll
        for (int k = 0; k < N; ++k)
            r.d[k][l] = a.has(k) && b.has(k) ? a.d[k][l] - b.d[k][l] : a.has(k) ? a.d[k][l] : b.has(k) ? -b.d[k][l] : T(0);
    }
    return r;
}
template <class T, int N, int V>
BCAD_HD VDual<T, N, V> operator*(const VDual<T, N, V>& a, const VDual<T, N, V>& b) {
    VDual<T, N, V> r;
    r.nz = a.nz | b.nz;
    BCAD_VLANES {
        r.v[l] = a.v[l] * b.v[l];
#pragma unroll
        for (int k = 0; k < N; ++k)
            r.d[k][l] = a.has(k) && b.has(k) ? a.d[k][l] * b.v[l] + a.v[l] * b.d[k][l]
                        : a.has(k)            ? a.d[k][l] * b.v[l]
                        : b.has(k)            ? a.v[l] * b.d[k][l]
                                              : T(0);
    }
    return r;
}
template <class T, int N, int V>
BCAD_HD VDual<T, N, V> operator/(const VDual<T, N, V>& a, const VDual<T, N, V>& b) {
    VDual<T, N, V> r;
    r.nz = a.nz | b.nz;
    BCAD_VLANES {
        if (b.v[l] == T(0)) raise_status(kDevDivisionByZero);
        r.v[l] = a.v[l] / b.v[l];
        const T denom = b.v[l] * b.v[l];
#pragma unroll
        for (int k = 0; k < N; ++k)
            r.d[k][l] = a.has(k) && b.has(k) ? (a.d[k][l] * b.v[l] - a.v[l] * b.d[k][l]) / denom
                        : a.has(k)            ? (a.d[k][l] * b.v[l]) / denom
                        : b.has(k)            ? (-(a.v[l] * b.d[k][l])) / denom
                                              : T(0);
    }
    return r;
}
template <class T, int N, int V>
BCAD_HD VDual<T, N, V> shifted(const VDual<T, N, V>& a, T s) {
    VDual<T, N, V> r = a;
    BCAD_VLANES r.v[l] = a.v[l] + s;
    return r;
}
template <class T, int N, int V>
BCAD_HD VDual<T, N, V> scaled(const VDual<T, N, V>& a, T s) {
    VDual<T, N, V> r;
    r.nz = a.nz;
    BCAD_VLANES {
        r.v[l] = a.v[l] * s;
#pragma unroll
        for (int k = 0; k < N; ++k) r.d[k][l] = a.has(k) ? a.d[k][l] * s : T(0);
    }
    return r;
}
template <class T, int N, int V> BCAD_HD VDual<T, N, V> operator+(const VDual<T, N, V>& a, double s) { return shifted(a, T(s)); }
template <class T, int N, int V> BCAD_HD VDual<T, N, V> operator+(double s, const VDual<T, N, V>& a) { return shifted(a, T(s)); }
template <class T, int N, int V> BCAD_HD VDual<T, N, V> operator-(const VDual<T, N, V>& a, double s) { return shifted(a, -T(s)); }
template <class T, int N, int V> BCAD_HD VDual<T, N, V> operator-(double s, const VDual<T, N, V>& a) { return shifted(-a, T(s)); }
template <class T, int N, int V> BCAD_HD VDual<T, N, V> operator*(const VDual<T, N, V>& a, double s) { return scaled(a, T(s)); }
template <class T, int N, int V> BCAD_HD VDual<T, N, V> operator*(double s, const VDual<T, N, V>& a) { return scaled(a, T(s)); }
template <class T, int N, int V>
BCAD_HD VDual<T, N, V> operator/(const VDual<T, N, V>& a, double s) {
    const T rs = T(s);
    if (rs == T(0)) raise_status(kDevDivisionByZero);
    return scaled(a, T(1) / rs);
}
template <class T, int N, int V>
BCAD_HD VDual<T, N, V> operator/(double s, const VDual<T, N, V>& b) {
    VDual<T, N, V> r;
    r.nz = b.nz;
    const T rs = T(s);
    BCAD_VLANES {
        if (b.v[l] == T(0)) raise_status(kDevDivisionByZero);
        r.v[l] = rs / b.v[l];
        const T scale = -rs / (b.v[l] * b.v[l]);
#pragma unroll
        for (int k = 0; k < N; ++k) r.d[k][l] = b.has(k) ? scale * b.d[k][l] : T(0);
    }
    return r;
}
// Lane-0 comparisons (uniform predicates only; see above).
template <class T, int N, int V> BCAD_HD bool operator<(const VDual<T, N, V>& a, double s) { return a.v[0] < T(s); }
template <class T, int N, int V> BCAD_HD bool operator>(const VDual<T, N, V>& a, double s) { return a.v[0] > T(s); }
template <class T, int N, int V> BCAD_HD bool operator<=(const VDual<T, N, V>& a, double s) { return a.v[0] <= T(s); }
template <class T, int N, int V> BCAD_HD bool operator>=(const VDual<T, N, V>& a, double s) { return a.v[0] >= T(s); }
template <class T, int N, int V> BCAD_HD bool operator==(const VDual<T, N, V>& a, double s) { return a.v[0] == T(s); }
template <class T, int N, int V> BCAD_HD bool operator!=(const VDual<T, N, V>& a, double s) { return a.v[0] != T(s); }

template <class T, int N, int V, class F>
BCAD_HD VDual<T, N, V> vchain(const VDual<T, N, V>& a, F&& prim_and_scale) {
    VDual<T, N, V> r;
    r.nz = a.nz;
    BCAD_VLANES {
        T p, scale;
        prim_and_scale(a.v[l], p, scale);
        r.v[l] = p;
#pragma unroll
        for (int k = 0; k < N; ++k) r.d[k][l] = a.has(k) ? scale * a.d[k][l] : T(0);
    }
    return r;
}
template <class T, int N, int V> BCAD_HD VDual<T, N, V> exp(const VDual<T, N, V>& a) {
    return vchain(a, [](T x, T& p, T& s) { p = d_exp(x); s = p; });
}
template <class T, int N, int V> BCAD_HD VDual<T, N, V> log(const VDual<T, N, V>& a) {
    return vchain(a, [](T x, T& p, T& s) {
        if (!(x > T(0))) raise_status(kDevDomainError);
        p = d_log(x);
        s = T(1) / x;
    });
}
template <class T, int N, int V> BCAD_HD VDual<T, N, V> sin(const VDual<T, N, V>& a) {
    return vchain(a, [](T x, T& p, T& s) { p = d_sin(x); s = d_cos(x); });
}
template <class T, int N, int V> BCAD_HD VDual<T, N, V> cos(const VDual<T, N, V>& a) {
    return vchain(a, [](T x, T& p, T& s) { p = d_cos(x); s = -d_sin(x); });
}
template <class T, int N, int V> BCAD_HD VDual<T, N, V> tanh(const VDual<T, N, V>& a) {
    return vchain(a, [](T x, T& p, T& s) { p = d_tanh(x); s = T(1) - p * p; });
}
template <class T, int N, int V> BCAD_HD VDual<T, N, V> sigmoid(const VDual<T, N, V>& a) {
    return vchain(a, [](T x, T& p, T& s) { p = raw_sigmoid(x); s = p * (T(1) - p); });
}
template <class T, int N, int V> BCAD_HD VDual<T, N, V> sqrt(const VDual<T, N, V>& a) {
    return vchain(a, [](T x, T& p, T& s) {
        if (x < T(0)) raise_status(kDevDomainError);
        p = d_sqrt(x);
        s = T(1) / (T(2) * p);
    });
}
template <class T, int N, int V> BCAD_HD VDual<T, N, V> pow(const VDual<T, N, V>& a, double exponent) {
    const T c = T(exponent);
    return vchain(a, [c](T x, T& p, T& s) {
        if (x < T(0) && c != d_floor(c)) raise_status(kDevDomainError);
        p = d_pow(x, c);
        s = c * d_pow(x, c - T(1));
    });
}
template <class T, int N, int V> BCAD_HD VDual<T, N, V> abs(const VDual<T, N, V>& a) {
    VDual<T, N, V> r;
    r.nz = a.nz;
    BCAD_VLANES {
        if (a.v[l] == T(0)) raise_status(kDevNonDifferentiable);
        const bool pos = a.v[l] > T(0);
        r.v[l] = pos ? a.v[l] : -a.v[l];
#pragma unroll
        for (int k = 0; k < N; ++k) r.d[k][l] = a.has(k) ? (pos ? a.d[k][l] : -a.d[k][l]) : T(0);
    }
    return r;
}
#undef BCAD_VLANES


}  // namespace bcad_dev
