// ORACLE — TEST INFRASTRUCTURE ONLY.
//
// CPU restatement of the reference's mixed-mode broadcast differentiation
// (arXiv 1810.08297, reference library `bcad` under /root/reference/proj).
// Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline /
// `--impl reference` legs may load this library, and only as the checker.
// The product path (paper_1810_08297_b200/, include/) never links it.
//
// Parity pinning: tests/test_oracle.py checks this restatement bit-for-bit
// against oracle/_ref/libbcad_ref.so (the reference headers compiled from
// /root/reference by oracle/Makefile) and against the committed golden
// vectors in tests/golden/ that the same reference build produced.
//
// Built with the reference's numerics flags (-ffp-contract=off,
// proj/src/CMakeLists.txt:9-14): one rounding per source operation.
//
// Restated pieces (reference file:line):
//   * forward-mode duals            proj/include/bcad/dual.hpp:68-244, 280-342
//   * two-branch sigmoid            proj/include/bcad/dual.hpp:38-48
//   * first-axis broadcast shapes   proj/include/bcad/shape.hpp:70-90, 98-111
//   * fused diag-Jacobian forward   proj/include/bcad/forward.hpp:98-150
//   * primal-only broadcast_apply   proj/include/bcad/broadcast.hpp:102-125
//   * backprop_diag + scatter_add   proj/include/bcad/mixed.hpp:27-41,
//                                   proj/include/bcad/broadcast.hpp:174-183, 210-217,
//                                   proj/include/bcad/tape.hpp:179-183
//   * Rng / random_pm1 / binary     proj/include/bcad/rng.hpp:11-31,
//                                   proj/include/bcad/tensor.hpp:71-84
//   * mix_seed                      proj/src/bench.cpp:31-37
//   * kernel bodies                 proj/include/bcad/hmlstm.hpp:49-61,
//                                   proj/include/bcad/arity_workload.hpp:12-28,
//                                   proj/tests/support/kernel_pool.hpp:19-102,
//                                   proj/tests/test_mixed.cpp, test_broadcast.cpp
// On top of the reference's serial fp32/fp64 scatter_add this oracle also
// reports an fp64-accumulated sum of the same rounded terms:
// the comparator for device reductions of fp32 data.

#include <cmath>
#include <cstdint>
#include <cstring>
#include <random>
#include <stdexcept>
#include <string>
#include <vector>

namespace {

// ---------------------------------------------------------------- errors
// Status codes shared with include/bcad_cu.h (bcad_cu_status).
enum Status {
    kOk = 0,
    kTagMismatch = 1,
    kDivisionByZero = 2,
    kDomainError = 3,
    kNonDifferentiable = 4,
    kShapeMismatch = 5,
    kArityMismatch = 6,
    kSeedShapeMismatch = 7,
    kUnknownPrimitive = 8,
    kGeneric = 15,
};

struct OracleError : std::runtime_error {
    int code;
    OracleError(int c, const std::string& m) : std::runtime_error(m), code(c) {}
};

thread_local std::string g_last_error;

// ----------------------------------------------------------------- duals
// Fixed-width restatement of bcad::Dual (dual.hpp:68-244). A single
// differentiation per cell means every live dual shares one tag; constants
// carry zero partials, which is arithmetically what the reference's
// width-0 constant duals contribute (dual.hpp:89, 218-226).
template <class T, int N>
struct Dual {
    T v{};
    T d[N > 0 ? N : 1]{};

    Dual() = default;
    Dual(T x) : v(x) {  // NOLINT constant embedding, dual.hpp:78
        for (int k = 0; k < N; ++k) d[k] = T(0);
    }
};

template <class T, int N>
Dual<T, N> operator-(const Dual<T, N>& a) {
    Dual<T, N> r;
    r.v = -a.v;
    for (int k = 0; k < N; ++k) r.d[k] = -a.d[k];
    return r;
}
template <class T, int N>
Dual<T, N> operator+(const Dual<T, N>& a, const Dual<T, N>& b) {
    Dual<T, N> r;
    r.v = a.v + b.v;
    for (int k = 0; k < N; ++k) r.d[k] = a.d[k] + b.d[k];
    return r;
}
template <class T, int N>
Dual<T, N> operator-(const Dual<T, N>& a, const Dual<T, N>& b) {
    Dual<T, N> r;
    r.v = a.v - b.v;
    for (int k = 0; k < N; ++k) r.d[k] = a.d[k] - b.d[k];
    return r;
}
template <class T, int N>
Dual<T, N> operator*(const Dual<T, N>& a, const Dual<T, N>& b) {
    Dual<T, N> r;
    r.v = a.v * b.v;
    for (int k = 0; k < N; ++k) r.d[k] = a.d[k] * b.v + a.v * b.d[k];
    return r;
}
template <class T, int N>
Dual<T, N> operator/(const Dual<T, N>& a, const Dual<T, N>& b) {
    if (b.v == T(0)) throw OracleError(kDivisionByZero, "dual division by zero primal");
    Dual<T, N> r;
    r.v = a.v / b.v;
    const T denom = b.v * b.v;
    for (int k = 0; k < N; ++k) r.d[k] = (a.d[k] * b.v - a.v * b.d[k]) / denom;
    return r;
}
// Scalar forms: shifted / scaled (dual.hpp:130-166, 229-240).
template <class T, int N>
Dual<T, N> shifted(const Dual<T, N>& a, T s) {
    Dual<T, N> r = a;
    r.v = a.v + s;
    return r;
}
template <class T, int N>
Dual<T, N> scaled(const Dual<T, N>& a, T s) {
    Dual<T, N> r;
    r.v = a.v * s;
    for (int k = 0; k < N; ++k) r.d[k] = a.d[k] * s;
    return r;
}
template <class T, int N> Dual<T, N> operator+(const Dual<T, N>& a, double s) { return shifted(a, T(s)); }
template <class T, int N> Dual<T, N> operator+(double s, const Dual<T, N>& a) { return shifted(a, T(s)); }
template <class T, int N> Dual<T, N> operator-(const Dual<T, N>& a, double s) { return shifted(a, -T(s)); }
template <class T, int N> Dual<T, N> operator-(double s, const Dual<T, N>& a) { return shifted(-a, T(s)); }
template <class T, int N> Dual<T, N> operator*(const Dual<T, N>& a, double s) { return scaled(a, T(s)); }
template <class T, int N> Dual<T, N> operator*(double s, const Dual<T, N>& a) { return scaled(a, T(s)); }
template <class T, int N>
Dual<T, N> operator/(const Dual<T, N>& a, double s) {
    const T rs = T(s);
    if (rs == T(0)) throw OracleError(kDivisionByZero, "dual division by zero scalar");
    return scaled(a, T(1) / rs);
}
template <class T, int N>
Dual<T, N> operator/(double s, const Dual<T, N>& b) {
    if (b.v == T(0)) throw OracleError(kDivisionByZero, "dual division by zero primal");
    const T rs = T(s);
    Dual<T, N> r;
    r.v = rs / b.v;
    const T scale = -rs / (b.v * b.v);
    for (int k = 0; k < N; ++k) r.d[k] = scale * b.d[k];
    return r;
}
// Comparisons act on primals only (dual.hpp:177-208).
template <class T, int N> bool operator>(const Dual<T, N>& a, double s) { return a.v > T(s); }
template <class T, int N> bool operator==(const Dual<T, N>& a, double s) { return a.v == T(s); }

// chain rule f(x + y e) = f(x) + f'(x) y e (dual.hpp:211-215)
template <class T, int N>
Dual<T, N> chain(const Dual<T, N>& a, T p, T scale) {
    Dual<T, N> r;
    r.v = p;
    for (int k = 0; k < N; ++k) r.d[k] = scale * a.d[k];
    return r;
}

// Real-valued primitives (dual.hpp:38-63).
template <class F>
F raw_sigmoid(F x) {
    if (x >= F(0)) {
        const F e = std::exp(-x);
        return F(1) / (F(1) + e);
    }
    const F e = std::exp(x);
    return e / (F(1) + e);
}
inline float sigmoid(float x) { return raw_sigmoid(x); }
inline double sigmoid(double x) { return raw_sigmoid(x); }
inline float tanh(float x) { return std::tanh(x); }
inline double tanh(double x) { return std::tanh(x); }
inline float exp(float x) { return std::exp(x); }
inline double exp(double x) { return std::exp(x); }
inline float log(float x) { return std::log(x); }
inline double log(double x) { return std::log(x); }
inline float sin(float x) { return std::sin(x); }
inline double sin(double x) { return std::sin(x); }
inline float cos(float x) { return std::cos(x); }
inline double cos(double x) { return std::cos(x); }
inline float sqrt(float x) { return std::sqrt(x); }
inline double sqrt(double x) { return std::sqrt(x); }
inline float abs(float x) { return std::fabs(x); }
inline double abs(double x) { return std::fabs(x); }
// A float base with a double literal exponent resolves to ::pow(double,
// double) in the reference's generic lambdas (no bcad::pow<F> deduction).
inline double pow(float x, double c) { return std::pow(double(x), c); }
inline double pow(double x, double c) { return std::pow(x, c); }

// Dual unary rules (dual.hpp:280-342).
template <class T, int N> Dual<T, N> exp(const Dual<T, N>& a) {
    const T p = std::exp(a.v);
    return chain(a, p, p);
}
template <class T, int N> Dual<T, N> log(const Dual<T, N>& a) {
    if (!(a.v > T(0))) throw OracleError(kDomainError, "log requires a positive primal");
    return chain(a, std::log(a.v), T(1) / a.v);
}
template <class T, int N> Dual<T, N> sin(const Dual<T, N>& a) {
    return chain(a, std::sin(a.v), std::cos(a.v));
}
template <class T, int N> Dual<T, N> cos(const Dual<T, N>& a) {
    return chain(a, std::cos(a.v), -std::sin(a.v));
}
template <class T, int N> Dual<T, N> tanh(const Dual<T, N>& a) {
    const T t = std::tanh(a.v);
    return chain(a, t, T(1) - t * t);
}
template <class T, int N> Dual<T, N> sigmoid(const Dual<T, N>& a) {
    const T s = raw_sigmoid(a.v);
    return chain(a, s, s * (T(1) - s));
}
template <class T, int N> Dual<T, N> sqrt(const Dual<T, N>& a) {
    if (a.v < T(0)) throw OracleError(kDomainError, "sqrt requires a non-negative primal");
    const T s = std::sqrt(a.v);
    return chain(a, s, T(1) / (T(2) * s));
}
template <class T, int N> Dual<T, N> abs(const Dual<T, N>& a) {
    if (a.v == T(0)) throw OracleError(kNonDifferentiable, "abs is not differentiable at 0");
    return a.v > T(0) ? a : -a;
}
template <class T, int N> Dual<T, N> pow(const Dual<T, N>& a, double exponent) {
    const T c = T(exponent);
    if (a.v < T(0) && c != std::floor(c))
        throw OracleError(kDomainError, "pow of a negative primal by a non-integer exponent");
    const T p = std::pow(a.v, c);
    return chain(a, p, c * std::pow(a.v, c - T(1)));
}

// ---------------------------------------------------------- kernel bodies
// Each body is written once, generically over the scalar type S, exactly
// as the reference lambdas are (real and dual instantiation of one body).
template <class S> S reflect_below_half(S x) { return x > 0.5 ? x : -x; }  // arity_workload.hpp:12-15

template <class S>
S cell_update_scalar(S c, S f, S i, S g, S z1, S z2) {  // hmlstm.hpp:49-54
    if (z1 == 0.0 && z2 == 1.0) return sigmoid(f) * c + sigmoid(i) * tanh(g);
    if (z1 == 0.0 && z2 == 0.0) return c;
    return sigmoid(i) * tanh(g);
}

template <int A>
struct TanhProduct {  // arity_workload.hpp:19-28
    static constexpr int kIn = A, kOut = 1;
    template <class S> static void body(const S* in, S* out) {
        S acc = tanh(reflect_below_half(in[0]));
        for (int j = 1; j < A; ++j) acc = acc * tanh(reflect_below_half(in[j]));
        out[0] = acc;
    }
};

#define BODY(NAME, NIN, NOUT, ...)                                           \
    struct NAME {                                                            \
        static constexpr int kIn = NIN, kOut = NOUT;                         \
        template <class S> static void body(const S* in, S* out) { __VA_ARGS__; } \
    };

BODY(KIdentity, 1, 1, out[0] = in[0])
BODY(KReflect, 1, 1, out[0] = reflect_below_half(in[0]))
BODY(KTanhSigmoid, 1, 1, out[0] = tanh(in[0]) * sigmoid(in[0]))
BODY(KProduct, 2, 1, out[0] = in[0] * in[1])
BODY(KPlus, 2, 1, out[0] = in[0] + in[1])
BODY(KGated, 2, 1, out[0] = in[0] + sigmoid(in[1]) * tanh(in[0]))
BODY(KProdDiff, 2, 2, out[0] = in[0] * in[1]; out[1] = in[0] - in[1])
BODY(KBlend, 3, 1, S w = sigmoid(in[0]); out[0] = w * in[1] + (1.0 - w) * in[2])
BODY(KCurl, 3, 2, out[0] = in[0] * in[1] + cos(in[2]); out[1] = in[2] * tanh(in[0]))
BODY(KHmlstm, 6, 1, out[0] = cell_update_scalar(in[0], in[1], in[2], in[3], in[4], in[5]))
BODY(KHmlstmBias, 9, 1,
     out[0] = cell_update_scalar(in[0], in[1] + in[4], in[2] + in[5], in[3] + in[6], in[7], in[8]))
BODY(KFanout, 2, 3, out[0] = in[0] + in[1]; out[1] = in[0] * in[1];
     out[2] = sigmoid(in[0]) - tanh(in[1]))
BODY(KFiveway, 5, 1, out[0] = in[0] * in[1] + in[2] * in[3] * in[4])
BODY(KWave, 3, 1, out[0] = sin(in[0]) * exp(-(in[1] * in[1])) + cos(in[2]))
BODY(KGate, 2, 1, out[0] = sigmoid(in[0]) * tanh(in[1]) + in[0])
BODY(KSigTanh, 2, 1, out[0] = sigmoid(in[0]) * tanh(in[1]))
BODY(KSquareGate, 2, 1, out[0] = sigmoid(in[0]) * in[1])
BODY(KTwo, 2, 2, out[0] = in[0] * in[1]; out[1] = sigmoid(in[0]) + tanh(in[1]))
BODY(KLog, 1, 1, out[0] = log(in[0]))
BODY(KDiv, 2, 1, out[0] = in[0] / in[1])
BODY(KSqrt, 1, 1, out[0] = sqrt(in[0]))
BODY(KAbs, 1, 1, out[0] = abs(in[0]))
BODY(KPowHalf, 1, 1, out[0] = pow(in[0], 0.5))
BODY(KRecip, 1, 1, out[0] = 1.0 / in[0])
BODY(KExp, 1, 1, out[0] = exp(in[0]))
#undef BODY

// ------------------------------------------------------------- shapes
constexpr int kMaxRank = 8;
struct OShape {  // layout shared with bcad_cu_shape
    int32_t rank;
    int32_t pad;
    int64_t dims[kMaxRank];
};

int64_t dim_of(const OShape& s, int k) { return k < s.rank ? s.dims[k] : 1; }
int64_t volume(const OShape& s) {
    int64_t v = 1;
    for (int k = 0; k < s.rank; ++k) v *= s.dims[k];
    return v;
}

// First-axis alignment with trailing length-1 padding (shape.hpp:70-90).
OShape broadcast_shape(const OShape* shapes, int n) {
    OShape out{};
    for (int j = 0; j < n; ++j) {
        if (shapes[j].rank < 0 || shapes[j].rank > kMaxRank)
            throw OracleError(kShapeMismatch, "rank out of range");
        for (int k = 0; k < shapes[j].rank; ++k)
            if (shapes[j].dims[k] < 1) throw OracleError(kShapeMismatch, "shape dimensions must be >= 1");
        if (shapes[j].rank > out.rank) out.rank = shapes[j].rank;
    }
    for (int k = 0; k < out.rank; ++k) {
        int64_t len = 1;
        for (int j = 0; j < n; ++j) {
            const int64_t d = dim_of(shapes[j], k);
            if (d == 1) continue;
            if (len == 1) len = d;
            else if (d != len)
                throw OracleError(kShapeMismatch, "broadcast shape mismatch at dim " + std::to_string(k) +
                                                      ": lengths " + std::to_string(len) + " vs " +
                                                      std::to_string(d));
        }
        out.dims[k] = len;
    }
    return out;
}

// virtual_index (shape.hpp:98-111) for a row-major walk of `out`.
struct Walker {
    OShape out;
    std::vector<int64_t> coords;
    explicit Walker(const OShape& o) : out(o), coords(size_t(o.rank), 0) {}
    int64_t index_in(const OShape& arg) const {
        int64_t flat = 0;
        for (int k = 0; k < arg.rank; ++k) {
            const int64_t len = arg.dims[k];
            const int64_t c = coords[size_t(k)] < len - 1 ? coords[size_t(k)] : len - 1;
            flat = flat * len + c;
        }
        return flat;
    }
    void advance() {
        for (int k = out.rank - 1; k >= 0; --k) {
            if (++coords[size_t(k)] < out.dims[k]) return;
            coords[size_t(k)] = 0;
        }
    }
    std::string index_string() const {
        std::string s = "(";
        for (int k = 0; k < out.rank; ++k) {
            if (k) s += ", ";
            s += std::to_string(coords[size_t(k)]);
        }
        return s + ")";
    }
};

// ------------------------------------------------------------- forward
// broadcast_diag_jacobian (forward.hpp:98-150) and broadcast_apply
// (broadcast.hpp:102-125), one visit per output cell in row-major order.
template <class K, class T>
void forward_impl(const void* const* in_v, const OShape* shapes, void* const* primal_v,
                  void* const* partials_v, bool real_body) {
    constexpr int N = K::kIn, M = K::kOut;
    const OShape out = broadcast_shape(shapes, N);
    const int64_t vol = volume(out);
    const T* const* in = reinterpret_cast<const T* const*>(in_v);
    Walker w(out);
    for (int64_t cell = 0; cell < vol; ++cell, w.advance()) {
        if (real_body) {
            T x[N], y[M];
            for (int j = 0; j < N; ++j) x[j] = in[j][w.index_in(shapes[j])];
            K::template body<T>(x, y);
            for (int i = 0; i < M; ++i)
                if (primal_v && primal_v[i]) static_cast<T*>(primal_v[i])[cell] = y[i];
            continue;
        }
        Dual<T, N> x[N], y[M];
        for (int j = 0; j < N; ++j) {  // seed x_j + e_j (forward.hpp:121-126)
            x[j] = Dual<T, N>(in[j][w.index_in(shapes[j])]);
            x[j].d[j] = T(1);
        }
        try {
            K::template body<Dual<T, N>>(x, y);
        } catch (const OracleError& e) {
            throw OracleError(e.code, std::string(e.what()) + " at output index " + w.index_string());
        }
        for (int i = 0; i < M; ++i) {
            if (primal_v && primal_v[i]) static_cast<T*>(primal_v[i])[cell] = y[i].v;
            if (partials_v)
                for (int j = 0; j < N; ++j)
                    if (partials_v[i * N + j]) static_cast<T*>(partials_v[i * N + j])[cell] = y[i].d[j];
        }
    }
}

// ------------------------------------------------------------- pullback
// backprop_diag (mixed.hpp:27-41): for every output i with an adjoint and
// every input j, accumulate_adjoint(ins[j], w_i (.) D_ij) where the zip
// rounds each product (broadcast.hpp:174-183) and scatter_add walks the
// cells serially in row-major order (broadcast.hpp:210-217). First touch of
// a slot zero-initialises it (tape.hpp:179-183); `accumulate[j]` says the
// slot already exists. Repeated pointers model one Var used twice.
template <class T>
void pullback_impl(int n, int m, const OShape* shapes, const void* const* out_adj_v,
                   const void* const* partials_v, void* const* in_adj_v,
                   const unsigned char* accumulate, double* const* acc64) {
    const OShape out = broadcast_shape(shapes, n);
    const int64_t vol = volume(out);
    std::vector<const void*> touched;
    auto first_touch = [&](int j) {
        for (const void* p : touched)
            if (p == in_adj_v[j]) return false;
        touched.push_back(in_adj_v[j]);
        return !(accumulate && accumulate[j]);
    };
    for (int j = 0; j < n; ++j) {
        if (!in_adj_v[j]) continue;
        if (first_touch(j)) {
            T* a = static_cast<T*>(in_adj_v[j]);
            const int64_t v = volume(shapes[j]);
            for (int64_t e = 0; e < v; ++e) a[e] = T(0);
            if (acc64 && acc64[j])
                for (int64_t e = 0; e < v; ++e) acc64[j][e] = 0.0;
        } else if (acc64 && acc64[j]) {
            // Existing slot: the fp64 comparator starts from its current value
            // unless an earlier j in this call already seeded it.
            bool seeded = false;
            for (int k = 0; k < j; ++k)
                if (in_adj_v[k] == in_adj_v[j]) seeded = true;
            if (!seeded) {
                const T* a = static_cast<const T*>(in_adj_v[j]);
                const int64_t v = volume(shapes[j]);
                for (int64_t e = 0; e < v; ++e) acc64[j][e] = double(a[e]);
            }
        }
    }
    for (int i = 0; i < m; ++i) {
        const T* w = static_cast<const T*>(out_adj_v[i]);
        if (!w) continue;
        for (int j = 0; j < n; ++j) {
            if (!in_adj_v[j]) continue;
            const T* D = static_cast<const T*>(partials_v[i * n + j]);
            T* a = static_cast<T*>(in_adj_v[j]);
            double* a64 = acc64 ? acc64[j] : nullptr;
            // Repeated slot: share the first occurrence's fp64 accumulator.
            for (int k = 0; k < j && acc64; ++k)
                if (in_adj_v[k] == in_adj_v[j]) { a64 = acc64[k]; break; }
            Walker wk(out);
            for (int64_t cell = 0; cell < vol; ++cell, wk.advance()) {
                const T term = w[cell] * D[cell];
                const int64_t e = wk.index_in(shapes[j]);
                a[e] += term;
                if (a64) a64[e] += double(term);
            }
        }
    }
    if (acc64)  // mirror the shared accumulator into every repeated j
        for (int j = 0; j < n; ++j)
            for (int k = 0; k < j; ++k)
                if (acc64[j] && acc64[k] && in_adj_v[k] == in_adj_v[j]) {
                    std::memcpy(acc64[j], acc64[k], size_t(volume(shapes[j])) * sizeof(double));
                    break;
                }
}

// ------------------------------------------------------------- registry
struct Entry {
    const char* name;
    int n_in, m_out;
    void (*fwd32)(const void* const*, const OShape*, void* const*, void* const*, bool);
    void (*fwd64)(const void* const*, const OShape*, void* const*, void* const*, bool);
};

#define ENTRY(NAME, K) {NAME, K::kIn, K::kOut, &forward_impl<K, float>, &forward_impl<K, double>}
const Entry kEntries[] = {
    ENTRY("identity", KIdentity),
    ENTRY("reflect", KReflect),
    ENTRY("tanh_sigmoid", KTanhSigmoid),
    ENTRY("product", KProduct),
    ENTRY("mul", KProduct),
    ENTRY("plus", KPlus),
    ENTRY("gated", KGated),
    ENTRY("prod_diff", KProdDiff),
    ENTRY("blend", KBlend),
    ENTRY("curl", KCurl),
    ENTRY("hmlstm_update", KHmlstm),
    ENTRY("hmlstm_update_bias", KHmlstmBias),
    ENTRY("fanout", KFanout),
    ENTRY("fiveway", KFiveway),
    ENTRY("wave", KWave),
    ENTRY("gate", KGate),
    ENTRY("sig_tanh", KSigTanh),
    ENTRY("square_gate", KSquareGate),
    ENTRY("two", KTwo),
    ENTRY("log", KLog),
    ENTRY("div", KDiv),
    ENTRY("sqrt", KSqrt),
    ENTRY("abs", KAbs),
    ENTRY("pow_half", KPowHalf),
    ENTRY("recip", KRecip),
    ENTRY("exp", KExp),
    ENTRY("tanh_product_1", TanhProduct<1>),
    ENTRY("tanh_product_2", TanhProduct<2>),
    ENTRY("tanh_product_3", TanhProduct<3>),
    ENTRY("tanh_product_4", TanhProduct<4>),
    ENTRY("tanh_product_5", TanhProduct<5>),
    ENTRY("tanh_product_8", TanhProduct<8>),
    ENTRY("tanh_product_16", TanhProduct<16>),
    ENTRY("tanh_product_18", TanhProduct<18>),
    ENTRY("tanh_product_32", TanhProduct<32>),
};
#undef ENTRY

const Entry& find(const char* name) {
    for (const Entry& e : kEntries)
        if (std::strcmp(e.name, name) == 0) return e;
    throw OracleError(kUnknownPrimitive, std::string("unknown kernel ") + name);
}

template <class Fn>
int guarded(Fn&& fn) {
    try {
        fn();
        return kOk;
    } catch (const OracleError& e) {
        g_last_error = e.what();
        return e.code;
    } catch (const std::exception& e) {
        g_last_error = e.what();
        return kGeneric;
    }
}

}  // namespace

extern "C" {

const char* oracle_last_error(void) { return g_last_error.c_str(); }

int oracle_kernel_count(void) { return int(sizeof(kEntries) / sizeof(kEntries[0])); }
const char* oracle_kernel_name(int idx) { return kEntries[idx].name; }

int oracle_kernel_info(const char* name, int* n_in, int* m_out) {
    return guarded([&] {
        const Entry& e = find(name);
        *n_in = e.n_in;
        *m_out = e.m_out;
    });
}

// bench.cpp:31-37
uint64_t oracle_mix_seed(uint64_t seed, uint64_t salt) {
    uint64_t x = seed ^ (salt * 0x9e3779b97f4a7c15ULL);
    x ^= x >> 30;
    x *= 0xbf58476d1ce4e5b9ULL;
    x ^= x >> 27;
    return x;
}

// One Rng(seed) (rng.hpp:11-31) drawn in tensor order: kind 0 = random_pm1
// (2*u01 - 1, cast), kind 1 = random_binary(p=0.5) (tensor.hpp:71-84).
int oracle_gen(uint64_t seed, int dtype, int n, const int64_t* volumes, const int* kinds,
               void* const* outs) {
    return guarded([&] {
        std::mt19937_64 gen(seed);
        for (int t = 0; t < n; ++t) {
            for (int64_t e = 0; e < volumes[t]; ++e) {
                const double u = double(gen() >> 11) * 0x1.0p-53;
                const double v = kinds[t] == 1 ? (u < 0.5 ? 1.0 : 0.0) : 2.0 * u - 1.0;
                if (dtype == 0) static_cast<float*>(outs[t])[e] = float(v);
                else static_cast<double*>(outs[t])[e] = v;
            }
        }
    });
}

int oracle_broadcast_shape(int n, const OShape* shapes, OShape* out) {
    return guarded([&] { *out = broadcast_shape(shapes, n); });
}

// primal_out: M pointers (entries nullable); partials_out: M*N pointers or
// NULL. real_body != 0 runs the real instantiation (broadcast_apply).
int oracle_forward(const char* name, int dtype, int n_in, const void* const* in,
                   const OShape* shapes, void* const* primal_out, void* const* partials_out,
                   int real_body) {
    return guarded([&] {
        const Entry& e = find(name);
        if (n_in != e.n_in)
            throw OracleError(kArityMismatch, std::string("kernel ") + name + " expects " +
                                                  std::to_string(e.n_in) + " arguments, got " +
                                                  std::to_string(n_in));
        (dtype == 0 ? e.fwd32 : e.fwd64)(in, shapes, primal_out, partials_out, real_body != 0);
    });
}

int oracle_pullback(int dtype, int n_in, int m_out, const OShape* shapes, const void* const* out_adj,
                    const void* const* partials, void* const* in_adj, const unsigned char* accumulate,
                    double* const* acc64) {
    return guarded([&] {
        if (dtype == 0)
            pullback_impl<float>(n_in, m_out, shapes, out_adj, partials, in_adj, accumulate, acc64);
        else
            pullback_impl<double>(n_in, m_out, shapes, out_adj, partials, in_adj, accumulate, acc64);
    });
}

// scatter_add(acc, contribution) alone (broadcast.hpp:210-217).
int oracle_scatter_add(int dtype, void* acc, const OShape* acc_shape, const void* contrib,
                       const OShape* contrib_shape) {
    return guarded([&] {
        const OShape both[2] = {*acc_shape, *contrib_shape};
        const OShape out = broadcast_shape(both, 2);
        const int64_t vol = volume(out);
        Walker w(out);
        for (int64_t cell = 0; cell < vol; ++cell, w.advance()) {
            const int64_t a = w.index_in(*acc_shape), c = w.index_in(*contrib_shape);
            if (dtype == 0) static_cast<float*>(acc)[a] += static_cast<const float*>(contrib)[c];
            else static_cast<double*>(acc)[a] += static_cast<const double*>(contrib)[c];
        }
    });
}

}  // extern "C"
