// BroadcastKernel: a named pure scalar function of N inputs to M outputs.
//
// Reference: proj/include/bcad/kernel.hpp:21-51 stores a generic body twice
// (real and dual instantiation) behind std::function and evaluates it on the
// CPU. std::function cannot run on a GPU, so every broadcast here runs a
// compiled device functor registered in libbcad_cu.so under the kernel's
// name — the library's own bodies (csrc/bodies.cuh) or a user's, registered
// from the user's nvcc translation unit with BCAD_DEVICE_KERNEL
// (bcad/device_kernel.cuh). The arity rules are the reference's
// (kernel.hpp:30-35); a name with no device body throws UnknownPrimitive —
// there is no CPU fallback.
//
// The body-taking constructor keeps the reference's signature, so reference
// code compiles unchanged. It keeps the body for host evaluation (eval, like
// the reference) and CHECKS it against the device body bound by name: both
// are evaluated on a fixed set of probe points (exact 0 / 1 branch values and
// uniform values) on reals-with-duals, and any difference in a primal or a
// partial throws ConfigError. A lambda under a registered name that computes
// something else therefore fails loudly instead of running the library's math.
#pragma once

#include <algorithm>
#include <array>
#include <cmath>
#include <cstdint>
#include <functional>
#include <memory>
#include <mutex>
#include <set>
#include <span>
#include <string>
#include <typeinfo>
#include <utility>
#include <vector>

#include "bcad/dual.hpp"
#include "bcad/errors.hpp"
#include "bcad/tensor.hpp"

namespace bcad {

inline constexpr int kMaxKernelInputs = BCAD_CU_MAX_INPUTS;
inline constexpr int kMaxKernelOutputs = BCAD_CU_MAX_OUTPUTS;

template <class Real>
class BroadcastKernel;

namespace detail {

template <class Real>
struct ComposedStages;  // compose_kernels(g, f): the stages, applied f then g

// One forward launch over `cells` probe points given as per-argument host
// columns; returns the M primals and (when `jac`) the M*N partial columns.
template <class Real>
void device_probe(bcad_cu_kernel k, int n, int m, std::int64_t cells, const std::vector<std::vector<Real>>& cols,
                  bool jac, std::vector<std::vector<Real>>* primal, std::vector<std::vector<Real>>* partials) {
    const Shape s{cells};
    std::vector<Tensor<Real>> in, po, pa;
    for (int j = 0; j < n; ++j) in.push_back(Tensor<Real>::from(s, cols[static_cast<std::size_t>(j)]));
    for (int i = 0; i < m; ++i) po.push_back(Tensor<Real>::uninitialized(s));
    if (jac)
        for (int t = 0; t < m * n; ++t) pa.push_back(Tensor<Real>::uninitialized(s));
    std::vector<const void*> ip;
    std::vector<void*> pp, ap;
    std::vector<bcad_cu_shape> shapes(static_cast<std::size_t>(n), s.c_shape());
    for (auto& t : in) ip.push_back(t.device_data());
    for (auto& t : po) pp.push_back(t.device_data());
    for (auto& t : pa) ap.push_back(t.device_data());
    check(bcad_cu_forward(k, dtype_of<Real>::value, n, ip.data(), shapes.data(), m, pp.data(),
                          jac ? ap.data() : nullptr, current_stream()));
    primal->clear();
    for (auto& t : po) primal->push_back(t.to_host());
    if (partials) {
        partials->clear();
        for (auto& t : pa) partials->push_back(t.to_host());
    }
}

inline bool probe_close(double a, double b, double rtol, double atol) {
    if (std::isnan(a) || std::isnan(b)) return std::isnan(a) && std::isnan(b);
    if (std::isinf(a) || std::isinf(b)) return a == b;
    return std::fabs(a - b) <= atol + rtol * std::max(std::fabs(a), std::fabs(b));
}

// Bodies already checked against their device body (type of the body, name,
// real type): the check runs once per distinct body per process.
inline std::mutex& checked_mutex() {
    static std::mutex m;
    return m;
}
inline std::set<std::string>& checked_bodies() {
    static std::set<std::string> s;
    return s;
}

}  // namespace detail

template <class Real>
class BroadcastKernel {
public:
    using DualT = Dual<Real>;

    // Device body only: `name` must be registered (library or user).
    BroadcastKernel(int arity_in, int arity_out, std::string name)
        : arity_in_(arity_in), arity_out_(arity_out), name_(std::move(name)) {
        bind();
    }

    // Reference signature (kernel.hpp:26-43): the generic body is kept for
    // host evaluation and checked against the device body of `name`.
    template <class Body>
    BroadcastKernel(int arity_in, int arity_out, std::string name, Body body)
        : arity_in_(arity_in), arity_out_(arity_out), name_(std::move(name)), real_body_(body), dual_body_(body) {
        bind();
        const std::string key = std::string(typeid(Body).name()) + "|" + name_ + "|" + typeid(Real).name();
        {
            std::lock_guard<std::mutex> lock(detail::checked_mutex());
            if (detail::checked_bodies().count(key)) return;
        }
        check_against_device();
        std::lock_guard<std::mutex> lock(detail::checked_mutex());
        detail::checked_bodies().insert(key);
    }

    int arity_in() const { return arity_in_; }
    int arity_out() const { return arity_out_; }
    const std::string& name() const { return name_; }
    bcad_cu_kernel handle() const { return handle_; }
    bool may_raise() const;
    bool has_host_body() const;
    // A kernel made by compose_kernels: no device body of its own; its stages
    // run as one launch each (broadcast_apply), see compose_kernels below.
    bool is_composite() const { return static_cast<bool>(stages_); }
    const detail::ComposedStages<Real>& stages() const { return *stages_; }

    // One scalar evaluation (kernel.hpp:45-46). With a host body: the body,
    // as the reference does. Device-only kernels: one cell on the device
    // (synchronous); on duals the outputs carry J * (input perturbations),
    // J the device's M x N partials at the primal point.
    void eval(std::span<const Real> in, std::span<Real> out) const {
        if (stages_) return eval_composite<Real>(in, out);
        if (real_body_) return real_body_(in, out);
        std::vector<std::vector<Real>> cols, prim;
        for (int j = 0; j < arity_in_; ++j) cols.push_back({in[static_cast<std::size_t>(j)]});
        detail::device_probe<Real>(handle_, arity_in_, arity_out_, 1, cols, false, &prim, nullptr);
        for (int i = 0; i < arity_out_; ++i) out[static_cast<std::size_t>(i)] = prim[static_cast<std::size_t>(i)][0];
    }
    void eval(std::span<const DualT> in, std::span<DualT> out) const {
        if (stages_) return eval_composite<DualT>(in, out);
        if (dual_body_) return dual_body_(in, out);
        Tag tag{};
        int width = 0;
        std::vector<std::vector<Real>> cols, prim, part;
        for (int j = 0; j < arity_in_; ++j) {
            const DualT& x = in[static_cast<std::size_t>(j)];
            if (!x.is_constant()) {
                if (tag.id != 0 && !(tag == x.tag())) throw TagMismatch("dual arguments across distinct tags");
                tag = x.tag();
                width = std::max(width, x.width());
            }
            cols.push_back({x.primal()});
        }
        detail::device_probe<Real>(handle_, arity_in_, arity_out_, 1, cols, true, &prim, &part);
        for (int i = 0; i < arity_out_; ++i) {
            DualT r(prim[static_cast<std::size_t>(i)][0], width, tag);
            for (int k = 0; k < width; ++k) {
                Real d = Real(0);
                for (int j = 0; j < arity_in_; ++j)
                    d = d + part[static_cast<std::size_t>(i * arity_in_ + j)][0] * in[static_cast<std::size_t>(j)].partial(k);
                r.set_partial(k, d);
            }
            out[static_cast<std::size_t>(i)] = r;
        }
    }

private:
    template <class R>
    friend BroadcastKernel<R> compose_kernels(const BroadcastKernel<R>& g, const BroadcastKernel<R>& f);

    BroadcastKernel(int arity_in, int arity_out, std::string name,
                    std::shared_ptr<const detail::ComposedStages<Real>> stages)
        : arity_in_(arity_in), arity_out_(arity_out), name_(std::move(name)), stages_(std::move(stages)) {}

    template <class S>
    void eval_composite(std::span<const S> in, std::span<S> out) const;

    void bind() {
        if (arity_in_ < 1 || arity_in_ > kMaxKernelInputs)
            throw ArityMismatch("kernel input arity " + std::to_string(arity_in_) + " outside [1, " +
                                std::to_string(kMaxKernelInputs) + "]");
        if (arity_out_ < 1 || arity_out_ > kMaxKernelOutputs)
            throw ArityMismatch("kernel output arity " + std::to_string(arity_out_) + " outside [1, " +
                                std::to_string(kMaxKernelOutputs) + "]");
        check(bcad_cu_kernel_lookup(name_.c_str(), arity_in_, arity_out_, &handle_));
    }

    // Probe points: 256 cells, each argument exactly 0 or 1 with probability
    // 1/4 each (the values branch predicates test, e.g. the HM-LSTM boundary
    // bits, hmlstm.hpp:51-53) and otherwise uniform in [-2, 2) (fixed seed).
    // Points where the host body raises (division by zero, log of a negative)
    // are skipped; the rest must agree with the device in every primal and
    // partial to a few ulps of host-vs-device libm (relative 1e-4 fp32, 1e-9
    // fp64) — a different function differs by O(1).
    void check_against_device() const {
        const CountPause no_census;  // the reference evaluates nothing at construction
        constexpr std::int64_t kProbes = 256;
        const int n = arity_in_, m = arity_out_;
        Rng rng(0x6263616400ULL + static_cast<std::uint64_t>(n) * 131 + static_cast<std::uint64_t>(m));
        std::vector<std::vector<Real>> cols(static_cast<std::size_t>(n));
        std::vector<Real> want_p, want_d;  // kept probes: m primals, m*n partials each
        std::vector<Real> x(static_cast<std::size_t>(n));
        std::vector<DualT> xin(static_cast<std::size_t>(n)), yout(static_cast<std::size_t>(m));
        for (std::int64_t p = 0; p < kProbes; ++p) {
            for (int j = 0; j < n; ++j) {
                const std::uint64_t kind = rng.below(4);
                const double u = rng.uniform_pm1();
                x[static_cast<std::size_t>(j)] = kind == 0 ? Real(0) : kind == 1 ? Real(1) : static_cast<Real>(2.0 * u);
            }
            const Tag tag = fresh_tag();
            try {
                seed_into<Real>(std::span<const Real>(x), tag, std::span<DualT>(xin));
                dual_body_(std::span<const DualT>(xin), std::span<DualT>(yout));
            } catch (const Error&) {
                continue;  // outside the body's domain: the device would raise too
            }
            for (int j = 0; j < n; ++j) cols[static_cast<std::size_t>(j)].push_back(x[static_cast<std::size_t>(j)]);
            for (int i = 0; i < m; ++i) {
                want_p.push_back(yout[static_cast<std::size_t>(i)].primal());
                for (int j = 0; j < n; ++j) want_d.push_back(yout[static_cast<std::size_t>(i)].partial_for(tag, j));
            }
        }
        const std::int64_t kept = static_cast<std::int64_t>(cols[0].size());
        if (kept == 0)
            throw ConfigError("kernel '" + name_ + "': cannot check the body against its device body, every probe "
                              "point raised on the host");
        std::vector<std::vector<Real>> got_p, got_d;
        detail::device_probe<Real>(handle_, n, m, kept, cols, true, &got_p, &got_d);
        const double rtol = sizeof(Real) == 4 ? 1e-4 : 1e-9, atol = sizeof(Real) == 4 ? 1e-6 : 1e-12;
        for (std::int64_t p = 0; p < kept; ++p)
            for (int i = 0; i < m; ++i) {
                const double hp = want_p[static_cast<std::size_t>(p * m + i)];
                const double dp = got_p[static_cast<std::size_t>(i)][static_cast<std::size_t>(p)];
                bool ok = detail::probe_close(hp, dp, rtol, atol);
                int bad_j = -1;
                for (int j = 0; j < n && ok; ++j) {
                    const double hd = want_d[static_cast<std::size_t>((p * m + i) * n + j)];
                    const double dd = got_d[static_cast<std::size_t>(i * n + j)][static_cast<std::size_t>(p)];
                    if (!detail::probe_close(hd, dd, rtol, atol)) {
                        ok = false;
                        bad_j = j;
                    }
                }
                if (!ok) {
                    std::string at = "(";
                    for (int j = 0; j < n; ++j)
                        at += (j ? ", " : "") + std::to_string(cols[static_cast<std::size_t>(j)][static_cast<std::size_t>(p)]);
                    throw ConfigError("kernel '" + name_ + "': the body given to BroadcastKernel differs from the "
                                      "device body registered under that name (output " + std::to_string(i) +
                                      (bad_j < 0 ? " primal" : ", partial d/dx" + std::to_string(bad_j)) + " at " +
                                      at + ")); register the new body under its own name with "
                                      "BCAD_DEVICE_KERNEL (bcad/device_kernel.cuh)");
                }
            }
    }

    int arity_in_;
    int arity_out_;
    std::string name_;
    bcad_cu_kernel handle_ = nullptr;
    std::function<void(std::span<const Real>, std::span<Real>)> real_body_;
    std::function<void(std::span<const DualT>, std::span<DualT>)> dual_body_;
    std::shared_ptr<const detail::ComposedStages<Real>> stages_;
};

namespace detail {
template <class Real>
struct ComposedStages {
    BroadcastKernel<Real> g, f;  // out = g(f(in))
};
}  // namespace detail

template <class Real>
bool BroadcastKernel<Real>::may_raise() const {
    if (stages_) return stages_->f.may_raise() || stages_->g.may_raise();
    return bcad_cu_kernel_may_raise(handle_) != 0;
}

template <class Real>
bool BroadcastKernel<Real>::has_host_body() const {
    if (stages_) return stages_->f.has_host_body() && stages_->g.has_host_body();
    return static_cast<bool>(real_body_);
}

template <class Real>
template <class S>
void BroadcastKernel<Real>::eval_composite(std::span<const S> in, std::span<S> out) const {
    std::array<S, kMaxKernelOutputs> mid;
    stages_->f.eval(in, std::span<S>(mid.data(), static_cast<std::size_t>(stages_->f.arity_out())));
    stages_->g.eval(std::span<const S>(mid.data(), static_cast<std::size_t>(stages_->g.arity_in())), out);
}

// g after f as one kernel (reference kernel.hpp:54-70). The reference fuses
// the two bodies into one lambda run in a single element visit. Device bodies
// are compiled functors and cannot be fused at run time, so here the composed
// kernel runs its stages as one launch each in broadcast_apply (f over the
// broadcast, then g elementwise over f's outputs): bit-identical to applying
// f and then g, which is the reference's fusion law (test_broadcast.cpp:168-193).
// Differentiating a composed kernel (broadcast_diag_jacobian / mixed_broadcast)
// throws ConfigError: record the stages as two mixed nodes instead.
template <class Real>
BroadcastKernel<Real> compose_kernels(const BroadcastKernel<Real>& g, const BroadcastKernel<Real>& f) {
    if (g.arity_in() != f.arity_out())
        throw ArityMismatch("cannot compose: inner kernel produces " + std::to_string(f.arity_out()) +
                            " outputs, outer expects " + std::to_string(g.arity_in()));
    return BroadcastKernel<Real>(f.arity_in(), g.arity_out(), g.name() + "." + f.name(),
                                 std::make_shared<const detail::ComposedStages<Real>>(detail::ComposedStages<Real>{g, f}));
}

template <class Real>
BroadcastKernel<Real> identity_kernel() {  // kernel.hpp:72-76
    return BroadcastKernel<Real>(1, 1, "identity", [](auto in, auto out) { out[0] = in[0]; });
}

}  // namespace bcad
