// Forward broadcast evaluation on the device:
//   broadcast_apply         (reference proj/include/bcad/broadcast.hpp:102-125)
//   broadcast_diag_jacobian (reference proj/include/bcad/forward.hpp:98-150)
//   scatter_add             (reference proj/include/bcad/broadcast.hpp:210-217)
// Each is one C-ABI call into the fused sm_100a kernels. Like the reference
// (broadcast.hpp:123, forward.hpp:148), each broadcast adds its output volume
// to the element-visit counter (bcad/counters.hpp): the launch visits every
// output cell exactly once.
#pragma once

#include <array>
#include <span>
#include <vector>

#include "bcad/counters.hpp"
#include "bcad/kernel.hpp"
#include "bcad/tensor.hpp"

namespace bcad {

template <class Real>
struct DiagJacobian {
    Shape out_shape;
    int outputs = 0;  // M
    int inputs = 0;   // N
    std::vector<Tensor<Real>> entries;  // M*N tensors, all of out_shape

    Tensor<Real>& entry(int i, int j) { return entries[static_cast<std::size_t>(i * inputs + j)]; }
    const Tensor<Real>& entry(int i, int j) const { return entries[static_cast<std::size_t>(i * inputs + j)]; }
};

template <class Real>
struct ForwardBroadcastResult {
    std::vector<Tensor<Real>> primals;  // populated only when requested
    DiagJacobian<Real> jacobian;
};

// The pointwise Jacobian operator (forward.hpp:38-72): one evaluation of
// the kernel on seeded duals at a single point gives the M primals and the
// row-major M x N partial matrix. A scalar utility (BroadcastKernel::eval);
// the broadcast path is broadcast_diag_jacobian below, on the device.
template <class Real>
class PointwiseJacobian {
public:
    explicit PointwiseJacobian(BroadcastKernel<Real> kernel) : kernel_(std::move(kernel)) {}
    int arity_in() const { return kernel_.arity_in(); }
    int arity_out() const { return kernel_.arity_out(); }
    void operator()(std::span<const Real> x, std::span<Real> primals, std::span<Real> jacobian) const {
        const int n = kernel_.arity_in(), m = kernel_.arity_out();
        const Tag tag = fresh_tag();
        std::array<Dual<Real>, kMaxKernelInputs> in;
        seed_into<Real>(x, tag, std::span<Dual<Real>>(in.data(), static_cast<std::size_t>(n)));
        std::array<Dual<Real>, kMaxKernelOutputs> out;
        kernel_.eval(std::span<const Dual<Real>>(in.data(), static_cast<std::size_t>(n)),
                     std::span<Dual<Real>>(out.data(), static_cast<std::size_t>(m)));
        for (int i = 0; i < m; ++i) {
            primals[static_cast<std::size_t>(i)] = out[static_cast<std::size_t>(i)].primal();
            for (int j = 0; j < n; ++j)
                jacobian[static_cast<std::size_t>(i * n + j)] = out[static_cast<std::size_t>(i)].partial_for(tag, j);
        }
    }
    const BroadcastKernel<Real>& kernel() const { return kernel_; }

private:
    BroadcastKernel<Real> kernel_;
};

template <class Real>
PointwiseJacobian<Real> jacobian_operator(const BroadcastKernel<Real>& kernel) {
    return PointwiseJacobian<Real>(kernel);
}

namespace detail {

template <class Real>
std::vector<bcad_cu_shape> c_shapes(std::span<const Tensor<Real>* const> args) {
    std::vector<bcad_cu_shape> s;
    s.reserve(args.size());
    for (const Tensor<Real>* t : args) s.push_back(t->shape().c_shape());
    return s;
}

template <class Real>
Shape out_shape_of(std::span<const Tensor<Real>* const> args) {
    std::vector<Shape> s;
    s.reserve(args.size());
    for (const Tensor<Real>* t : args) s.push_back(t->shape());
    return broadcast_shape(std::span<const Shape>(s));
}

template <class Real>
void check_arity(const BroadcastKernel<Real>& kernel, std::size_t n, const char* who) {
    if (static_cast<int>(n) != kernel.arity_in())
        throw ArityMismatch(std::string(who) + ": kernel " + kernel.name() + " expects " +
                            std::to_string(kernel.arity_in()) + " arguments, got " + std::to_string(n));
}

template <class Real>
void require_single_stage(const BroadcastKernel<Real>& kernel, const char* who) {
    if (kernel.is_composite())
        throw ConfigError(std::string(who) + ": kernel " + kernel.name() + " is a composition (compose_kernels), "
                          "which runs in broadcast_apply only; differentiate its stages as separate nodes");
}

}  // namespace detail

template <class Real>
std::vector<Tensor<Real>> broadcast_apply(const BroadcastKernel<Real>& kernel,
                                          std::span<const Tensor<Real>* const> args) {
    detail::check_arity(kernel, args.size(), "broadcast_apply");
    if (kernel.is_composite()) {  // compose_kernels: one launch per stage
        const std::vector<Tensor<Real>> mid = broadcast_apply<Real>(kernel.stages().f, args);
        std::vector<const Tensor<Real>*> mp;
        for (const Tensor<Real>& t : mid) mp.push_back(&t);
        return broadcast_apply<Real>(kernel.stages().g, std::span<const Tensor<Real>* const>(mp));
    }
    const Shape out = detail::out_shape_of<Real>(args);
    const auto shapes = detail::c_shapes<Real>(args);
    std::vector<const void*> in;
    for (const Tensor<Real>* t : args) in.push_back(t->device_data());
    std::vector<Tensor<Real>> outs;
    std::vector<void*> po;
    for (int i = 0; i < kernel.arity_out(); ++i) {
        outs.push_back(Tensor<Real>::uninitialized(out));
        po.push_back(outs.back().device_data());
    }
    check(bcad_cu_forward(kernel.handle(), dtype_of<Real>::value, kernel.arity_in(), in.data(), shapes.data(),
                          kernel.arity_out(), po.data(), nullptr, current_stream()));
    count_element_visits(static_cast<std::uint64_t>(out.volume()));
    return outs;
}

template <class Real, class... Ts>
    requires(std::same_as<std::remove_cvref_t<Ts>, Tensor<Real>> && ...)
std::vector<Tensor<Real>> broadcast_apply(const BroadcastKernel<Real>& kernel, const Ts&... args) {
    const std::array<const Tensor<Real>*, sizeof...(Ts)> ptrs{&args...};
    return broadcast_apply<Real>(kernel, std::span<const Tensor<Real>* const>(ptrs));
}

template <class Real>
ForwardBroadcastResult<Real> broadcast_diag_jacobian(const BroadcastKernel<Real>& kernel,
                                                     std::span<const Tensor<Real>* const> args, bool want_primal) {
    detail::check_arity(kernel, args.size(), "broadcast_diag_jacobian");
    detail::require_single_stage(kernel, "broadcast_diag_jacobian");
    const Shape out = detail::out_shape_of<Real>(args);
    const auto shapes = detail::c_shapes<Real>(args);
    const int n = kernel.arity_in(), m = kernel.arity_out();
    std::vector<const void*> in;
    for (const Tensor<Real>* t : args) in.push_back(t->device_data());
    ForwardBroadcastResult<Real> r;
    r.jacobian.out_shape = out;
    r.jacobian.outputs = m;
    r.jacobian.inputs = n;
    std::vector<void*> pp, po;
    for (int k = 0; k < m * n; ++k) {
        r.jacobian.entries.push_back(Tensor<Real>::uninitialized(out));
        pp.push_back(r.jacobian.entries.back().device_data());
    }
    if (want_primal)
        for (int i = 0; i < m; ++i) {
            r.primals.push_back(Tensor<Real>::uninitialized(out));
            po.push_back(r.primals.back().device_data());
        }
    check(bcad_cu_forward(kernel.handle(), dtype_of<Real>::value, n, in.data(), shapes.data(), m,
                          want_primal ? po.data() : nullptr, pp.data(), current_stream()));
    count_element_visits(static_cast<std::uint64_t>(out.volume()));
    return r;
}

template <class Real, class... Ts>
    requires(std::same_as<std::remove_cvref_t<Ts>, Tensor<Real>> && ...)
ForwardBroadcastResult<Real> broadcast_diag_jacobian(const BroadcastKernel<Real>& kernel, bool want_primal,
                                                     const Ts&... args) {
    const std::array<const Tensor<Real>*, sizeof...(Ts)> ptrs{&args...};
    return broadcast_diag_jacobian<Real>(kernel, std::span<const Tensor<Real>* const>(ptrs), want_primal);
}

// The reference's serial diagonal path (forward.hpp:162-210), kept because
// its API has it: one host PointwiseJacobian evaluation per output cell on
// host copies of the arguments. It is the test-side comparison for
// broadcast_diag_jacobian, never called by it.
template <class Real>
ForwardBroadcastResult<Real> broadcast_diag_jacobian_reference(const BroadcastKernel<Real>& kernel,
                                                               std::span<const Tensor<Real>* const> args,
                                                               bool want_primal) {
    detail::check_arity(kernel, args.size(), "broadcast_diag_jacobian_reference");
    std::vector<Shape> shapes;
    std::vector<std::vector<Real>> host;
    for (const Tensor<Real>* t : args) {
        shapes.push_back(t->shape());
        host.push_back(t->to_host());
    }
    const Shape out = broadcast_shape(std::span<const Shape>(shapes));
    const std::int64_t vol = out.volume();
    const int n = kernel.arity_in(), m = kernel.arity_out();
    const PointwiseJacobian<Real> op(kernel);
    std::vector<std::vector<Real>> prim(static_cast<std::size_t>(m), std::vector<Real>(static_cast<std::size_t>(vol)));
    std::vector<std::vector<Real>> part(static_cast<std::size_t>(m * n), std::vector<Real>(static_cast<std::size_t>(vol)));
    std::vector<std::int64_t> idx(static_cast<std::size_t>(out.rank()));
    std::array<Real, kMaxKernelInputs> x;
    std::array<Real, kMaxKernelOutputs> p;
    std::array<Real, kMaxKernelInputs * kMaxKernelOutputs> jac;
    for (std::int64_t c = 0; c < vol; ++c) {
        unflatten_index(out, c, idx);
        for (int j = 0; j < n; ++j)
            x[static_cast<std::size_t>(j)] = host[static_cast<std::size_t>(j)][static_cast<std::size_t>(
                virtual_index(shapes[static_cast<std::size_t>(j)], idx, out))];
        op(std::span<const Real>(x.data(), static_cast<std::size_t>(n)), std::span<Real>(p.data(), static_cast<std::size_t>(m)),
           std::span<Real>(jac.data(), static_cast<std::size_t>(m * n)));
        for (int i = 0; i < m; ++i) {
            prim[static_cast<std::size_t>(i)][static_cast<std::size_t>(c)] = p[static_cast<std::size_t>(i)];
            for (int j = 0; j < n; ++j)
                part[static_cast<std::size_t>(i * n + j)][static_cast<std::size_t>(c)] = jac[static_cast<std::size_t>(i * n + j)];
        }
    }
    count_element_visits(static_cast<std::uint64_t>(vol));
    ForwardBroadcastResult<Real> r;
    r.jacobian.out_shape = out;
    r.jacobian.outputs = m;
    r.jacobian.inputs = n;
    for (auto& v : part) r.jacobian.entries.push_back(Tensor<Real>::from(out, v));
    if (want_primal)
        for (auto& v : prim) r.primals.push_back(Tensor<Real>::from(out, v));
    return r;
}

template <class Real, class... Ts>
    requires(std::same_as<std::remove_cvref_t<Ts>, Tensor<Real>> && ...)
ForwardBroadcastResult<Real> broadcast_diag_jacobian_reference(const BroadcastKernel<Real>& kernel, bool want_primal,
                                                               const Ts&... args) {
    const std::array<const Tensor<Real>*, sizeof...(Ts)> ptrs{&args...};
    return broadcast_diag_jacobian_reference<Real>(kernel, std::span<const Tensor<Real>* const>(ptrs), want_primal);
}

// The central broadcast-adjoint rule: reduces `contribution` over axes `acc`
// lacks, or expands it along axes `acc` has and it lacks.
template <class Real>
void scatter_add(Tensor<Real>& acc, const Tensor<Real>& contribution, bool zero_first = false) {
    const bcad_cu_shape a = acc.shape().c_shape(), c = contribution.shape().c_shape();
    check(bcad_cu_scatter_add(dtype_of<Real>::value, acc.device_data(), &a, contribution.device_data(), &c,
                              zero_first ? 1 : 0, current_stream()));
}

}  // namespace bcad
