// The reference's broadcast header (proj/include/bcad/broadcast.hpp), so code
// that includes "bcad/broadcast.hpp" compiles against this repo:
//
//   BroadcastPlan / make_broadcast_plan   host shape arithmetic (per-argument
//                                         strides, 0 on broadcast axes), as in
//                                         the reference (broadcast.hpp:19-41)
//   broadcast_apply                       the device forward (bcad/forward.hpp)
//   broadcast_apply_reference             the reference's serial per-cell path
//                                         (broadcast.hpp:129-160): host bodies
//                                         on host copies, virtual_index per
//                                         cell — a test-side comparison, never
//                                         called by broadcast_apply
//   scatter_add / reduce_sum_keepdims     the device adjoint reduction
//                                         (bcad/forward.hpp, broadcast.hpp:
//                                         205-232)
//
// Not provided: tensor_zip / tensor_zip3 / tensor_map and detail::
// plan_for_each (broadcast.hpp:56-96, 164-200), the reference's host loops
// over arbitrary host lambdas that its CPU tape primitives are built from.
// Here the w ⊙ D zip is fused into the pullback kernel and the tape
// primitives are device kernels (bcad/tape.hpp), so there is no host loop to
// hand a lambda to.
#pragma once

#include <array>
#include <cstdint>
#include <span>
#include <string>
#include <vector>

#include "bcad/counters.hpp"
#include "bcad/forward.hpp"
#include "bcad/kernel.hpp"
#include "bcad/parallel.hpp"
#include "bcad/shape.hpp"
#include "bcad/tensor.hpp"

namespace bcad {

struct BroadcastPlan {
    Shape out_shape;
    std::int64_t volume = 1;
    std::vector<std::vector<std::int64_t>> arg_strides;  // [arg][out axis]
};

inline BroadcastPlan make_broadcast_plan(std::span<const Shape> shapes) {
    BroadcastPlan plan;
    plan.out_shape = broadcast_shape(shapes);
    plan.volume = plan.out_shape.volume();
    const int rank = plan.out_shape.rank();
    for (const Shape& s : shapes) {
        // first-axis broadcasting (shape.hpp:13-16): axis k of the argument
        // is axis k of the output
        std::vector<std::int64_t> strides(static_cast<std::size_t>(rank), 0);
        std::int64_t running = 1;
        for (int k = s.rank() - 1; k >= 0; --k) {
            strides[static_cast<std::size_t>(k)] = s.dim(k) == 1 ? 0 : running;
            running *= s.dim(k);
        }
        plan.arg_strides.push_back(std::move(strides));
    }
    return plan;
}

namespace detail {

template <class Real>
std::vector<Shape> gather_shapes(std::span<const Tensor<Real>* const> args) {
    std::vector<Shape> shapes;
    shapes.reserve(args.size());
    for (const Tensor<Real>* t : args) shapes.push_back(t->shape());
    return shapes;
}

}  // namespace detail

// One host evaluation of the kernel per output cell on host copies of the
// arguments (the kernel's host body, or its device body one cell at a time
// when it has none). Host and device transcendentals may differ in the last
// bits, so against broadcast_apply it is a tolerance comparison, not a
// bitwise one (tests/cpp/test_libm_ulps_gpu.cpp measures the distance).
template <class Real>
std::vector<Tensor<Real>> broadcast_apply_reference(const BroadcastKernel<Real>& kernel,
                                                    std::span<const Tensor<Real>* const> args) {
    if (static_cast<int>(args.size()) != kernel.arity_in())
        throw ArityMismatch("broadcast_apply_reference: wrong argument count");
    const std::vector<Shape> shapes = detail::gather_shapes(args);
    const Shape out_shape = broadcast_shape(std::span<const Shape>(shapes));
    const std::int64_t vol = out_shape.volume();
    const int n = kernel.arity_in();
    const int m = kernel.arity_out();
    std::vector<std::vector<Real>> host;
    for (const Tensor<Real>* t : args) host.push_back(t->to_host());
    std::vector<std::vector<Real>> outs(static_cast<std::size_t>(m), std::vector<Real>(static_cast<std::size_t>(vol)));
    std::vector<std::int64_t> index(static_cast<std::size_t>(out_shape.rank()), 0);
    std::array<Real, kMaxKernelInputs> in;
    std::array<Real, kMaxKernelOutputs> out;
    for (std::int64_t flat = 0; flat < vol; ++flat) {
        unflatten_index(out_shape, flat, index);
        for (int j = 0; j < n; ++j)
            in[static_cast<std::size_t>(j)] = host[static_cast<std::size_t>(j)][static_cast<std::size_t>(
                virtual_index(shapes[static_cast<std::size_t>(j)], index, out_shape))];
        kernel.eval(std::span<const Real>(in.data(), static_cast<std::size_t>(n)),
                    std::span<Real>(out.data(), static_cast<std::size_t>(m)));
        for (int i = 0; i < m; ++i)
            outs[static_cast<std::size_t>(i)][static_cast<std::size_t>(flat)] = out[static_cast<std::size_t>(i)];
    }
    count_element_visits(static_cast<std::uint64_t>(vol));
    std::vector<Tensor<Real>> result;
    for (auto& v : outs) result.push_back(Tensor<Real>::from(out_shape, v));
    return result;
}

template <class Real, class... Ts>
    requires(std::same_as<std::remove_cvref_t<Ts>, Tensor<Real>> && ...)
std::vector<Tensor<Real>> broadcast_apply_reference(const BroadcastKernel<Real>& kernel, const Ts&... args) {
    const std::array<const Tensor<Real>*, sizeof...(Ts)> ptrs{&args...};
    return broadcast_apply_reference<Real>(kernel, std::span<const Tensor<Real>* const>(ptrs));
}

// Sum over the given axes, keeping them as length 1 (broadcast.hpp:220-232):
// one device scatter_add into a zero-filled result.
template <class Real>
Tensor<Real> reduce_sum_keepdims(const Tensor<Real>& a, std::span<const int> axes) {
    std::vector<std::int64_t> dims(a.shape().dims().begin(), a.shape().dims().end());
    for (int axis : axes) {
        if (axis < 0 || axis >= a.shape().rank())
            throw ShapeMismatch("reduce axis " + std::to_string(axis) + " out of range for " + a.shape().str());
        dims[static_cast<std::size_t>(axis)] = 1;
    }
    Tensor<Real> out = Tensor<Real>::uninitialized(Shape(std::move(dims)));
    scatter_add(out, a, /*zero_first=*/true);
    return out;
}

}  // namespace bcad
