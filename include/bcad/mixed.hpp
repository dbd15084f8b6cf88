// Mixed-mode broadcast node: forward-mode per element on the device, one
// reverse tape node (reference proj/include/bcad/mixed.hpp:17-130).
//
//   CacheForward     K1 writes the primal and the M*N Jacobian diagonals in
//                    one pass (bcad_cu_forward); they ride the node cache;
//                    the node's backward is ONE K2 launch (bcad_cu_pullback)
//                    that multiplies the output adjoints into the cached
//                    diagonals and sum-reduces over broadcast axes.
//   RecomputeReverse K1p writes the primal only (real body); the backward is
//                    ONE fused K2r launch that re-derives the diagonals from
//                    the inputs in registers and reduces — nothing cached.
#pragma once

#include <initializer_list>
#include <memory>
#include <span>
#include <utility>
#include <vector>

#include "bcad/forward.hpp"
#include "bcad/tape.hpp"

namespace bcad {

enum class MixedPolicy {
    CacheForward,
    RecomputeReverse,
};

namespace detail {

// backprop_diag (mixed.hpp:27-41) as one device pullback. The node's output
// adjoints are the w_i; each input's slot is created on first touch, or added
// into when it already holds contributions. An input that appears twice
// pulls into a scratch tensor that is then accumulated into the shared slot
// (the kernel's adjoint pointers must not alias).
template <class Real>
void backprop_diag_device(Tape<Real>& tape, int node, const BroadcastKernel<Real>& kernel, bool cached) {
    const std::span<const Var<Real>> ins = tape.node_inputs(node);
    const int n = kernel.arity_in(), m = kernel.arity_out();
    std::vector<bcad_cu_shape> shapes;
    std::vector<const void*> in_ptrs, w(static_cast<std::size_t>(m), nullptr), parts;
    for (const Var<Real>& v : ins) {
        shapes.push_back(tape.value(v).shape().c_shape());
        in_ptrs.push_back(tape.value(v).device_data());
    }
    for (int i = 0; i < m; ++i)
        if (const Tensor<Real>* a = tape.adjoint_or_null(node, i)) w[static_cast<std::size_t>(i)] = a->device_data();
    if (cached)
        for (const Tensor<Real>& t : tape.node_cache(node)) parts.push_back(t.device_data());

    std::vector<void*> adj(static_cast<std::size_t>(n), nullptr);
    std::vector<unsigned char> acc(static_cast<std::size_t>(n), 0);
    std::vector<std::pair<int, Tensor<Real>>> dup;  // (first index, scratch) for repeated inputs
    for (int j = 0; j < n; ++j) {
        int first = j;
        for (int l = 0; l < j; ++l)
            if (ins[static_cast<std::size_t>(l)].node == ins[static_cast<std::size_t>(j)].node &&
                ins[static_cast<std::size_t>(l)].slot == ins[static_cast<std::size_t>(j)].slot) {
                first = l;
                break;
            }
        if (first != j) {
            dup.emplace_back(first, Tensor<Real>::uninitialized(tape.value(ins[static_cast<std::size_t>(j)]).shape()));
            adj[static_cast<std::size_t>(j)] = dup.back().second.device_data();
            continue;
        }
        bool existed = false;
        Tensor<Real>& slot = tape.adjoint_slot(ins[static_cast<std::size_t>(j)], &existed);
        adj[static_cast<std::size_t>(j)] = slot.device_data();
        acc[static_cast<std::size_t>(j)] = existed ? 1 : 0;
    }
    std::size_t ws_bytes = 0;
    check(bcad_cu_pullback_workspace(kernel.handle(), dtype_of<Real>::value, n, shapes.data(), m, &ws_bytes));
    void* ws = tape.workspace(node, ws_bytes);
    check(bcad_cu_pullback(kernel.handle(), dtype_of<Real>::value, n, shapes.data(), m, w.data(),
                           cached ? parts.data() : nullptr, in_ptrs.data(), adj.data(), acc.data(), ws,
                           tape.workspace_bytes(node), current_stream()));
    // RecomputeReverse re-derives the diagonals in K2r, visiting every output
    // cell again (the reference reruns broadcast_diag_jacobian, mixed.hpp:85)
    if (!cached) count_element_visits(static_cast<std::uint64_t>(tape.value(Var<Real>{&tape, node, 0}).volume()));
    for (auto& [first, scratch] : dup) tape.accumulate_adjoint(ins[static_cast<std::size_t>(first)], scratch);
}

}  // namespace detail

// Records a whole broadcast kernel as ONE tape node (mixed.hpp:49-91).
template <class Real>
std::vector<Var<Real>> mixed_broadcast(Tape<Real>& tape, const BroadcastKernel<Real>& kernel,
                                       std::span<const Var<Real>> inputs, MixedPolicy policy) {
    if (static_cast<int>(inputs.size()) != kernel.arity_in())
        throw ArityMismatch("mixed_broadcast: kernel " + kernel.name() + " expects " +
                            std::to_string(kernel.arity_in()) + " inputs, got " + std::to_string(inputs.size()));
    detail::require_single_stage(kernel, "mixed_broadcast");
    std::vector<const Tensor<Real>*> args;
    for (const Var<Real>& v : inputs) args.push_back(&tape.value(v));
    auto k = std::make_shared<BroadcastKernel<Real>>(kernel);
    if (policy == MixedPolicy::CacheForward) {
        ForwardBroadcastResult<Real> fwd =
            broadcast_diag_jacobian<Real>(kernel, std::span<const Tensor<Real>* const>(args), /*want_primal=*/true);
        return tape.append_custom("mixed[" + kernel.name() + "]", inputs, std::move(fwd.primals),
                                  std::move(fwd.jacobian.entries), [k](Tape<Real>& t, int node) {
                                      detail::backprop_diag_device<Real>(t, node, *k, /*cached=*/true);
                                  });
    }
    std::vector<Tensor<Real>> primals = broadcast_apply<Real>(kernel, std::span<const Tensor<Real>* const>(args));
    return tape.append_custom("mixed[" + kernel.name() + "]", inputs, std::move(primals), {},
                              [k](Tape<Real>& t, int node) {
                                  detail::backprop_diag_device<Real>(t, node, *k, /*cached=*/false);
                              });
}

template <class Real>
std::vector<Var<Real>> mixed_broadcast(Tape<Real>& tape, const BroadcastKernel<Real>& kernel,
                                       std::initializer_list<Var<Real>> inputs, MixedPolicy policy) {
    return mixed_broadcast(tape, kernel, std::span<const Var<Real>>(inputs.begin(), inputs.size()), policy);
}

// Both policies on fresh tapes, every output seeded with ones; true when all
// input gradients are bit-identical (mixed.hpp:103-130).
template <class Real>
bool policy_equivalence_check(const BroadcastKernel<Real>& kernel, std::span<const Tensor<Real>> inputs) {
    auto run = [&](MixedPolicy policy) {
        Tape<Real> tape;
        std::vector<Var<Real>> vars;
        for (const Tensor<Real>& t : inputs) vars.push_back(tape.input(t));
        std::vector<Var<Real>> outs = mixed_broadcast<Real>(tape, kernel, vars, policy);
        std::vector<std::pair<Var<Real>, Tensor<Real>>> seeds;
        for (Var<Real> o : outs) seeds.emplace_back(o, Tensor<Real>(tape.value(o).shape(), Real(1)));
        Gradients<Real> grads = tape.backward(std::span<const std::pair<Var<Real>, Tensor<Real>>>(seeds));
        std::vector<std::vector<Real>> out;
        for (Var<Real> v : vars) out.push_back(grads.at(v).to_host());
        return out;
    };
    const auto cached = run(MixedPolicy::CacheForward);
    const auto recomputed = run(MixedPolicy::RecomputeReverse);
    for (std::size_t k = 0; k < cached.size(); ++k)
        for (std::size_t e = 0; e < cached[k].size(); ++e)
            if (cached[k][e] != recomputed[k][e]) return false;
    return true;
}

}  // namespace bcad
