// libbcad_host.so: the end-to-end host entry (include/bcad_host.h) written
// against the C++ drop-in API, exactly the reference's run_cell_once
// sequence (proj/src/bench.cpp:112-128) with device tensors.
#include "bcad_host.h"

#include <span>
#include <string>
#include <vector>

#include "bcad/bcad.hpp"

namespace {

thread_local std::string g_err;

int code_of(const std::exception& e) {
    using namespace bcad;
    if (dynamic_cast<const TagMismatch*>(&e)) return BCAD_CU_ERR_TAG_MISMATCH;
    if (dynamic_cast<const DivisionByZero*>(&e)) return BCAD_CU_ERR_DIVISION_BY_ZERO;
    if (dynamic_cast<const DomainError*>(&e)) return BCAD_CU_ERR_DOMAIN;
    if (dynamic_cast<const NonDifferentiablePoint*>(&e)) return BCAD_CU_ERR_NON_DIFFERENTIABLE;
    if (dynamic_cast<const ShapeMismatch*>(&e)) return BCAD_CU_ERR_SHAPE_MISMATCH;
    if (dynamic_cast<const ArityMismatch*>(&e)) return BCAD_CU_ERR_ARITY_MISMATCH;
    if (dynamic_cast<const SeedShapeMismatch*>(&e)) return BCAD_CU_ERR_SEED_SHAPE_MISMATCH;
    if (dynamic_cast<const UnknownPrimitive*>(&e)) return BCAD_CU_ERR_UNKNOWN_PRIMITIVE;
    if (dynamic_cast<const ConfigError*>(&e)) return BCAD_CU_ERR_CONFIG;
    if (dynamic_cast<const CudaError*>(&e)) return BCAD_CU_ERR_CUDA;
    if (dynamic_cast<const NcclError*>(&e)) return BCAD_CU_ERR_NCCL;
    return BCAD_CU_ERR_GENERIC;
}

template <class Real>
void step(const char* name, int n_in, const void* const* host_in, const bcad_cu_shape* shapes, int m_out,
          int policy, const void* const* host_seeds, void* const* host_primal, void* const* host_grads,
          int64_t* peak) {
    using namespace bcad;
    Tape<Real> tape;
    std::vector<Var<Real>> vars;
    for (int j = 0; j < n_in; ++j)
        vars.push_back(tape.input(Tensor<Real>::from_host(Shape::from_c(shapes[j]), static_cast<const Real*>(host_in[j]))));
    const BroadcastKernel<Real> kernel(n_in, m_out, name);
    const std::vector<Var<Real>> outs = mixed_broadcast<Real>(
        tape, kernel, std::span<const Var<Real>>(vars), policy == 0 ? MixedPolicy::CacheForward : MixedPolicy::RecomputeReverse);
    std::vector<std::pair<Var<Real>, Tensor<Real>>> seeds;
    for (int i = 0; i < m_out; ++i) {
        const Tensor<Real>& v = tape.value(outs[static_cast<std::size_t>(i)]);
        if (host_primal && host_primal[i])
            check(bcad_cu_memcpy(host_primal[i], v.device_data(), v.bytes(), 1, current_stream()));
        if (host_seeds && host_seeds[i])
            seeds.emplace_back(outs[static_cast<std::size_t>(i)],
                               Tensor<Real>::from_host(v.shape(), static_cast<const Real*>(host_seeds[i])));
    }
    const Gradients<Real> grads = tape.backward(std::span<const std::pair<Var<Real>, Tensor<Real>>>(seeds));
    for (int j = 0; j < n_in; ++j) {
        if (!host_grads || !host_grads[j]) continue;
        const Tensor<Real>& g = grads.at(vars[static_cast<std::size_t>(j)]);
        check(bcad_cu_memcpy(host_grads[j], g.device_data(), g.bytes(), 1, current_stream()));
    }
    check(bcad_cu_stream_synchronize(current_stream()));
    if (peak) *peak = tape.peak_cached_bytes();
}

template <class Real>
void cell_grads(int impl, int64_t n, const void* const* dev_in, const void* dev_seed, void* const* dev_grads,
                int64_t* nodes, int64_t* peak) {
    using namespace bcad;
    const Shape mat{n, n}, vec{n};
    auto dev = [](const Shape& s, const void* p) { return Tensor<Real>::from_device(s, static_cast<const Real*>(p)); };
    const CellInputs<Real> in{dev(mat, dev_in[0]), dev(mat, dev_in[1]), dev(mat, dev_in[2]),
                              dev(mat, dev_in[3]), dev(vec, dev_in[4]), dev(vec, dev_in[5])};
    const Tensor<Real> seed = dev(mat, dev_seed);
    Tape<Real> tape;
    CellGraph<Real> graph;
    if (impl == 0) graph = cell_update_fused(tape, in, MixedPolicy::CacheForward);
    else if (impl == 1) graph = cell_update_fused(tape, in, MixedPolicy::RecomputeReverse);
    else if (impl == 2) graph = cell_update_unfused(tape, in);
    else throw ConfigError("impl must be 0 (mixed-cache), 1 (mixed-recompute) or 2 (reverse-unfused)");
    const Gradients<Real> g = tape.backward(graph.out, seed);
    const Var<Real> leaves[4] = {graph.c_prev, graph.f, graph.i, graph.g};
    for (int k = 0; k < 4; ++k) {
        const Tensor<Real>& t = g.at(leaves[k]);
        check(bcad_cu_memcpy(dev_grads[k], t.device_data(), t.bytes(), 2, current_stream()));
    }
    if (nodes) *nodes = static_cast<int64_t>(tape.size());
    if (peak) *peak = tape.peak_cached_bytes();
}

}  // namespace

extern "C" {

int bcad_host_cell_gradients(int impl, int dtype, int64_t n, const void* const* dev_in, const void* dev_seed,
                             void* const* dev_grads, int64_t* tape_nodes, int64_t* peak_cached_bytes, void* stream) {
    try {
        bcad::StreamGuard guard(stream);
        if (dtype == BCAD_CU_F32) cell_grads<float>(impl, n, dev_in, dev_seed, dev_grads, tape_nodes, peak_cached_bytes);
        else if (dtype == BCAD_CU_F64) cell_grads<double>(impl, n, dev_in, dev_seed, dev_grads, tape_nodes, peak_cached_bytes);
        else throw bcad::ConfigError("dtype must be F32 or F64");
        return BCAD_CU_OK;
    } catch (const std::exception& e) {
        g_err = e.what();
        return code_of(e);
    }
}

const char* bcad_host_last_error(void) { return g_err.c_str(); }

int bcad_host_mixed_step(const char* kernel, int dtype, int n_in, const void* const* host_in,
                         const bcad_cu_shape* in_shapes, int m_out, int policy, const void* const* host_seeds,
                         void* const* host_primal, void* const* host_grads, int64_t* peak_cached_bytes,
                         void* stream) {
    try {
        bcad::StreamGuard guard(stream);
        if (dtype == BCAD_CU_F32)
            step<float>(kernel, n_in, host_in, in_shapes, m_out, policy, host_seeds, host_primal, host_grads, peak_cached_bytes);
        else if (dtype == BCAD_CU_F64)
            step<double>(kernel, n_in, host_in, in_shapes, m_out, policy, host_seeds, host_primal, host_grads, peak_cached_bytes);
        else
            throw bcad::ConfigError("dtype must be F32 or F64");
        return BCAD_CU_OK;
    } catch (const std::exception& e) {
        g_err = e.what();
        return code_of(e);
    }
}

}  // extern "C"
