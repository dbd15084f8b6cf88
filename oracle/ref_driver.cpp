// ORACLE — TEST INFRASTRUCTURE ONLY.
//
// C-ABI driver around the UNMODIFIED reference library (/root/reference/proj,
// header-only bcad + src/counters.cpp + src/parallel.cpp), compiled where the
// sources lie by oracle/Makefile into oracle/_ref/libbcad_ref.so with the
// reference's Release numerics (-O3 -ffp-contract=off -fopenmp). Nothing of
// the reference is copied: this file only includes its headers and calls its
// public API, exactly as proj/src/bench.cpp:94-129 (run_cell_once) does.
//
// Uses: (1) pin oracle/oracle.cpp bit-for-bit, (2) produce tests/golden/
// fixtures, (3) the CPU baseline / `bench.py --impl reference` arm.
// The product never links this library.

#include <algorithm>
#include <chrono>
#include <cstdint>
#include <cstring>
#include <stdexcept>
#include <string>
#include <vector>

#include "bcad/arity_workload.hpp"
#include "bcad/counters.hpp"
#include "bcad/hmlstm.hpp"
#include "bcad/mixed.hpp"
#include "bcad/parallel.hpp"

#ifdef _OPENMP
#include <omp.h>
#endif

using namespace bcad;

namespace {

struct OShape {  // layout shared with bcad_cu_shape / oracle.cpp
    int32_t rank;
    int32_t pad;
    int64_t dims[8];
};

Shape to_shape(const OShape& s) {
    return Shape(std::vector<std::int64_t>(s.dims, s.dims + s.rank));
}

thread_local std::string g_last_error;

// Status codes of include/bcad_cu.h, one per errors.hpp type.
int code_of(const std::exception& e) {
    if (dynamic_cast<const TagMismatch*>(&e)) return 1;
    if (dynamic_cast<const DivisionByZero*>(&e)) return 2;
    if (dynamic_cast<const DomainError*>(&e)) return 3;
    if (dynamic_cast<const NonDifferentiablePoint*>(&e)) return 4;
    if (dynamic_cast<const ShapeMismatch*>(&e)) return 5;
    if (dynamic_cast<const ArityMismatch*>(&e)) return 6;
    if (dynamic_cast<const SeedShapeMismatch*>(&e)) return 7;
    if (dynamic_cast<const UnknownPrimitive*>(&e)) return 8;
    return 15;
}

template <class Fn>
int guarded(Fn&& fn) {
    try {
        fn();
        return 0;
    } catch (const std::exception& e) {
        g_last_error = e.what();
        return code_of(e);
    }
}

// The kernel set, written as the reference writes them (hmlstm.hpp:56-61,
// arity_workload.hpp:19-28, tests/support/kernel_pool.hpp:19-102,
// tests/test_mixed.cpp, tests/test_broadcast.cpp).
template <class Real>
BroadcastKernel<Real> make_kernel(const std::string& name) {
    using K = BroadcastKernel<Real>;
    if (name == "identity") return identity_kernel<Real>();
    if (name == "reflect") return K(1, 1, name, [](auto in, auto out) { out[0] = reflect_below_half(in[0]); });
    if (name == "tanh_sigmoid")
        return K(1, 1, name, [](auto in, auto out) { out[0] = tanh(in[0]) * sigmoid(in[0]); });
    if (name == "product" || name == "mul")
        return K(2, 1, name, [](auto in, auto out) { out[0] = in[0] * in[1]; });
    if (name == "plus") return K(2, 1, name, [](auto in, auto out) { out[0] = in[0] + in[1]; });
    if (name == "gated")
        return K(2, 1, name, [](auto in, auto out) { out[0] = in[0] + sigmoid(in[1]) * tanh(in[0]); });
    if (name == "prod_diff")
        return K(2, 2, name, [](auto in, auto out) {
            out[0] = in[0] * in[1];
            out[1] = in[0] - in[1];
        });
    if (name == "blend")
        return K(3, 1, name, [](auto in, auto out) {
            auto w = sigmoid(in[0]);
            out[0] = w * in[1] + (1.0 - w) * in[2];
        });
    if (name == "curl")
        return K(3, 2, name, [](auto in, auto out) {
            out[0] = in[0] * in[1] + cos(in[2]);
            out[1] = in[2] * tanh(in[0]);
        });
    if (name == "hmlstm_update") return cell_update_kernel<Real>();
    if (name == "hmlstm_update_bias")  // SURVEY §8(d) config 3 / 5 bias variant
        return K(9, 1, name, [](auto in, auto out) {
            out[0] = cell_update_scalar(in[0], in[1] + in[4], in[2] + in[5], in[3] + in[6], in[7], in[8]);
        });
    if (name == "fanout")
        return K(2, 3, name, [](auto in, auto out) {
            out[0] = in[0] + in[1];
            out[1] = in[0] * in[1];
            out[2] = sigmoid(in[0]) - tanh(in[1]);
        });
    if (name == "fiveway")
        return K(5, 1, name, [](auto in, auto out) { out[0] = in[0] * in[1] + in[2] * in[3] * in[4]; });
    if (name == "wave")
        return K(3, 1, name, [](auto in, auto out) {
            out[0] = sin(in[0]) * exp(-(in[1] * in[1])) + cos(in[2]);
        });
    if (name == "gate")
        return K(2, 1, name, [](auto in, auto out) { out[0] = sigmoid(in[0]) * tanh(in[1]) + in[0]; });
    if (name == "sig_tanh")
        return K(2, 1, name, [](auto in, auto out) { out[0] = sigmoid(in[0]) * tanh(in[1]); });
    if (name == "square_gate")
        return K(2, 1, name, [](auto in, auto out) { out[0] = sigmoid(in[0]) * in[1]; });
    if (name == "two")
        return K(2, 2, name, [](auto in, auto out) {
            out[0] = in[0] * in[1];
            out[1] = sigmoid(in[0]) + tanh(in[1]);
        });
    if (name == "log") return K(1, 1, name, [](auto in, auto out) { out[0] = log(in[0]); });
    if (name == "div") return K(2, 1, name, [](auto in, auto out) { out[0] = in[0] / in[1]; });
    if (name == "sqrt") return K(1, 1, name, [](auto in, auto out) { out[0] = sqrt(in[0]); });
    if (name == "abs") return K(1, 1, name, [](auto in, auto out) { out[0] = abs(in[0]); });
    if (name == "pow_half") return K(1, 1, name, [](auto in, auto out) { out[0] = pow(in[0], 0.5); });
    if (name == "recip") return K(1, 1, name, [](auto in, auto out) { out[0] = 1.0 / in[0]; });
    if (name == "exp") return K(1, 1, name, [](auto in, auto out) { out[0] = exp(in[0]); });
    if (name.rfind("tanh_product_", 0) == 0) return tanh_product_kernel<Real>(std::stoi(name.substr(13)));
    throw UnknownPrimitive("unknown kernel " + name);
}

template <class Real>
std::vector<Tensor<Real>> wrap_inputs(int n, const void* const* in, const OShape* shapes) {
    std::vector<Tensor<Real>> t;
    t.reserve(size_t(n));
    for (int j = 0; j < n; ++j) {
        const Shape s = to_shape(shapes[j]);
        const Real* p = static_cast<const Real*>(in[j]);
        t.push_back(Tensor<Real>::from(s, std::vector<Real>(p, p + s.volume())));
    }
    return t;
}

template <class Real>
void copy_out(const Tensor<Real>& t, void* dst) {
    if (dst) std::memcpy(dst, t.data().data(), size_t(t.volume()) * sizeof(Real));
}

template <class Real>
void forward_t(const char* name, int n, const void* const* in, const OShape* shapes,
               void* const* primal_out, void* const* partials_out, int real_body) {
    const BroadcastKernel<Real> k = make_kernel<Real>(name);
    const auto args = wrap_inputs<Real>(n, in, shapes);
    std::vector<const Tensor<Real>*> ptrs;
    for (const auto& a : args) ptrs.push_back(&a);
    if (real_body) {
        const auto outs = broadcast_apply<Real>(k, ptrs);
        for (size_t i = 0; i < outs.size(); ++i)
            if (primal_out) copy_out(outs[i], primal_out[i]);
        return;
    }
    const auto fwd = broadcast_diag_jacobian<Real>(k, ptrs, primal_out != nullptr);
    const int m = fwd.jacobian.outputs, nn = fwd.jacobian.inputs;
    for (int i = 0; i < m; ++i) {
        if (primal_out) copy_out(fwd.primals[size_t(i)], primal_out[i]);
        if (partials_out)
            for (int j = 0; j < nn; ++j) copy_out(fwd.jacobian.entry(i, j), partials_out[i * nn + j]);
    }
}

std::uint64_t now_ns();

// One mixed step through the reference's tape (bench.cpp:112-128):
// inputs -> mixed_broadcast(policy) -> backward(seeds) -> leaf gradients.
// t_mid (optional) receives the clock after mixed_broadcast (forward / backward split).
template <class Real>
std::int64_t mixed_step_t(const BroadcastKernel<Real>& k, const std::vector<Tensor<Real>>& args,
                          int policy, const void* const* seeds, void* const* primal_out,
                          void* const* grads_out, std::uint64_t* t_mid = nullptr) {
    Tape<Real> tape;
    std::vector<Var<Real>> vars;
    for (const auto& a : args) vars.push_back(tape.input(a));
    const auto outs = mixed_broadcast<Real>(
        tape, k, vars, policy == 0 ? MixedPolicy::CacheForward : MixedPolicy::RecomputeReverse);
    if (t_mid) *t_mid = now_ns();
    std::vector<std::pair<Var<Real>, Tensor<Real>>> sv;
    for (size_t i = 0; i < outs.size(); ++i) {
        const Tensor<Real>& val = tape.value(outs[i]);
        if (primal_out) copy_out(val, primal_out[i]);
        if (seeds && seeds[i]) {
            const Real* p = static_cast<const Real*>(seeds[i]);
            sv.emplace_back(outs[i], Tensor<Real>::from(val.shape(), std::vector<Real>(p, p + val.volume())));
        }
    }
    const Gradients<Real> g =
        tape.backward(std::span<const std::pair<Var<Real>, Tensor<Real>>>(sv.data(), sv.size()));
    if (grads_out)
        for (size_t j = 0; j < vars.size(); ++j) copy_out(g.at(vars[j]), grads_out[j]);
    return tape.peak_cached_bytes();
}

std::uint64_t now_ns() {
    return std::uint64_t(std::chrono::duration_cast<std::chrono::nanoseconds>(
                             std::chrono::steady_clock::now().time_since_epoch())
                             .count());
}

}  // namespace

extern "C" {

const char* ref_last_error(void) { return g_last_error.c_str(); }

int ref_gen(uint64_t seed, int dtype, int n, const int64_t* volumes, const int* kinds, void* const* outs) {
    return guarded([&] {
        Rng rng(seed);
        for (int t = 0; t < n; ++t) {
            const Shape s{volumes[t]};
            if (dtype == 0) {
                const auto x = kinds[t] == 1 ? random_binary<float>(s, rng) : random_pm1<float>(s, rng);
                copy_out(x, outs[t]);
            } else {
                const auto x = kinds[t] == 1 ? random_binary<double>(s, rng) : random_pm1<double>(s, rng);
                copy_out(x, outs[t]);
            }
        }
    });
}

int ref_broadcast_shape(int n, const OShape* shapes, OShape* out) {
    return guarded([&] {
        std::vector<Shape> s;
        for (int j = 0; j < n; ++j) s.push_back(to_shape(shapes[j]));
        const Shape b = broadcast_shape(std::span<const Shape>(s));
        *out = OShape{};
        out->rank = b.rank();
        for (int k = 0; k < b.rank(); ++k) out->dims[k] = b.dim(k);
    });
}

int ref_forward(const char* name, int dtype, int n_in, const void* const* in, const OShape* shapes,
                void* const* primal_out, void* const* partials_out, int real_body) {
    return guarded([&] {
        if (dtype == 0) forward_t<float>(name, n_in, in, shapes, primal_out, partials_out, real_body);
        else forward_t<double>(name, n_in, in, shapes, primal_out, partials_out, real_body);
    });
}

int ref_mixed_step(const char* name, int dtype, int n_in, const void* const* in, const OShape* shapes,
                   int policy, const void* const* seeds, void* const* primal_out, void* const* grads_out,
                   int64_t* peak_cached_bytes) {
    return guarded([&] {
        std::int64_t peak = 0;
        if (dtype == 0) {
            const auto k = make_kernel<float>(name);
            if (k.arity_in() != n_in) throw ArityMismatch("wrong input count");
            peak = mixed_step_t<float>(k, wrap_inputs<float>(n_in, in, shapes), policy, seeds, primal_out, grads_out);
        } else {
            const auto k = make_kernel<double>(name);
            if (k.arity_in() != n_in) throw ArityMismatch("wrong input count");
            peak = mixed_step_t<double>(k, wrap_inputs<double>(n_in, in, shapes), policy, seeds, primal_out, grads_out);
        }
        if (peak_cached_bytes) *peak_cached_bytes = peak;
    });
}

int ref_scatter_add(int dtype, void* acc, const OShape* acc_shape, const void* contrib,
                    const OShape* contrib_shape) {
    return guarded([&] {
        if (dtype == 0) {
            auto a = wrap_inputs<float>(1, &acc, acc_shape);
            auto c = wrap_inputs<float>(1, &contrib, contrib_shape);
            scatter_add(a[0], c[0]);
            copy_out(a[0], acc);
        } else {
            auto a = wrap_inputs<double>(1, &acc, acc_shape);
            auto c = wrap_inputs<double>(1, &contrib, contrib_shape);
            scatter_add(a[0], c[0]);
            copy_out(a[0], acc);
        }
    });
}

int ref_max_threads(void) {
#ifdef _OPENMP
    return omp_get_max_threads();
#else
    return 1;
#endif
}

// CPU baseline: `reps` timed mixed steps after `warmup`, each exactly what
// run_cell_once("mixed-cache"/"mixed-recompute") times (bench.cpp:112-128)
// with a ones seed (bench.cpp:173), on `threads` OpenMP threads
// (set_broadcast_threads, parallel.hpp:18-20; 0 = all). Per-rep ns go to
// out_ns[reps].
int ref_time_mixed(const char* name, int dtype, int n_in, const void* const* in, const OShape* shapes,
                   int policy, int threads, int warmup, int reps, uint64_t* out_ns) {
    return guarded([&] {
        set_broadcast_threads(threads);
        auto run = [&](auto tag) {
            using Real = decltype(tag);
            const auto k = make_kernel<Real>(name);
            const auto args = wrap_inputs<Real>(n_in, in, shapes);
            std::vector<Shape> s;
            for (const auto& a : args) s.push_back(a.shape());
            const Shape out = broadcast_shape(std::span<const Shape>(s));
            std::vector<Real> ones(size_t(out.volume()), Real(1));
            std::vector<const void*> seeds(size_t(k.arity_out()), ones.data());
            for (int w = 0; w < warmup; ++w) mixed_step_t<Real>(k, args, policy, seeds.data(), nullptr, nullptr);
            for (int r = 0; r < reps; ++r) {
                const std::uint64_t t0 = now_ns();
                mixed_step_t<Real>(k, args, policy, seeds.data(), nullptr, nullptr);
                out_ns[r] = now_ns() - t0;
            }
        };
        if (dtype == 0) run(float{});
        else run(double{});
        set_broadcast_threads(0);
    });
}

// The same steps split at the end of mixed_broadcast: forward (tape inputs +
// the mixed node's forward) and backward (seed + Tape::backward + gradient
// copies) ns per rep (SURVEY §8(d) asks for both).
int ref_time_mixed_split(const char* name, int dtype, int n_in, const void* const* in, const OShape* shapes,
                         int policy, int threads, int reps, uint64_t* fwd_ns, uint64_t* bwd_ns) {
    return guarded([&] {
        set_broadcast_threads(threads);
        auto run = [&](auto tag) {
            using Real = decltype(tag);
            const auto k = make_kernel<Real>(name);
            const auto args = wrap_inputs<Real>(n_in, in, shapes);
            std::vector<Shape> s;
            for (const auto& a : args) s.push_back(a.shape());
            const Shape out = broadcast_shape(std::span<const Shape>(s));
            std::vector<Real> ones(size_t(out.volume()), Real(1));
            std::vector<const void*> seeds(size_t(k.arity_out()), ones.data());
            for (int r = 0; r < reps; ++r) {
                std::uint64_t mid = 0;
                const std::uint64_t t0 = now_ns();
                mixed_step_t<Real>(k, args, policy, seeds.data(), nullptr, nullptr, &mid);
                const std::uint64_t t1 = now_ns();
                fwd_ns[r] = mid - t0;
                bwd_ns[r] = t1 - mid;
            }
        };
        if (dtype == 0) run(float{});
        else run(double{});
        set_broadcast_threads(0);
    });
}

}  // extern "C"
