// BroadcastKernel: a named pure scalar function of N inputs to M outputs.
//
// Reference: proj/include/bcad/kernel.hpp:21-51 stores a generic body twice
// (real and dual instantiation) behind std::function and evaluates it on the
// CPU. std::function cannot run on a GPU, so here the body is a compiled
// device functor registered in libbcad_cu.so under the reference kernel's
// name (paper_1810_08297_b200/csrc/bodies.cuh); constructing a kernel binds
// the name to that device body and enforces the same arity rules
// (kernel.hpp:30-35). A name with no device body throws UnknownPrimitive —
// there is no CPU fallback. The body-taking constructor keeps the reference's
// signature so user code compiles unchanged; the host body is not evaluated.
#pragma once

#include <string>
#include <utility>

#include "bcad/errors.hpp"

namespace bcad {

inline constexpr int kMaxPartials = BCAD_CU_MAX_INPUTS;
inline constexpr int kMaxKernelInputs = BCAD_CU_MAX_INPUTS;
inline constexpr int kMaxKernelOutputs = BCAD_CU_MAX_OUTPUTS;

template <class Real>
class BroadcastKernel {
public:
    BroadcastKernel(int arity_in, int arity_out, std::string name)
        : arity_in_(arity_in), arity_out_(arity_out), name_(std::move(name)) {
        if (arity_in_ < 1 || arity_in_ > kMaxKernelInputs)
            throw ArityMismatch("kernel input arity " + std::to_string(arity_in_) + " outside [1, " +
                                std::to_string(kMaxKernelInputs) + "]");
        if (arity_out_ < 1 || arity_out_ > kMaxKernelOutputs)
            throw ArityMismatch("kernel output arity " + std::to_string(arity_out_) + " outside [1, " +
                                std::to_string(kMaxKernelOutputs) + "]");
        check(bcad_cu_kernel_lookup(name_.c_str(), arity_in_, arity_out_, &handle_));
    }

    template <class Body>
    BroadcastKernel(int arity_in, int arity_out, std::string name, Body&&)
        : BroadcastKernel(arity_in, arity_out, std::move(name)) {}

    int arity_in() const { return arity_in_; }
    int arity_out() const { return arity_out_; }
    const std::string& name() const { return name_; }
    bcad_cu_kernel handle() const { return handle_; }
    bool may_raise() const { return bcad_cu_kernel_may_raise(handle_) != 0; }

private:
    int arity_in_;
    int arity_out_;
    std::string name_;
    bcad_cu_kernel handle_ = nullptr;
};

template <class Real>
BroadcastKernel<Real> identity_kernel() {  // kernel.hpp:72-76
    return BroadcastKernel<Real>(1, 1, "identity");
}

}  // namespace bcad
