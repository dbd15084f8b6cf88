// Name-keyed registry of device kernel bodies (the device-side stand-in for
// the reference's type-erased BroadcastKernel, proj/include/bcad/kernel.hpp:21-51).
#pragma once

#include <cstddef>
#include <string>

#include <cuda_runtime.h>

#include "bcad_cu.h"
#include "plan.hpp"

namespace bcad_cu_impl {

struct FwdArgs {
    int dtype;
    const void* const* in;
    void* const* primal;
    void* const* partials;  // null => real body, primal only
    cudaStream_t stream;
    unsigned long long* err;
    const Plan* plan;
    const Tiling* tiling = nullptr;  // tuning override (tests / scripts/lab); null = choose_tiling
    unsigned long long* tcount = nullptr;  // transcendental counter slots (null: counting not armed)
};

struct PullArgs {
    int dtype;
    const void* const* out_adj;
    const void* const* partials;  // null => recompute from `in`
    const void* const* in;
    void* const* in_adj;
    const unsigned char* accumulate;
    void* workspace;
    size_t ws_bytes;
    cudaStream_t stream;
    unsigned long long* err;
    const Plan* plan;
    const Tiling* tiling = nullptr;  // tuning override (tests / scripts/lab); null = choose_tiling
    const PeerParams* peer = nullptr;  // fused allreduce of the (1,H)-class adjoints over a peer group
    unsigned long long* tcount = nullptr;  // transcendental counter slots (null: counting not armed)
};

size_t pull_ws_any(const Plan& plan, int dtype);

}  // namespace bcad_cu_impl

struct bcad_cu_kernel_entry {
    const char* name;
    int n_in, m_out;
    bool may_raise;
    int (*fwd)(const bcad_cu_impl::FwdArgs&, std::string*);
    int (*pull)(const bcad_cu_impl::PullArgs&, std::string*);
};

// One registration group per translation unit (compiled in parallel).
int bcad_reg_hmlstm(const bcad_cu_kernel_entry** out);
int bcad_reg_pool(const bcad_cu_kernel_entry** out);
int bcad_reg_pool_b(const bcad_cu_kernel_entry** out);
int bcad_reg_probe(const bcad_cu_kernel_entry** out);
int bcad_reg_arity(const bcad_cu_kernel_entry** out);
int bcad_reg_arity_wide(const bcad_cu_kernel_entry** out);
int bcad_reg_arity_wide32(const bcad_cu_kernel_entry** out);
int bcad_reg_prims(const bcad_cu_kernel_entry** out);
