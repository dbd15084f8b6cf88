// C-ABI implementation (include/bcad_cu.h): registry lookup, plan checks,
// launches, error-word decoding, device memory, streams and NCCL.
#include <cuda_runtime.h>
#include <dlfcn.h>
#include <unistd.h>

#include <cstdint>
#include <cstring>
#include <atomic>
#include <mutex>
#include <string>
#include <vector>

#include "bcad_cu.h"
#include "plan.hpp"
#include "registry.hpp"

using namespace bcad_cu_impl;

namespace {

thread_local std::string g_err;

int fail(int code, const std::string& msg) {
    g_err = msg;
    return code;
}

int cuda_fail(cudaError_t e, const char* what) {
    return fail(BCAD_CU_ERR_CUDA, std::string(what) + ": " + cudaGetErrorString(e));
}

#define CU_TRY(expr, what)                          \
    do {                                            \
        const cudaError_t e_ = (expr);              \
        if (e_ != cudaSuccess) return cuda_fail(e_, what); \
    } while (0)

// ---------------------------------------------------------------- registry
// The library's bodies (registration groups, one per translation unit) plus
// bodies registered at load time from users' nvcc translation units
// (bcad/device_kernel.cuh -> bcad_cu_register_kernel). Entries are never
// removed, so a handle stays valid for the life of the process.
struct Registry {
    std::mutex mu;
    std::vector<const bcad_cu_kernel_entry*> all;
    Registry() {
        int (*groups[])(const bcad_cu_kernel_entry**) = {&bcad_reg_hmlstm,       &bcad_reg_pool,  &bcad_reg_pool_b,
                                                         &bcad_reg_probe,        &bcad_reg_prims, &bcad_reg_arity,
                                                         &bcad_reg_arity_wide,   &bcad_reg_arity_wide32};
        for (auto g : groups) {
            const bcad_cu_kernel_entry* e = nullptr;
            const int n = g(&e);
            for (int i = 0; i < n; ++i) all.push_back(e + i);
        }
    }
};

Registry& registry() {
    static Registry r;
    return r;
}

// ---------------------------------------------------------- error words
// A may-raise launch needs a device error word of its own: calls on
// different streams / threads run concurrently, so each call takes a word
// from a per-device pool (slabs of 64, grown on demand, never freed) and
// returns it after decoding. No two in-flight calls share a word.
constexpr int kMaxDevices = 64;
constexpr int kSlab = 64;
struct ErrorWordPool {
    std::mutex mu;
    std::vector<unsigned long long*> free_words[kMaxDevices];
};
ErrorWordPool& word_pool() {
    static ErrorWordPool p;
    return p;
}

class ErrorWord {
public:
    ErrorWord() = default;
    ErrorWord(const ErrorWord&) = delete;
    ErrorWord& operator=(const ErrorWord&) = delete;
    ~ErrorWord() {
        if (!word_) return;
        std::lock_guard<std::mutex> lock(word_pool().mu);
        word_pool().free_words[dev_].push_back(word_);
    }
    int acquire() {
        CU_TRY(cudaGetDevice(&dev_), "cudaGetDevice");
        if (dev_ < 0 || dev_ >= kMaxDevices) return fail(BCAD_CU_ERR_CUDA, "device ordinal out of range");
        std::lock_guard<std::mutex> lock(word_pool().mu);
        auto& fl = word_pool().free_words[dev_];
        if (fl.empty()) {
            void* p = nullptr;
            CU_TRY(cudaMalloc(&p, kSlab * sizeof(unsigned long long)), "cudaMalloc(error words)");
            for (int i = kSlab - 1; i >= 0; --i) fl.push_back(static_cast<unsigned long long*>(p) + i);
        }
        word_ = fl.back();
        fl.pop_back();
        return BCAD_CU_OK;
    }
    unsigned long long* get() const { return word_; }

private:
    int dev_ = 0;
    unsigned long long* word_ = nullptr;
};

// ---------------------------------------------- transcendental counters
// Device census of transcendental evaluations (the reference's
// EvalCounters::transcendental_evals). Armed by the first
// bcad_cu_eval_counters call: from then on every body-evaluating launch on a
// thread that has not paused counting is followed by a census launch
// (launch.cuh launch_census) that adds into the current device's kCountSlots
// slots. Programs that never read the counters never arm them.
struct CountState {
    std::mutex mu;
    std::atomic<bool> armed{false};
    unsigned long long* slots[kMaxDevices] = {};
};
CountState& count_state() {
    static CountState c;
    return c;
}
thread_local int t_count_pause = 0;

int count_slots_alloc(int dev, unsigned long long** out) {
    CountState& c = count_state();
    std::lock_guard<std::mutex> lock(c.mu);
    if (!c.slots[dev]) {
        void* p = nullptr;
        CU_TRY(cudaMalloc(&p, kCountSlots * sizeof(unsigned long long)), "cudaMalloc(counter slots)");
        CU_TRY(cudaMemset(p, 0, kCountSlots * sizeof(unsigned long long)), "cudaMemset(counter slots)");
        c.slots[dev] = static_cast<unsigned long long*>(p);
    }
    *out = c.slots[dev];
    return BCAD_CU_OK;
}

// The slots a launch should count into (null: not armed, or paused on this
// thread). Allocated when armed, so a launch under graph capture never
// allocates.
unsigned long long* count_slots_for_launch() {
    CountState& c = count_state();
    if (!c.armed.load(std::memory_order_acquire) || t_count_pause > 0) return nullptr;
    int dev = 0;
    if (cudaGetDevice(&dev) != cudaSuccess || dev < 0 || dev >= kMaxDevices) return nullptr;
    std::lock_guard<std::mutex> lock(c.mu);
    return c.slots[dev];
}

// A may-raise launch decodes its error word synchronously, which a stream
// under CUDA-graph capture cannot do: refuse explicitly instead.
int refuse_if_capturing(cudaStream_t s, const char* kernel) {
    cudaStreamCaptureStatus st = cudaStreamCaptureStatusNone;
    CU_TRY(cudaStreamIsCapturing(s, &st), "cudaStreamIsCapturing");
    if (st != cudaStreamCaptureStatusNone)
        return fail(BCAD_CU_ERR_CONFIG, std::string("kernel ") + kernel +
                                            " may raise a domain error, which is checked synchronously after the "
                                            "launch; it cannot be captured into a CUDA graph");
    return BCAD_CU_OK;
}

std::string index_string(const Plan& plan, int64_t flat) {  // forward.hpp:76-87
    int64_t idx[kMaxRank] = {};
    for (int k = plan.out_rank - 1; k >= 0; --k) {
        idx[k] = flat % plan.out_dims[k];
        flat /= plan.out_dims[k];
    }
    std::string s = "(";
    for (int k = 0; k < plan.out_rank; ++k) {
        if (k) s += ", ";
        s += std::to_string(idx[k]);
    }
    return s + ")";
}

int check_error_word(unsigned long long* word, cudaStream_t stream, const Plan& plan) {
    unsigned long long host = 0;
    CU_TRY(cudaMemcpyAsync(&host, word, sizeof(host), cudaMemcpyDeviceToHost, stream), "cudaMemcpyAsync(error word)");
    CU_TRY(cudaStreamSynchronize(stream), "cudaStreamSynchronize");
    if (host == ~0ull) return BCAD_CU_OK;
    const int code = int(host >> 56);
    const int64_t flat = int64_t(host & ((1ull << 56) - 1));
    const char* what = code == BCAD_CU_ERR_DIVISION_BY_ZERO   ? "dual division by zero"
                       : code == BCAD_CU_ERR_DOMAIN           ? "primal outside the primitive's domain"
                       : code == BCAD_CU_ERR_NON_DIFFERENTIABLE ? "primitive is not differentiable at this primal"
                                                               : "kernel error";
    return fail(code, std::string(what) + " at output index " + index_string(plan, flat));
}

int arity_check(const bcad_cu_kernel_entry* k, int n_in, int m_out) {
    if (!k) return fail(BCAD_CU_ERR_UNKNOWN_PRIMITIVE, "null kernel handle");
    if (n_in != k->n_in)
        return fail(BCAD_CU_ERR_ARITY_MISMATCH, std::string("kernel ") + k->name + " expects " +
                                                    std::to_string(k->n_in) + " arguments, got " +
                                                    std::to_string(n_in));
    if (m_out != k->m_out)
        return fail(BCAD_CU_ERR_ARITY_MISMATCH, std::string("kernel ") + k->name + " produces " +
                                                    std::to_string(k->m_out) + " outputs, got " +
                                                    std::to_string(m_out));
    return BCAD_CU_OK;
}

int dtype_check(int dtype) {
    if (dtype != BCAD_CU_F32 && dtype != BCAD_CU_F64) return fail(BCAD_CU_ERR_CONFIG, "dtype must be F32 or F64");
    return BCAD_CU_OK;
}

// --------------------------------------------------------- utility kernels
template <class T>
__global__ void fill_kernel(T* p, int64_t n, T v) {
    for (int64_t i = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; i < n; i += int64_t(gridDim.x) * blockDim.x)
        p[i] = v;
}

template <class T>
__global__ void add_same_kernel(T* acc, const T* c, int64_t n, bool zero_first) {
    for (int64_t i = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; i < n; i += int64_t(gridDim.x) * blockDim.x)
        acc[i] = (zero_first ? T(0) : acc[i]) + c[i];
}

struct ScatterGeom {
    int rank;
    int64_t out_dims[kMaxRank];
    int64_t acc_strides[kMaxRank];
    int64_t con_strides[kMaxRank];
    int64_t acc_vol;
};

// One thread per slot element: the expanded cells of `acc` are walked in
// row-major order (broadcast.hpp:210-217); reductions accumulate in fp64.
template <class T>
__global__ void scatter_add_kernel(T* acc, const T* con, ScatterGeom g, bool zero_first) {
    for (int64_t e = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; e < g.acc_vol;
         e += int64_t(gridDim.x) * blockDim.x) {
        int64_t coord[kMaxRank];
        int64_t rem = e, cnt = 1;
        for (int k = g.rank - 1; k >= 0; --k) {
            if (g.acc_strides[k] != 0) {
                coord[k] = rem % g.out_dims[k];
                rem /= g.out_dims[k];
            } else {
                coord[k] = 0;
                cnt *= g.out_dims[k];
            }
        }
        T exact = zero_first ? T(0) : acc[e];
        double sum = 0.0;
        for (int64_t q = 0; q < cnt; ++q) {
            int64_t ci = 0;
            for (int k = 0; k < g.rank; ++k) ci += coord[k] * g.con_strides[k];
            if (cnt == 1) exact = exact + con[ci];
            else sum += double(con[ci]);
            for (int k = g.rank - 1; k >= 0; --k) {
                if (g.acc_strides[k] != 0 || g.out_dims[k] == 1) continue;
                if (++coord[k] < g.out_dims[k]) break;
                coord[k] = 0;
            }
        }
        acc[e] = cnt == 1 ? exact : T((zero_first ? 0.0 : double(acc[e])) + sum);
    }
}

// Multi-buffer device copy: blockIdx.y selects the buffer, 16-byte vectors
// when both ends are 16-byte aligned, a byte loop for the rest.
constexpr int kCopyBatch = 64;
struct CopyBatchDesc {
    char* dst[kCopyBatch];
    const char* src[kCopyBatch];
    size_t bytes[kCopyBatch];
};

__global__ void copy_batch_kernel(const __grid_constant__ CopyBatchDesc d) {
    const int k = blockIdx.y;
    char* dst = d.dst[k];
    const char* src = d.src[k];
    const size_t nb = d.bytes[k];
    const bool vec = ((reinterpret_cast<uintptr_t>(dst) | reinterpret_cast<uintptr_t>(src)) & 15u) == 0;
    const size_t n16 = vec ? nb / 16 : 0;
    const size_t stride = size_t(gridDim.x) * blockDim.x;
    for (size_t i = blockIdx.x * size_t(blockDim.x) + threadIdx.x; i < n16; i += stride)
        reinterpret_cast<int4*>(dst)[i] = __ldcs(reinterpret_cast<const int4*>(src) + i);
    for (size_t i = n16 * 16 + blockIdx.x * size_t(blockDim.x) + threadIdx.x; i < nb; i += stride) dst[i] = src[i];
}

int grid_for(int64_t n) {
    const int64_t b = (n + 255) / 256;
    return int(b < 1 ? 1 : (b > 148 * 16 ? 148 * 16 : b));
}

// ------------------------------------------------------------------ NCCL
// Minimal run-time binding (nccl.h ABI: ncclUniqueId is 128 bytes; enum
// values ncclFloat32 = 7, ncclFloat64 = 8, ncclSum = 0).
struct Nccl {
    void* h = nullptr;
    int (*GetUniqueId)(void*) = nullptr;
    int (*CommInitRank)(void**, int, const void*, int) = nullptr;  // id passed by value (128 B)
    int (*CommDestroy)(void*) = nullptr;
    int (*CommCount)(void*, int*) = nullptr;
    int (*AllReduce)(const void*, void*, size_t, int, int, void*, cudaStream_t) = nullptr;
    int (*GroupStart)() = nullptr;
    int (*GroupEnd)() = nullptr;
    const char* (*GetErrorString)(int) = nullptr;
    bool ok = false;
};

struct NcclUniqueId {
    char internal[128];
};

Nccl& nccl() {
    static Nccl n = [] {
        Nccl x;
        for (const char* name : {"libnccl.so.2", "libnccl.so"}) {
            x.h = dlopen(name, RTLD_NOW | RTLD_GLOBAL);
            if (x.h) break;
        }
        if (!x.h) return x;
        x.GetUniqueId = reinterpret_cast<int (*)(void*)>(dlsym(x.h, "ncclGetUniqueId"));
        x.CommInitRank = reinterpret_cast<int (*)(void**, int, const void*, int)>(dlsym(x.h, "ncclCommInitRank"));
        x.CommDestroy = reinterpret_cast<int (*)(void*)>(dlsym(x.h, "ncclCommDestroy"));
        x.CommCount = reinterpret_cast<int (*)(void*, int*)>(dlsym(x.h, "ncclCommCount"));
        x.AllReduce = reinterpret_cast<int (*)(const void*, void*, size_t, int, int, void*, cudaStream_t)>(
            dlsym(x.h, "ncclAllReduce"));
        x.GroupStart = reinterpret_cast<int (*)()>(dlsym(x.h, "ncclGroupStart"));
        x.GroupEnd = reinterpret_cast<int (*)()>(dlsym(x.h, "ncclGroupEnd"));
        x.GetErrorString = reinterpret_cast<const char* (*)(int)>(dlsym(x.h, "ncclGetErrorString"));
        x.ok = x.GetUniqueId && x.CommInitRank && x.CommDestroy && x.AllReduce && x.GroupStart && x.GroupEnd;
        return x;
    }();
    return n;
}

int nccl_fail(int r, const char* what) {
    const Nccl& n = nccl();
    return fail(BCAD_CU_ERR_NCCL,
                std::string(what) + ": " + (n.GetErrorString ? n.GetErrorString(r) : "nccl error"));
}

}  // namespace

size_t bcad_cu_impl::pull_ws_any(const Plan& plan, int dtype) {
    return dtype == BCAD_CU_F32 ? pull_ws_t<float>(plan) : pull_ws_t<double>(plan);
}

extern "C" {

int bcad_cu_version(void) { return BCAD_CU_VERSION; }

const char* bcad_cu_last_error(void) { return g_err.c_str(); }

int bcad_cu_kernel_count(void) {
    std::lock_guard<std::mutex> lock(registry().mu);
    return int(registry().all.size());
}

const char* bcad_cu_kernel_name(int index) {
    std::lock_guard<std::mutex> lock(registry().mu);
    const auto& all = registry().all;
    return index >= 0 && index < int(all.size()) ? all[size_t(index)]->name : nullptr;
}

int bcad_cu_register_kernel(const bcad_cu_kernel_entry* entry) {
    if (!entry || !entry->name || !entry->fwd || !entry->pull) return fail(BCAD_CU_ERR_CONFIG, "incomplete kernel entry");
    if (entry->n_in < 1 || entry->n_in > BCAD_CU_MAX_INPUTS || entry->m_out < 1 || entry->m_out > BCAD_CU_MAX_OUTPUTS)
        return fail(BCAD_CU_ERR_ARITY_MISMATCH, std::string("kernel ") + entry->name + ": arity (" +
                                                    std::to_string(entry->n_in) + " -> " + std::to_string(entry->m_out) +
                                                    ") outside [1, 32] -> [1, 8]");
    std::lock_guard<std::mutex> lock(registry().mu);
    for (const bcad_cu_kernel_entry* e : registry().all)
        if (std::strcmp(e->name, entry->name) == 0)
            return fail(BCAD_CU_ERR_CONFIG, std::string("a device body is already registered under the name '") +
                                                entry->name + "'; registering a second body under it is refused");
    registry().all.push_back(entry);
    return BCAD_CU_OK;
}

int bcad_cu_kernel_lookup(const char* name, int n_in, int m_out, bcad_cu_kernel* out) {
    if (!name || !out) return fail(BCAD_CU_ERR_CONFIG, "null argument");
    // kernel.hpp:30-35
    if (n_in < 1 || n_in > BCAD_CU_MAX_INPUTS)
        return fail(BCAD_CU_ERR_ARITY_MISMATCH,
                    "kernel input arity " + std::to_string(n_in) + " outside [1, " + std::to_string(BCAD_CU_MAX_INPUTS) + "]");
    if (m_out < 1 || m_out > BCAD_CU_MAX_OUTPUTS)
        return fail(BCAD_CU_ERR_ARITY_MISMATCH, "kernel output arity " + std::to_string(m_out) + " outside [1, " +
                                                    std::to_string(BCAD_CU_MAX_OUTPUTS) + "]");
    std::lock_guard<std::mutex> lock(registry().mu);
    for (const bcad_cu_kernel_entry* e : registry().all) {
        if (std::strcmp(e->name, name) != 0) continue;
        if (e->n_in != n_in || e->m_out != m_out)
            return fail(BCAD_CU_ERR_ARITY_MISMATCH, std::string("kernel ") + name + " is registered as (" +
                                                        std::to_string(e->n_in) + " -> " + std::to_string(e->m_out) +
                                                        "), requested (" + std::to_string(n_in) + " -> " +
                                                        std::to_string(m_out) + ")");
        *out = e;
        return BCAD_CU_OK;
    }
    return fail(BCAD_CU_ERR_UNKNOWN_PRIMITIVE, std::string("no device body registered for kernel ") + name);
}

int bcad_cu_kernel_arity(bcad_cu_kernel k, int* n_in, int* m_out) {
    if (!k) return fail(BCAD_CU_ERR_UNKNOWN_PRIMITIVE, "null kernel handle");
    if (n_in) *n_in = k->n_in;
    if (m_out) *m_out = k->m_out;
    return BCAD_CU_OK;
}

int bcad_cu_kernel_may_raise(bcad_cu_kernel k) { return k && k->may_raise ? 1 : 0; }

int bcad_cu_broadcast_shape(int n, const bcad_cu_shape* shapes, bcad_cu_shape* out) {
    if (n < 1) return fail(BCAD_CU_ERR_SHAPE_MISMATCH, "broadcast_shape of an empty shape list");
    if (n > BCAD_CU_MAX_INPUTS) return fail(BCAD_CU_ERR_ARITY_MISMATCH, "too many shapes");
    Plan plan;
    std::string err;
    const int rc = make_plan(n, shapes, &plan, &err);
    if (rc) return fail(rc, err);
    *out = bcad_cu_shape{};
    out->rank = plan.out_rank;
    for (int k = 0; k < plan.out_rank; ++k) out->dims[k] = plan.out_dims[k];
    return BCAD_CU_OK;
}

int bcad_cu_eval_counters(unsigned long long* transcendental_evals) {
    if (!transcendental_evals) return fail(BCAD_CU_ERR_CONFIG, "null output");
    int dev = 0;
    CU_TRY(cudaGetDevice(&dev), "cudaGetDevice");
    if (dev < 0 || dev >= kMaxDevices) return fail(BCAD_CU_ERR_CUDA, "device ordinal out of range");
    unsigned long long* cur = nullptr;
    if (const int rc = count_slots_alloc(dev, &cur)) return rc;
    count_state().armed.store(true, std::memory_order_release);
    unsigned long long total = 0;
    std::vector<unsigned long long> h(kCountSlots);
    for (int d = 0; d < kMaxDevices; ++d) {
        unsigned long long* slots = nullptr;
        {
            std::lock_guard<std::mutex> lock(count_state().mu);
            slots = count_state().slots[d];
        }
        if (!slots) continue;
        CU_TRY(cudaSetDevice(d), "cudaSetDevice");
        CU_TRY(cudaDeviceSynchronize(), "cudaDeviceSynchronize");
        CU_TRY(cudaMemcpy(h.data(), slots, kCountSlots * sizeof(unsigned long long), cudaMemcpyDeviceToHost),
               "cudaMemcpy(counter slots)");
        for (unsigned long long v : h) total += v;
    }
    CU_TRY(cudaSetDevice(dev), "cudaSetDevice");
    *transcendental_evals = total;
    return BCAD_CU_OK;
}

int bcad_cu_count_pause(int pause) {
    t_count_pause += pause ? 1 : -1;
    if (t_count_pause < 0) t_count_pause = 0;
    return BCAD_CU_OK;
}

int bcad_cu_forward(bcad_cu_kernel k, int dtype, int n_in, const void* const* in, const bcad_cu_shape* in_shapes,
                    int m_out, void* const* primal_out, void* const* partials_out, void* stream) {
    int rc = arity_check(k, n_in, m_out);
    if (rc) return rc;
    if ((rc = dtype_check(dtype))) return rc;
    if (!in || !in_shapes) return fail(BCAD_CU_ERR_CONFIG, "null inputs");
    for (int j = 0; j < n_in; ++j)
        if (!in[j]) return fail(BCAD_CU_ERR_CONFIG, "null input pointer " + std::to_string(j));
    Plan plan;
    std::string err;
    if ((rc = make_plan(n_in, in_shapes, &plan, &err))) return fail(rc, err);
    cudaStream_t s = static_cast<cudaStream_t>(stream);
    ErrorWord ew;
    const bool check = k->may_raise && partials_out != nullptr;
    if (check) {
        if ((rc = refuse_if_capturing(s, k->name)) || (rc = ew.acquire())) return rc;
        CU_TRY(cudaMemsetAsync(ew.get(), 0xff, sizeof(unsigned long long), s), "cudaMemsetAsync(error word)");
    }
    unsigned long long* word = ew.get();
    FwdArgs a{dtype, in, primal_out, partials_out, s, word, &plan};
    a.tcount = count_slots_for_launch();
    if ((rc = k->fwd(a, &err))) return fail(rc, err);
    if (check) return check_error_word(word, s, plan);
    return BCAD_CU_OK;
}

int bcad_cu_pullback_workspace(bcad_cu_kernel k, int dtype, int n_in, const bcad_cu_shape* in_shapes, int m_out,
                               size_t* bytes) {
    int rc = arity_check(k, n_in, m_out);
    if (rc) return rc;
    if ((rc = dtype_check(dtype))) return rc;
    Plan plan;
    std::string err;
    if ((rc = make_plan(n_in, in_shapes, &plan, &err))) return fail(rc, err);
    *bytes = pull_ws_any(plan, dtype);
    return BCAD_CU_OK;
}

int bcad_cu_pullback_workspace_init(void* workspace, size_t bytes, void* stream) {
    if (bytes == 0) return BCAD_CU_OK;
    if (!workspace) return fail(BCAD_CU_ERR_CONFIG, "null workspace");
    CU_TRY(cudaMemsetAsync(workspace, 0, bytes, static_cast<cudaStream_t>(stream)), "cudaMemsetAsync(workspace)");
    return BCAD_CU_OK;
}

int bcad_cu_pullback_launches(bcad_cu_kernel k, int dtype, int n_in, const bcad_cu_shape* in_shapes, int m_out,
                              int* launches) {
    int rc = arity_check(k, n_in, m_out);
    if (rc) return rc;
    if ((rc = dtype_check(dtype))) return rc;
    Plan plan;
    std::string err;
    if ((rc = make_plan(n_in, in_shapes, &plan, &err))) return fail(rc, err);
    *launches = dtype == BCAD_CU_F32 ? pull_launches_t<float>(plan) : pull_launches_t<double>(plan);
    return BCAD_CU_OK;
}

namespace {
int pullback_impl(bcad_cu_kernel k, int dtype, int n_in, const bcad_cu_shape* in_shapes, int m_out,
                  const void* const* out_adj, const void* const* partials, const void* const* in,
                  void* const* in_adj, const unsigned char* accumulate, void* workspace, size_t workspace_bytes,
                  void* stream, const PeerParams* peer);
}

int bcad_cu_pullback(bcad_cu_kernel k, int dtype, int n_in, const bcad_cu_shape* in_shapes, int m_out,
                     const void* const* out_adj, const void* const* partials, const void* const* in,
                     void* const* in_adj, const unsigned char* accumulate, void* workspace, size_t workspace_bytes,
                     void* stream) {
    return pullback_impl(k, dtype, n_in, in_shapes, m_out, out_adj, partials, in, in_adj, accumulate, workspace,
                         workspace_bytes, stream, nullptr);
}

namespace {
int pullback_impl(bcad_cu_kernel k, int dtype, int n_in, const bcad_cu_shape* in_shapes, int m_out,
                  const void* const* out_adj, const void* const* partials, const void* const* in,
                  void* const* in_adj, const unsigned char* accumulate, void* workspace, size_t workspace_bytes,
                  void* stream, const PeerParams* peer) {
    int rc = arity_check(k, n_in, m_out);
    if (rc) return rc;
    if ((rc = dtype_check(dtype))) return rc;
    if (!out_adj || !in_adj || !in_shapes) return fail(BCAD_CU_ERR_CONFIG, "null argument array");
    const bool recompute = partials == nullptr;
    if (recompute) {
        if (!in) return fail(BCAD_CU_ERR_CONFIG, "recompute pullback needs the inputs");
        for (int j = 0; j < n_in; ++j)
            if (!in[j]) return fail(BCAD_CU_ERR_CONFIG, "null input pointer " + std::to_string(j));
    } else {
        for (int i = 0; i < m_out; ++i)
            for (int j = 0; j < n_in; ++j)
                if (out_adj[i] && in_adj[j] && !partials[i * n_in + j])
                    return fail(BCAD_CU_ERR_CONFIG, "null cached partial");
    }
    for (int j = 0; j < n_in; ++j)
        for (int l = 0; l < j; ++l)
            if (in_adj[j] && in_adj[j] == in_adj[l])
                return fail(BCAD_CU_ERR_CONFIG, "in_adj pointers must not alias");
    bool any_w = false, any_adj = false;
    for (int i = 0; i < m_out; ++i) any_w |= out_adj[i] != nullptr;
    for (int j = 0; j < n_in; ++j) any_adj |= in_adj[j] != nullptr;
    if (!any_w || !any_adj) return BCAD_CU_OK;  // tape.hpp:277-281: nothing flows
    Plan plan;
    std::string err;
    if ((rc = make_plan(n_in, in_shapes, &plan, &err))) return fail(rc, err);
    cudaStream_t s = static_cast<cudaStream_t>(stream);
    ErrorWord ew;
    const bool check = k->may_raise && recompute;
    if (check) {
        if ((rc = refuse_if_capturing(s, k->name)) || (rc = ew.acquire())) return rc;
        CU_TRY(cudaMemsetAsync(ew.get(), 0xff, sizeof(unsigned long long), s), "cudaMemsetAsync(error word)");
    }
    unsigned long long* word = ew.get();
    PullArgs a{dtype, out_adj, partials, in, in_adj, accumulate, workspace, workspace_bytes, s, word, &plan};
    a.peer = peer;
    a.tcount = count_slots_for_launch();
    if ((rc = k->pull(a, &err))) return fail(rc, err);
    if (check) return check_error_word(word, s, plan);
    return BCAD_CU_OK;
}
}  // namespace

int bcad_cu_scatter_add(int dtype, void* acc, const bcad_cu_shape* acc_shape, const void* contrib,
                        const bcad_cu_shape* contrib_shape, int zero_first, void* stream) {
    int rc = dtype_check(dtype);
    if (rc) return rc;
    const bcad_cu_shape both[2] = {*acc_shape, *contrib_shape};
    Plan plan;
    std::string err;
    if ((rc = make_plan(2, both, &plan, &err))) return fail(rc, err);
    cudaStream_t s = static_cast<cudaStream_t>(stream);
    const int64_t acc_vol = plan.arg_vol[0];
    if (acc_vol == plan.vol && plan.arg_vol[1] == plan.vol) {
        if (dtype == BCAD_CU_F32)
            add_same_kernel<float><<<grid_for(acc_vol), 256, 0, s>>>(static_cast<float*>(acc), static_cast<const float*>(contrib), acc_vol, zero_first != 0);
        else
            add_same_kernel<double><<<grid_for(acc_vol), 256, 0, s>>>(static_cast<double*>(acc), static_cast<const double*>(contrib), acc_vol, zero_first != 0);
    } else {
        ScatterGeom g{};
        g.rank = plan.out_rank;
        for (int k = 0; k < kMaxRank; ++k) {
            g.out_dims[k] = k < plan.out_rank ? plan.out_dims[k] : 1;
            g.acc_strides[k] = plan.strides[0][k];
            g.con_strides[k] = plan.strides[1][k];
        }
        g.acc_vol = acc_vol;
        if (dtype == BCAD_CU_F32)
            scatter_add_kernel<float><<<grid_for(acc_vol), 256, 0, s>>>(static_cast<float*>(acc), static_cast<const float*>(contrib), g, zero_first != 0);
        else
            scatter_add_kernel<double><<<grid_for(acc_vol), 256, 0, s>>>(static_cast<double*>(acc), static_cast<const double*>(contrib), g, zero_first != 0);
    }
    CU_TRY(cudaGetLastError(), "scatter_add launch");
    return BCAD_CU_OK;
}

int bcad_cu_fill(int dtype, void* ptr, int64_t count, double value, void* stream) {
    int rc = dtype_check(dtype);
    if (rc) return rc;
    if (count <= 0) return BCAD_CU_OK;
    cudaStream_t s = static_cast<cudaStream_t>(stream);
    if (dtype == BCAD_CU_F32) fill_kernel<float><<<grid_for(count), 256, 0, s>>>(static_cast<float*>(ptr), count, float(value));
    else fill_kernel<double><<<grid_for(count), 256, 0, s>>>(static_cast<double*>(ptr), count, value);
    CU_TRY(cudaGetLastError(), "fill launch");
    return BCAD_CU_OK;
}

// ------------------------------------------------------- device / memory
int bcad_cu_device_count(int* count) {
    CU_TRY(cudaGetDeviceCount(count), "cudaGetDeviceCount");
    return BCAD_CU_OK;
}
int bcad_cu_set_device(int device) {
    CU_TRY(cudaSetDevice(device), "cudaSetDevice");
    return BCAD_CU_OK;
}
int bcad_cu_get_device(int* device) {
    CU_TRY(cudaGetDevice(device), "cudaGetDevice");
    return BCAD_CU_OK;
}

int bcad_cu_malloc(void** ptr, size_t bytes, void* stream) {
    static std::once_flag pools_once[kMaxDevices];
    int dev = 0;
    CU_TRY(cudaGetDevice(&dev), "cudaGetDevice");
    if (dev >= 0 && dev < kMaxDevices)
        std::call_once(pools_once[dev], [dev] {
            cudaMemPool_t pool;
            if (cudaDeviceGetDefaultMemPool(&pool, dev) == cudaSuccess) {
                uint64_t threshold = UINT64_MAX;  // keep freed blocks cached
                cudaMemPoolSetAttribute(pool, cudaMemPoolAttrReleaseThreshold, &threshold);
            }
        });
    CU_TRY(cudaMallocAsync(ptr, bytes == 0 ? 1 : bytes, static_cast<cudaStream_t>(stream)), "cudaMallocAsync");
    return BCAD_CU_OK;
}
int bcad_cu_free(void* ptr, void* stream) {
    if (!ptr) return BCAD_CU_OK;
    CU_TRY(cudaFreeAsync(ptr, static_cast<cudaStream_t>(stream)), "cudaFreeAsync");
    return BCAD_CU_OK;
}
int bcad_cu_host_alloc(void** ptr, size_t bytes) {
    CU_TRY(cudaMallocHost(ptr, bytes == 0 ? 1 : bytes), "cudaMallocHost");
    return BCAD_CU_OK;
}
int bcad_cu_host_free(void* ptr) {
    if (!ptr) return BCAD_CU_OK;
    CU_TRY(cudaFreeHost(ptr), "cudaFreeHost");
    return BCAD_CU_OK;
}
int bcad_cu_host_is_pinned(const void* ptr) {
    cudaPointerAttributes at{};
    const bool pinned = cudaPointerGetAttributes(&at, ptr) == cudaSuccess && at.type == cudaMemoryTypeHost;
    (void)cudaGetLastError();
    return pinned ? 1 : 0;
}
int bcad_cu_memcpy(void* dst, const void* src, size_t bytes, int kind, void* stream) {
    if (bytes == 0) return BCAD_CU_OK;
    const cudaMemcpyKind k = kind == 0 ? cudaMemcpyHostToDevice : kind == 1 ? cudaMemcpyDeviceToHost : cudaMemcpyDeviceToDevice;
    CU_TRY(cudaMemcpyAsync(dst, src, bytes, k, static_cast<cudaStream_t>(stream)), "cudaMemcpyAsync");
    return BCAD_CU_OK;
}
int bcad_cu_memcpy_batch(size_t n, void* const* dsts, const void* const* srcs, const size_t* sizes, int kind,
                         void* stream) {
    cudaStream_t s = static_cast<cudaStream_t>(stream);
    if (kind < 0 || kind > 2) return fail(BCAD_CU_ERR_CONFIG, "memcpy kind must be 0, 1 or 2");
    std::vector<void*> d;
    std::vector<void*> sr;
    std::vector<size_t> sz;
    for (size_t k = 0; k < n; ++k)
        if (sizes[k]) {
            d.push_back(dsts[k]);
            sr.push_back(const_cast<void*>(srcs[k]));
            sz.push_back(sizes[k]);
        }
    if (d.empty()) return BCAD_CU_OK;
    if (kind == 2) {  // device copies on the SMs, kCopyBatch buffers per launch
        for (size_t k0 = 0; k0 < d.size(); k0 += kCopyBatch) {
            CopyBatchDesc desc{};
            const int m = int(std::min<size_t>(kCopyBatch, d.size() - k0));
            size_t most = 0;
            for (int k = 0; k < m; ++k) {
                desc.dst[k] = static_cast<char*>(d[k0 + k]);
                desc.src[k] = static_cast<const char*>(sr[k0 + k]);
                desc.bytes[k] = sz[k0 + k];
                most = std::max(most, sz[k0 + k]);
            }
            const size_t chunks = (most + 16 * 256 - 1) / (16 * 256);
            const unsigned gx = unsigned(std::max<size_t>(1, std::min<size_t>(chunks, std::max(1, 148 * 8 / m))));
            copy_batch_kernel<<<dim3(gx, unsigned(m)), 256, 0, s>>>(desc);
            CU_TRY(cudaGetLastError(), "copy_batch_kernel");
        }
        return BCAD_CU_OK;
    }
    cudaStreamCaptureStatus cap = cudaStreamCaptureStatusNone;
    if (s != nullptr && cudaStreamIsCapturing(s, &cap) != cudaSuccess) (void)cudaGetLastError();
    // The batch path is for pinned host memory; pageable buffers (which the
    // driver stages, and would otherwise lock page by page) go one by one.
    bool pinned = cap == cudaStreamCaptureStatusNone;
    for (size_t k = 0; k < d.size() && pinned; ++k) {
        cudaPointerAttributes at{};
        const void* host = kind == 0 ? sr[k] : d[k];
        if (cudaPointerGetAttributes(&at, host) != cudaSuccess || at.type != cudaMemoryTypeHost) pinned = false;
        (void)cudaGetLastError();
    }
    // legacy stream (rejected by the batch API), pageable memory, or a graph
    // capture (plain copy nodes; the per-call host cost is paid once)
    if (s == nullptr || d.size() == 1 || !pinned || cap != cudaStreamCaptureStatusNone) {
        for (size_t k = 0; k < d.size(); ++k)
            CU_TRY(cudaMemcpyAsync(d[k], sr[k], sz[k], kind == 0 ? cudaMemcpyHostToDevice : cudaMemcpyDeviceToHost, s),
                   "cudaMemcpyAsync");
        return BCAD_CU_OK;
    }
    cudaMemcpyAttributes attr{};
    attr.srcAccessOrder = cudaMemcpySrcAccessOrderStream;
    size_t first = 0, fail_idx = 0;
    if (cudaMemcpyBatchAsync(d.data(), sr.data(), sz.data(), d.size(), &attr, &first, 1, &fail_idx, s) != cudaSuccess) {
        (void)cudaGetLastError();  // an operand the batch path rejects: one call per copy instead
        for (size_t k = 0; k < d.size(); ++k)
            CU_TRY(cudaMemcpyAsync(d[k], sr[k], sz[k], kind == 0 ? cudaMemcpyHostToDevice : cudaMemcpyDeviceToHost, s),
                   "cudaMemcpyAsync");
    }
    return BCAD_CU_OK;
}
int bcad_cu_memset(void* ptr, int value, size_t bytes, void* stream) {
    if (bytes == 0) return BCAD_CU_OK;
    CU_TRY(cudaMemsetAsync(ptr, value, bytes, static_cast<cudaStream_t>(stream)), "cudaMemsetAsync");
    return BCAD_CU_OK;
}
int bcad_cu_stream_create(void** stream) {
    cudaStream_t s;
    CU_TRY(cudaStreamCreateWithFlags(&s, cudaStreamNonBlocking), "cudaStreamCreate");
    *stream = s;
    return BCAD_CU_OK;
}
int bcad_cu_stream_destroy(void* stream) {
    if (!stream) return BCAD_CU_OK;
    CU_TRY(cudaStreamDestroy(static_cast<cudaStream_t>(stream)), "cudaStreamDestroy");
    return BCAD_CU_OK;
}
int bcad_cu_stream_synchronize(void* stream) {
    CU_TRY(cudaStreamSynchronize(static_cast<cudaStream_t>(stream)), "cudaStreamSynchronize");
    return BCAD_CU_OK;
}
int bcad_cu_device_synchronize(void) {
    CU_TRY(cudaDeviceSynchronize(), "cudaDeviceSynchronize");
    return BCAD_CU_OK;
}
int bcad_cu_event_create(void** event) {
    cudaEvent_t e;
    CU_TRY(cudaEventCreateWithFlags(&e, cudaEventDisableTiming), "cudaEventCreate");
    *event = e;
    return BCAD_CU_OK;
}
int bcad_cu_event_destroy(void* event) {
    if (!event) return BCAD_CU_OK;
    CU_TRY(cudaEventDestroy(static_cast<cudaEvent_t>(event)), "cudaEventDestroy");
    return BCAD_CU_OK;
}
int bcad_cu_event_record(void* event, void* stream) {
    CU_TRY(cudaEventRecord(static_cast<cudaEvent_t>(event), static_cast<cudaStream_t>(stream)), "cudaEventRecord");
    return BCAD_CU_OK;
}
int bcad_cu_graph_capture_begin(void* stream) {
    CU_TRY(cudaStreamBeginCapture(static_cast<cudaStream_t>(stream), cudaStreamCaptureModeThreadLocal),
           "cudaStreamBeginCapture");
    return BCAD_CU_OK;
}
int bcad_cu_graph_capture_end(void* stream, void** graph_exec) {
    cudaGraph_t g = nullptr;
    CU_TRY(cudaStreamEndCapture(static_cast<cudaStream_t>(stream), &g), "cudaStreamEndCapture");
    cudaGraphExec_t e = nullptr;
    const cudaError_t rc = cudaGraphInstantiate(&e, g, 0);
    cudaGraphDestroy(g);
    CU_TRY(rc, "cudaGraphInstantiate");
    *graph_exec = e;
    return BCAD_CU_OK;
}
int bcad_cu_graph_launch(void* graph_exec, void* stream) {
    CU_TRY(cudaGraphLaunch(static_cast<cudaGraphExec_t>(graph_exec), static_cast<cudaStream_t>(stream)),
           "cudaGraphLaunch");
    return BCAD_CU_OK;
}
int bcad_cu_graph_destroy(void* graph_exec) {
    if (!graph_exec) return BCAD_CU_OK;
    CU_TRY(cudaGraphExecDestroy(static_cast<cudaGraphExec_t>(graph_exec)), "cudaGraphExecDestroy");
    return BCAD_CU_OK;
}
int bcad_cu_stream_wait_event(void* stream, void* event) {
    CU_TRY(cudaStreamWaitEvent(static_cast<cudaStream_t>(stream), static_cast<cudaEvent_t>(event), 0),
           "cudaStreamWaitEvent");
    return BCAD_CU_OK;
}

// ------------------------------------------------------ peer groups
// One buffer per rank, exported by CUDA IPC and mapped by every other rank
// (ranks in the same process pass the raw pointer). Layout (PeerParams):
// slots [2][world][n] fp64 | flags [world] u64 | step counter u64 | arrival u32.
struct bcad_cu_peer_group_s {
    int rank = 0, world = 0, device = 0;
    size_t n = 0;
    void* buf = nullptr;  // this rank's buffer
    std::vector<void*> opened;  // peers' buffers mapped by IPC (closed on destroy)
    PeerParams params{};
    bool connected = false;
};

namespace {
struct PeerHandle {  // BCAD_CU_PEER_HANDLE_BYTES, rank-order array in connect
    uint64_t magic;
    int32_t pid, device;
    uint64_t ptr, n, world;
    cudaIpcMemHandle_t ipc;
};
static_assert(sizeof(PeerHandle) <= BCAD_CU_PEER_HANDLE_BYTES, "peer handle blob too small");
constexpr uint64_t kPeerMagic = 0x62636164'70656572ull;  // "bcadpeer"

size_t peer_bytes(int world, size_t n) { return (2 * size_t(world) * n + world + 2) * 8; }

void peer_pointers(void* base, int world, size_t n, double** slots, unsigned long long** flags,
                   unsigned long long** epoch, unsigned int** arrive) {
    char* b = static_cast<char*>(base);
    *slots = reinterpret_cast<double*>(b);
    *flags = reinterpret_cast<unsigned long long*>(b + 2 * size_t(world) * n * 8);
    *epoch = *flags + world;
    *arrive = reinterpret_cast<unsigned int*>(*epoch + 1);
}
}  // namespace

int bcad_cu_peer_group_create(int rank, int world, size_t max_elems, bcad_cu_peer_group* out,
                              unsigned char handle[BCAD_CU_PEER_HANDLE_BYTES]) {
    if (!out || !handle) return fail(BCAD_CU_ERR_CONFIG, "null argument");
    if (world < 1 || world > kMaxPeers || rank < 0 || rank >= world)
        return fail(BCAD_CU_ERR_CONFIG, "peer group: rank / world outside [0, world) / [1, 8]");
    if (max_elems < 1) return fail(BCAD_CU_ERR_CONFIG, "peer group: max_elems must be >= 1");
    auto* g = new bcad_cu_peer_group_s();
    g->rank = rank;
    g->world = world;
    g->n = max_elems;
    if (cudaGetDevice(&g->device) != cudaSuccess || cudaMalloc(&g->buf, peer_bytes(world, max_elems)) != cudaSuccess ||
        cudaMemset(g->buf, 0, peer_bytes(world, max_elems)) != cudaSuccess || cudaDeviceSynchronize() != cudaSuccess) {
        const cudaError_t e = cudaGetLastError();
        if (g->buf) cudaFree(g->buf);
        delete g;
        return cuda_fail(e, "peer group buffer");
    }
    PeerHandle h{};
    h.magic = kPeerMagic;
    h.pid = int32_t(getpid());
    h.device = g->device;
    h.ptr = reinterpret_cast<uint64_t>(g->buf);
    h.n = max_elems;
    h.world = uint64_t(world);
    if (cudaIpcGetMemHandle(&h.ipc, g->buf) != cudaSuccess) {
        const cudaError_t e = cudaGetLastError();
        cudaFree(g->buf);
        delete g;
        return cuda_fail(e, "cudaIpcGetMemHandle");
    }
    std::memset(handle, 0, BCAD_CU_PEER_HANDLE_BYTES);
    std::memcpy(handle, &h, sizeof(h));
    *out = g;
    return BCAD_CU_OK;
}

int bcad_cu_peer_group_connect(bcad_cu_peer_group g, const unsigned char* handles) {
    if (!g || !handles) return fail(BCAD_CU_ERR_CONFIG, "null argument");
    if (g->connected) return fail(BCAD_CU_ERR_CONFIG, "peer group already connected");
    PeerParams& q = g->params;
    q = PeerParams{};
    q.rank = g->rank;
    q.world = g->world;
    q.n = int64_t(g->n);
    for (int k = 0; k < g->world; ++k) {
        PeerHandle h;
        std::memcpy(&h, handles + size_t(k) * BCAD_CU_PEER_HANDLE_BYTES, sizeof(h));
        if (h.magic != kPeerMagic || h.world != uint64_t(g->world) || h.n != g->n)
            return fail(BCAD_CU_ERR_CONFIG, "peer handle " + std::to_string(k) + " is not from a group of the same world / size");
        void* base = nullptr;
        if (k == g->rank) {
            base = g->buf;
        } else if (h.pid == int32_t(getpid())) {
            base = reinterpret_cast<void*>(h.ptr);  // a rank in this process
        } else {
            CU_TRY(cudaIpcOpenMemHandle(&base, h.ipc, cudaIpcMemLazyEnablePeerAccess), "cudaIpcOpenMemHandle");
            g->opened.push_back(base);
        }
        double* slots;
        unsigned long long *flags, *epoch;
        unsigned int* arrive;
        peer_pointers(base, g->world, g->n, &slots, &flags, &epoch, &arrive);
        q.slots[k] = slots;
        q.flags[k] = flags;
        if (k == g->rank) {
            q.epoch = epoch;
            q.arrive = arrive;
        }
    }
    g->connected = true;
    return BCAD_CU_OK;
}

int bcad_cu_peer_group_destroy(bcad_cu_peer_group g) {
    if (!g) return BCAD_CU_OK;
    for (void* p : g->opened) cudaIpcCloseMemHandle(p);
    if (g->buf) cudaFree(g->buf);
    delete g;
    return BCAD_CU_OK;
}

int bcad_cu_pullback_allreduce(bcad_cu_kernel k, int dtype, int n_in, const bcad_cu_shape* in_shapes, int m_out,
                               const void* const* out_adj, const void* const* partials, const void* const* in,
                               void* const* in_adj, const unsigned char* accumulate, void* workspace,
                               size_t workspace_bytes, bcad_cu_peer_group group, void* stream) {
    if (!group || !group->connected) return fail(BCAD_CU_ERR_CONFIG, "peer group not connected");
    return pullback_impl(k, dtype, n_in, in_shapes, m_out, out_adj, partials, in, in_adj, accumulate, workspace,
                         workspace_bytes, stream, &group->params);
}

// ------------------------------------------------------------------ NCCL
int bcad_cu_nccl_unique_id(unsigned char id[128]) {
    Nccl& n = nccl();
    if (!n.ok) return fail(BCAD_CU_ERR_NCCL, "libnccl.so.2 not loadable");
    NcclUniqueId u;
    const int r = n.GetUniqueId(&u);
    if (r) return nccl_fail(r, "ncclGetUniqueId");
    std::memcpy(id, u.internal, 128);
    return BCAD_CU_OK;
}

int bcad_cu_comm_init(void** comm, int nranks, const unsigned char id[128], int rank) {
    Nccl& n = nccl();
    if (!n.ok) return fail(BCAD_CU_ERR_NCCL, "libnccl.so.2 not loadable");
    NcclUniqueId u;
    std::memcpy(u.internal, id, 128);
    // ncclCommInitRank takes the id by value: call through the by-value type.
    auto init = reinterpret_cast<int (*)(void**, int, NcclUniqueId, int)>(n.CommInitRank);
    const int r = init(comm, nranks, u, rank);
    if (r) return nccl_fail(r, "ncclCommInitRank");
    return BCAD_CU_OK;
}

int bcad_cu_comm_destroy(void* comm) {
    Nccl& n = nccl();
    if (!n.ok) return fail(BCAD_CU_ERR_NCCL, "libnccl.so.2 not loadable");
    if (!comm) return BCAD_CU_OK;
    const int r = n.CommDestroy(comm);
    if (r) return nccl_fail(r, "ncclCommDestroy");
    return BCAD_CU_OK;
}

int bcad_cu_comm_count(void* comm, int* nranks) {
    Nccl& n = nccl();
    if (!n.ok || !n.CommCount) return fail(BCAD_CU_ERR_NCCL, "libnccl.so.2 not loadable");
    const int r = n.CommCount(comm, nranks);
    if (r) return nccl_fail(r, "ncclCommCount");
    return BCAD_CU_OK;
}

int bcad_cu_allreduce_adjoints(void* const* bufs, const size_t* counts, int n_bufs, int dtype, void* comm,
                               void* stream) {
    int rc = dtype_check(dtype);
    if (rc) return rc;
    Nccl& n = nccl();
    if (!n.ok) return fail(BCAD_CU_ERR_NCCL, "libnccl.so.2 not loadable");
    const int nccl_type = dtype == BCAD_CU_F32 ? 7 : 8;  // ncclFloat32 / ncclFloat64
    int r = n.GroupStart();
    if (r) return nccl_fail(r, "ncclGroupStart");
    for (int b = 0; b < n_bufs; ++b) {
        if (!bufs[b] || counts[b] == 0) continue;
        r = n.AllReduce(bufs[b], bufs[b], counts[b], nccl_type, /*ncclSum*/ 0, comm, static_cast<cudaStream_t>(stream));
        if (r) {
            n.GroupEnd();
            return nccl_fail(r, "ncclAllReduce");
        }
    }
    r = n.GroupEnd();
    if (r) return nccl_fail(r, "ncclGroupEnd");
    return BCAD_CU_OK;
}

}  // extern "C"
