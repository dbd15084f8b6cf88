// Config-2 memory floor probes (dev harness, not the product): where do the
// ~12 us of a copy kernel with K1's exact access pattern go, and do 1-D bulk
// copies (cp.async.bulk, the TMA's non-tensor form) beat LDG/STG there?
// K1's pattern at config 2 (canonical HM-LSTM, 1024 x 1024 fp32): read c, f,
// i, g (4 x 4 MiB) + z1, z2 (2 x 4 KiB), write 7 x 4 MiB. L2 flushed before
// every timed launch exactly like scripts/lab/lab.cu (1 GiB write + read).
// One JSON object per line.
#include <cuda_runtime.h>

#include <cstdint>

#include <algorithm>
#include <cstdio>
#include <cstdlib>
#include <functional>
#include <vector>

#define CK(x)                                                                                          \
    do {                                                                                               \
        cudaError_t e_ = (x);                                                                          \
        if (e_ != cudaSuccess) {                                                                       \
            std::fprintf(stderr, "%s:%d %s: %s\n", __FILE__, __LINE__, #x, cudaGetErrorString(e_));    \
            std::exit(1);                                                                              \
        }                                                                                              \
    } while (0)

constexpr int R = 1024, C = 1024;  // rows, cols
constexpr size_t E = size_t(R) * C;

__global__ void read_kernel(const float4* p, size_t n, float* out) {
    float s = 0.f;
    for (size_t i = blockIdx.x * size_t(blockDim.x) + threadIdx.x; i < n; i += size_t(gridDim.x) * blockDim.x) {
        const float4 v = __ldcs(p + i);
        s += v.x + v.y + v.z + v.w;
    }
    if (s == 1234.5f) *out = s;
}

struct Outs { float4* o[7]; };
struct Ins { const float4* x[4]; const float* z1; const float* z2; };

__global__ void empty_kernel(int* p) {
    if (p && threadIdx.x == 1023) *p = 0;
}

// read only: 4 streams + z
__global__ void read4_kernel(Ins in, float* sink) {
    const size_t k = blockIdx.x * size_t(blockDim.x) + threadIdx.x;
    if (k >= E / 4) return;
    const size_t r = k / (C / 4);
    const float a = __ldg(in.z1 + r) + __ldg(in.z2 + r);
    float4 s = __ldcs(in.x[0] + k), t = __ldcs(in.x[1] + k), u = __ldcs(in.x[2] + k), v = __ldcs(in.x[3] + k);
    const float q = s.x + t.y + u.z + v.w + a;
    if (q == 1234.5f) *sink = q;
}

// write only: 7 streams
__global__ void write7_kernel(Outs out) {
    const size_t k = blockIdx.x * size_t(blockDim.x) + threadIdx.x;
    if (k >= E / 4) return;
    const float a = float(k);
#pragma unroll
    for (int t = 0; t < 7; ++t) out.o[t][k] = make_float4(a, a + t, a, a);
}

// LDG/STG copy, one vector per thread (1024 CTAs) or two rows per thread (512)
template <int RPT>
__global__ void copy_kernel(Ins in, Outs out) {
    const int tid = threadIdx.x;
    const size_t r0 = size_t(blockIdx.x) * RPT;
#pragma unroll
    for (int k = 0; k < RPT; ++k) {
        const size_t r = r0 + k;
        const size_t i = r * (C / 4) + tid;
        const float a = __ldg(in.z1 + r) + __ldg(in.z2 + r);
        float4 x = __ldcs(in.x[0] + i), y = __ldcs(in.x[1] + i), u = __ldcs(in.x[2] + i), w = __ldcs(in.x[3] + i);
        out.o[0][i] = make_float4(x.x + a, x.y, x.z, x.w);
        out.o[1][i] = make_float4(y.x + a, y.y, y.z, y.w);
        out.o[2][i] = make_float4(u.x, u.y + a, u.z, u.w);
        out.o[3][i] = make_float4(w.x, w.y, w.z + a, w.w);
        out.o[4][i] = make_float4(a, a, a, a);
        out.o[5][i] = make_float4(a, 0, a, 0);
        out.o[6][i] = make_float4(x.x + a, x.y, x.z, x.w);
    }
}

// --------------------------------------------------------- bulk-copy forms
__device__ __forceinline__ uint32_t smem_u32(const void* p) {
    return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ void mbar_init(uint64_t* bar, int count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count));
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
}
__device__ __forceinline__ void mbar_expect_tx(uint64_t* bar, uint32_t bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)), "r"(bytes) : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t phase) {
    asm volatile(
        "{\n .reg .pred p;\n"
        "W: mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n"
        " @!p bra W;\n}\n" ::"r"(smem_u32(bar)),
        "r"(phase)
        : "memory");
}
__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, uint32_t bytes, uint64_t* bar) {
    asm volatile("cp.async.bulk.shared::cta.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(smem_u32(dst)),
                 "l"(src), "r"(bytes), "r"(smem_u32(bar))
                 : "memory");
}
__device__ __forceinline__ void bulk_s2g(void* dst, const void* src, uint32_t bytes) {
    asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], %2;" ::"l"(dst), "r"(smem_u32(src)), "r"(bytes)
                 : "memory");
}
__device__ __forceinline__ void bulk_commit() { asm volatile("cp.async.bulk.commit_group;" ::: "memory"); }
__device__ __forceinline__ void bulk_wait_read0() { asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory"); }
__device__ __forceinline__ void fence_proxy_async() { asm volatile("fence.proxy.async.shared::cta;" ::: "memory"); }
__device__ __forceinline__ void prefetch_l2_bulk(const void* p, uint32_t bytes) {
    asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(p), "r"(bytes) : "memory");
}

// One CTA per row (1024 CTAs x 256 threads, 4 floats each). BULK_IN: the 4
// input rows (4 x 4 KiB) arrive by cp.async.bulk into shared memory;
// BULK_OUT: the 7 output rows are staged in shared memory and leave by
// cp.async.bulk stores. Either side falls back to LDG / STG.
template <bool BULK_IN, bool BULK_OUT>
__global__ void bulk_row_kernel(Ins in, Outs out) {
    extern __shared__ __align__(128) float4 sm[];
    __shared__ __align__(8) uint64_t bar;
    float4* sin = sm;                          // 4 x 256 float4
    float4* sout = sm + (BULK_IN ? 4 * 256 : 0);  // 7 x 256 float4
    const int tid = threadIdx.x;
    const size_t r = blockIdx.x;
    const size_t i = r * (C / 4) + tid;
    if constexpr (BULK_IN) {
        if (tid == 0) {
            mbar_init(&bar, 1);
            mbar_expect_tx(&bar, 4 * C * 4);
#pragma unroll
            for (int s = 0; s < 4; ++s) bulk_g2s(sin + s * 256, in.x[s] + r * (C / 4), C * 4, &bar);
        }
        __syncthreads();
    }
    const float a = __ldg(in.z1 + r) + __ldg(in.z2 + r);
    float4 x, y, u, w;
    if constexpr (BULK_IN) {
        mbar_wait(&bar, 0);
        x = sin[tid]; y = sin[256 + tid]; u = sin[512 + tid]; w = sin[768 + tid];
    } else {
        x = __ldcs(in.x[0] + i); y = __ldcs(in.x[1] + i); u = __ldcs(in.x[2] + i); w = __ldcs(in.x[3] + i);
    }
    float4 o[7] = {make_float4(x.x + a, x.y, x.z, x.w), make_float4(y.x + a, y.y, y.z, y.w),
                   make_float4(u.x, u.y + a, u.z, u.w), make_float4(w.x, w.y, w.z + a, w.w),
                   make_float4(a, a, a, a), make_float4(a, 0, a, 0), make_float4(x.x + a, x.y, x.z, x.w)};
    if constexpr (BULK_OUT) {
#pragma unroll
        for (int t = 0; t < 7; ++t) sout[t * 256 + tid] = o[t];
        fence_proxy_async();
        __syncthreads();
        if (tid < 7) {
            bulk_s2g(out.o[tid] + r * (C / 4), sout + tid * 256, C * 4);
            bulk_commit();
            bulk_wait_read0();
        }
    } else {
#pragma unroll
        for (int t = 0; t < 7; ++t) out.o[t][i] = o[t];
    }
}

// L2 bulk prefetch of the CTA's input rows at entry, then the LDG/STG copy.
__global__ void prefetch_copy_kernel(Ins in, Outs out) {
    const int tid = threadIdx.x;
    const size_t r = blockIdx.x;
    if (tid < 4) prefetch_l2_bulk(in.x[tid] + r * (C / 4), C * 4);
    const size_t i = r * (C / 4) + tid;
    const float a = __ldg(in.z1 + r) + __ldg(in.z2 + r);
    float4 x = __ldcs(in.x[0] + i), y = __ldcs(in.x[1] + i), u = __ldcs(in.x[2] + i), w = __ldcs(in.x[3] + i);
    out.o[0][i] = make_float4(x.x + a, x.y, x.z, x.w);
    out.o[1][i] = make_float4(y.x + a, y.y, y.z, y.w);
    out.o[2][i] = make_float4(u.x, u.y + a, u.z, u.w);
    out.o[3][i] = make_float4(w.x, w.y, w.z + a, w.w);
    out.o[4][i] = make_float4(a, a, a, a);
    out.o[5][i] = make_float4(a, 0, a, 0);
    out.o[6][i] = make_float4(x.x + a, x.y, x.z, x.w);
}

struct Flush {
    float* buf = nullptr;
    float* sink = nullptr;
    size_t n = size_t(256) << 20;  // 1 GiB of floats
    Flush() {
        CK(cudaMalloc(&buf, n * 4));
        CK(cudaMalloc(&sink, 4));
    }
    void operator()(cudaStream_t s) {
        CK(cudaMemsetAsync(buf, 1, n * 4, s));
        read_kernel<<<148 * 8, 256, 0, s>>>(reinterpret_cast<const float4*>(buf), n / 4, sink);
    }
};

static cudaStream_t g_s;
static Flush* g_flush;

static double time_us(const std::function<void()>& fn, bool flush = true, int reps = 101) {
    std::vector<cudaEvent_t> a(reps), b(reps);
    for (int k = 0; k < reps; ++k) {
        CK(cudaEventCreate(&a[k]));
        CK(cudaEventCreate(&b[k]));
    }
    for (int k = 0; k < 3; ++k) {
        if (flush) (*g_flush)(g_s);
        fn();
    }
    for (int k = 0; k < reps; ++k) {
        if (flush) (*g_flush)(g_s);
        CK(cudaEventRecord(a[k], g_s));
        fn();
        CK(cudaEventRecord(b[k], g_s));
    }
    CK(cudaStreamSynchronize(g_s));
    CK(cudaGetLastError());
    std::vector<float> ms(reps);
    for (int k = 0; k < reps; ++k) CK(cudaEventElapsedTime(&ms[k], a[k], b[k]));
    std::sort(ms.begin(), ms.end());
    for (int k = 0; k < reps; ++k) {
        CK(cudaEventDestroy(a[k]));
        CK(cudaEventDestroy(b[k]));
    }
    // event timestamps advance in 2.048 us steps here: the mean of the
    // phase-randomised samples (outliers > 2x median dropped) is unbiased
    const float med = ms[reps / 2];
    double s = 0;
    int n = 0;
    for (float v : ms)
        if (v <= 2 * med) { s += v; ++n; }
    return s / n * 1e3;
}

int main() {
    CK(cudaSetDevice(0));
    CK(cudaStreamCreateWithFlags(&g_s, cudaStreamNonBlocking));
    g_flush = new Flush();
    Ins in{};
    Outs out{};
    for (int s = 0; s < 4; ++s) {
        float4* p;
        CK(cudaMalloc(&p, E * 4));
        CK(cudaMemset(p, 0, E * 4));
        in.x[s] = p;
    }
    float *z1, *z2, *sink;
    CK(cudaMalloc(&z1, R * 4));
    CK(cudaMalloc(&z2, R * 4));
    CK(cudaMalloc(&sink, 4));
    CK(cudaMemset(z1, 0, R * 4));
    CK(cudaMemset(z2, 0, R * 4));
    in.z1 = z1;
    in.z2 = z2;
    for (int t = 0; t < 7; ++t) CK(cudaMalloc(&out.o[t], E * 4));
    const double k1_bytes = double(E) * 4 * 11 + 2.0 * R * 4;
    auto emit = [&](const char* v, double us, bool flush) {
        std::printf("{\"exp\": \"floor_cfg2\", \"variant\": \"%s\", \"flush\": %d, \"us\": %.3f, \"k1_GBps\": %.1f}\n", v,
                    int(flush), us, k1_bytes / (us * 1e-6) / 1e9);
        std::fflush(stdout);
    };
    const size_t sm_in = 4 * 256 * 16, sm_out = 7 * 256 * 16;
    CK(cudaFuncSetAttribute(bulk_row_kernel<true, true>, cudaFuncAttributeMaxDynamicSharedMemorySize, int(sm_in + sm_out)));
    for (int blocks : {1, 148, 296, 592, 1024, 2048})
        for (int threads : {32, 256}) {
            const double us = time_us([&] { empty_kernel<<<blocks, threads, 0, g_s>>>(nullptr); }, true);
            std::printf("{\"exp\": \"empty_grid\", \"blocks\": %d, \"threads\": %d, \"flush\": 1, \"us\": %.3f}\n",
                        blocks, threads, us);
            std::fflush(stdout);
        }
    for (int rep = 0; rep < 2; ++rep)
        for (bool flush : {true, false}) {
            emit("empty_1024x256", time_us([&] { empty_kernel<<<1024, 256, 0, g_s>>>(nullptr); }, flush), flush);
            emit("read4_only", time_us([&] { read4_kernel<<<1024, 256, 0, g_s>>>(in, sink); }, flush), flush);
            emit("write7_only", time_us([&] { write7_kernel<<<1024, 256, 0, g_s>>>(out); }, flush), flush);
            emit("copy_ldg_1row", time_us([&] { copy_kernel<1><<<1024, 256, 0, g_s>>>(in, out); }, flush), flush);
            emit("copy_ldg_2rows", time_us([&] { copy_kernel<2><<<512, 256, 0, g_s>>>(in, out); }, flush), flush);
            emit("prefetch_l2_bulk_then_ldg", time_us([&] { prefetch_copy_kernel<<<1024, 256, 0, g_s>>>(in, out); }, flush),
                 flush);
            emit("bulk_in_stg_out",
                 time_us([&] { bulk_row_kernel<true, false><<<1024, 256, sm_in, g_s>>>(in, out); }, flush), flush);
            emit("ldg_in_bulk_out",
                 time_us([&] { bulk_row_kernel<false, true><<<1024, 256, sm_out, g_s>>>(in, out); }, flush), flush);
            emit("bulk_in_bulk_out",
                 time_us([&] { bulk_row_kernel<true, true><<<1024, 256, sm_in + sm_out, g_s>>>(in, out); }, flush),
                 flush);
        }
    return 0;
}
