// Dev probe: host-side cost of the CUDA runtime calls the tape path issues.
#include <chrono>
#include <cstdio>
#include <vector>
#include <cuda_runtime.h>

__global__ void noop(float* p) { if (p && threadIdx.x == 1234567) p[0] = 1.f; }

template <class F>
double per_call_us(F f, int n) {
    f();
    cudaDeviceSynchronize();
    auto t0 = std::chrono::steady_clock::now();
    for (int i = 0; i < n; ++i) f();
    auto t1 = std::chrono::steady_clock::now();
    cudaDeviceSynchronize();
    return std::chrono::duration<double, std::micro>(t1 - t0).count() / n;
}

int main() {
    cudaStream_t s;
    cudaStreamCreateWithFlags(&s, cudaStreamNonBlocking);
    cudaMemPool_t pool;
    cudaDeviceGetDefaultMemPool(&pool, 0);
    unsigned long long thr = ~0ull;
    cudaMemPoolSetAttribute(pool, cudaMemPoolAttrReleaseThreshold, &thr);
    void *a, *b;
    cudaMalloc(&a, 4 << 20);
    cudaMalloc(&b, 4 << 20);
    std::vector<void*> ptrs(64);
    printf("{\"mallocAsync+freeAsync_4MB_us\": %.2f,\n", per_call_us([&] {
        void* p; cudaMallocAsync(&p, 4 << 20, s); cudaFreeAsync(p, s); }, 2000));
    printf(" \"mallocAsync_x32_then_free_us_per_pair\": %.2f,\n", per_call_us([&] {
        for (int k = 0; k < 32; ++k) cudaMallocAsync(&ptrs[k], (4 << 20) + k * 256, s);
        for (int k = 0; k < 32; ++k) cudaFreeAsync(ptrs[k], s); }, 200) / 32);
    printf(" \"memcpyAsync_D2D_4MB_us\": %.2f,\n", per_call_us([&] { cudaMemcpyAsync(b, a, 4 << 20, cudaMemcpyDeviceToDevice, s); }, 200));
    printf(" \"memcpyAsync_D2D_64B_us\": %.2f,\n", per_call_us([&] { cudaMemcpyAsync(b, a, 64, cudaMemcpyDeviceToDevice, s); }, 2000));
    printf(" \"launch_noop_us\": %.2f,\n", per_call_us([&] { noop<<<1, 32, 0, s>>>(nullptr); }, 5000));
    printf(" \"memsetAsync_us\": %.2f,\n", per_call_us([&] { cudaMemsetAsync(b, 0, 256, s); }, 2000));
    cudaEvent_t e;
    cudaEventCreateWithFlags(&e, cudaEventDisableTiming);
    printf(" \"eventRecord_us\": %.2f,\n", per_call_us([&] { cudaEventRecord(e, s); }, 5000));
    printf(" \"streamSync_idle_us\": %.2f,\n", per_call_us([&] { cudaStreamSynchronize(s); }, 2000));
    {
        std::vector<void*> d(7), sr(7);
        std::vector<size_t> sz(7, 1 << 20);
        void* big; cudaMalloc(&big, 16 << 20);
        void* hbig; cudaMallocHost(&hbig, 16 << 20);
        for (int k = 0; k < 7; ++k) { d[k] = (char*)big + (k << 20); sr[k] = (char*)hbig + (k << 20); }
        cudaMemcpyAttributes at{};
        at.srcAccessOrder = cudaMemcpySrcAccessOrderStream;
        size_t idx = 0, fail = 0;
        printf(" \"memcpyBatchAsync_7xH2D_1MB_us_per_call\": %.2f,\n", per_call_us([&] {
            cudaMemcpyBatchAsync(d.data(), sr.data(), sz.data(), 7, &at, &idx, 1, &fail, s); }, 200));
        printf(" \"memcpyAsync_7xH2D_1MB_us_total\": %.2f,\n", per_call_us([&] {
            for (int k = 0; k < 7; ++k) cudaMemcpyAsync(d[k], sr[k], 1 << 20, cudaMemcpyHostToDevice, s); }, 200));
        printf(" \"pointerGetAttributes_us\": %.2f,\n", per_call_us([&] {
            cudaPointerAttributes at; cudaPointerGetAttributes(&at, sr[3]); }, 5000));
        printf(" \"streamIsCapturing_us\": %.2f,\n", per_call_us([&] {
            cudaStreamCaptureStatus st; cudaStreamIsCapturing(s, &st); }, 5000));
        printf(" \"memcpyAsync_H2D_64B_pinned_us\": %.2f,\n", per_call_us([&] {
            cudaMemcpyAsync(d[0], sr[0], 64, cudaMemcpyHostToDevice, s); }, 2000));
    }
    printf(" \"launch+sync_roundtrip_us\": %.2f}\n", per_call_us([&] { noop<<<1, 32, 0, s>>>(nullptr); cudaStreamSynchronize(s); }, 2000));
    return 0;
}
