// Dev tuning harness (not part of the product): times the HM-LSTM K1 / K2
// kernels on one GPU under explicit tilings and checks every variant's
// outputs bit-for-bit against the default tiling's. Build + run with
// scripts/lab/run.sh under gpurun. Prints one JSON object per line.
#include <algorithm>
#include <cstdio>
#include <cstring>
#include <functional>
#include <string>
#include <vector>

#include "bodies.cuh"
#include "launch.cuh"

using namespace bcad_cu_impl;

#define CK(x)                                                                              \
    do {                                                                                   \
        cudaError_t e_ = (x);                                                              \
        if (e_ != cudaSuccess) {                                                           \
            std::fprintf(stderr, "%s:%d %s: %s\n", __FILE__, __LINE__, #x, cudaGetErrorString(e_)); \
            std::exit(1);                                                                  \
        }                                                                                  \
    } while (0)

__device__ uint32_t hash32(uint32_t x) {
    x ^= x >> 16; x *= 0x7feb352du; x ^= x >> 15; x *= 0x846ca68bu; x ^= x >> 16;
    return x;
}
template <class T>
__global__ void init_kernel(T* p, size_t n, uint32_t seed, int binary) {
    for (size_t i = blockIdx.x * size_t(blockDim.x) + threadIdx.x; i < n; i += size_t(gridDim.x) * blockDim.x) {
        const uint32_t h = hash32(uint32_t(i) * 2654435761u ^ seed);
        p[i] = binary ? T(h & 1u) : T(double(h) / 4294967296.0 * 2.0 - 1.0);
    }
}
__global__ void read_kernel(const float4* p, size_t n, float* out) {
    float s = 0.f;
    for (size_t i = blockIdx.x * size_t(blockDim.x) + threadIdx.x; i < n; i += size_t(gridDim.x) * blockDim.x) {
        const float4 v = __ldcs(p + i);
        s += v.x + v.y + v.z + v.w;
    }
    if (s == 1234.5f) *out = s;
}
// memory-only floor of K1's access pattern: read c,f,i,g (+ z per row), write 7 tensors
__global__ void copy_floor_kernel(const float4* c, const float4* f, const float4* i, const float4* g, const float* z1,
                                  const float* z2, float4* const* outs, int vcols, size_t nvec) {
    for (size_t k = blockIdx.x * size_t(blockDim.x) + threadIdx.x; k < nvec; k += size_t(gridDim.x) * blockDim.x) {
        const size_t r = k / vcols;
        const float a = __ldg(z1 + r) + __ldg(z2 + r);
        float4 x = __ldcs(c + k), y = __ldcs(f + k), u = __ldcs(i + k), w = __ldcs(g + k);
        float4 o0 = make_float4(x.x + a, x.y, x.z, x.w), o1 = make_float4(y.x + a, y.y, y.z, y.w);
        float4 o2 = make_float4(u.x, u.y + a, u.z, u.w), o3 = make_float4(w.x, w.y, w.z + a, w.w);
        outs[0][k] = o0; outs[1][k] = o1; outs[2][k] = o2; outs[3][k] = o3;
        outs[4][k] = make_float4(a, a, a, a); outs[5][k] = make_float4(a, 0, a, 0); outs[6][k] = o0;
    }
}


// the same floor with 256-bit loads (ld.global.v8.f32, LDG.E.256 on sm_100a) and 2 x 128-bit stores
struct F8 { float v[8]; };
__device__ __forceinline__ F8 ld8(const float* p) {
    F8 r;
    asm volatile("ld.global.L1::no_allocate.v8.f32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];"
                 : "=f"(r.v[0]), "=f"(r.v[1]), "=f"(r.v[2]), "=f"(r.v[3]), "=f"(r.v[4]), "=f"(r.v[5]), "=f"(r.v[6]), "=f"(r.v[7])
                 : "l"(p));
    return r;
}
__device__ __forceinline__ void st8(float* p, const F8& a) {
    asm volatile("st.global.v8.f32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8};" ::"l"(p), "f"(a.v[0]), "f"(a.v[1]), "f"(a.v[2]),
                 "f"(a.v[3]), "f"(a.v[4]), "f"(a.v[5]), "f"(a.v[6]), "f"(a.v[7]) : "memory");
}
__global__ void copy_floor8_kernel(const float* c, const float* f, const float* i, const float* g, const float* z1,
                                   const float* z2, float* const* outs, int vcols8, size_t nvec8, int st256) {
    for (size_t k = blockIdx.x * size_t(blockDim.x) + threadIdx.x; k < nvec8; k += size_t(gridDim.x) * blockDim.x) {
        const size_t r = k / vcols8;
        const float a = __ldg(z1 + r) + __ldg(z2 + r);
        F8 x = ld8(c + 8 * k), y = ld8(f + 8 * k), u = ld8(i + 8 * k), w = ld8(g + 8 * k);
        F8 o[7];
        for (int e = 0; e < 8; ++e) {
            o[0].v[e] = x.v[e] + a; o[1].v[e] = y.v[e] * a; o[2].v[e] = u.v[e] - a; o[3].v[e] = w.v[e] + a;
            o[4].v[e] = a; o[5].v[e] = x.v[e]; o[6].v[e] = y.v[e];
        }
        for (int t = 0; t < 7; ++t) {
            if (st256) st8(outs[t] + 8 * k, o[t]);
            else {
                float4* d = reinterpret_cast<float4*>(outs[t] + 8 * k);
                d[0] = make_float4(o[t].v[0], o[t].v[1], o[t].v[2], o[t].v[3]);
                d[1] = make_float4(o[t].v[4], o[t].v[5], o[t].v[6], o[t].v[7]);
            }
        }
    }
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

static Flush* g_flush;
static bool g_recompute = false;  // pull(): RecomputeReverse (partials re-derived) instead of cached
static bool g_primal_only = false;
static bool g_skip_finish_variants = false;  // step_ab: also time every variant without K2f  // fwd(): primal only (K1p, broadcast_apply)
static cudaStream_t g_s;

double time_us(const std::function<void()>& fn, int reps = 61) {
    std::vector<cudaEvent_t> a(reps), b(reps);
    for (int k = 0; k < reps; ++k) {
        CK(cudaEventCreate(&a[k]));
        CK(cudaEventCreate(&b[k]));
    }
    for (int k = 0; k < 3; ++k) {
        (*g_flush)(g_s);
        fn();
    }
    for (int k = 0; k < reps; ++k) {
        (*g_flush)(g_s);
        CK(cudaEventRecord(a[k], g_s));
        fn();
        CK(cudaEventRecord(b[k], g_s));
    }
    CK(cudaStreamSynchronize(g_s));
    std::vector<double> t(reps);
    for (int k = 0; k < reps; ++k) {
        float ms;
        CK(cudaEventElapsedTime(&ms, a[k], b[k]));
        t[k] = ms * 1e3;
        cudaEventDestroy(a[k]);
        cudaEventDestroy(b[k]);
    }
    // CUDA event timestamps on this GPU advance in 2.048 us steps (every
    // median of a short kernel lands on a multiple); the flush before each
    // launch randomises the phase, so the MEAN of the quantised samples is an
    // unbiased estimate (outliers above 2x the median dropped).
    std::sort(t.begin(), t.end());
    const double med = t[reps / 2];
    double s = 0;
    int n = 0;
    for (double v : t)
        if (v <= 2 * med) { s += v; ++n; }
    return s / n;
}

template <class T>
struct Problem {
    int n;
    int64_t B, H;
    std::vector<bcad_cu_shape> shapes;
    std::vector<T*> in, partials, adj;
    T* primal = nullptr;
    T* w = nullptr;
    void* ws = nullptr;
    size_t ws_bytes = size_t(256) << 20;
    unsigned long long* err = nullptr;
    Plan plan;
    size_t step_bytes = 0, k1_bytes = 0, k2_bytes = 0;

    static bcad_cu_shape shp(std::initializer_list<int64_t> d) {
        bcad_cu_shape s{};
        s.rank = int(d.size());
        int k = 0;
        for (int64_t x : d) s.dims[k++] = x;
        return s;
    }
    static int64_t vol(const bcad_cu_shape& s) {
        int64_t v = 1;
        for (int k = 0; k < s.rank; ++k) v *= s.dims[k];
        return v;
    }
    // bias: the HM-LSTM bias variant; arity > 0: tanh_product_<arity> (all full, no binary args)
    Problem(bool bias, int64_t B_, int64_t H_, int arity = 0) : B(B_), H(H_) {
        for (int k = 0; k < (arity > 0 ? arity : 4); ++k) shapes.push_back(shp({B, H}));
        if (bias && arity == 0)
            for (int k = 0; k < 3; ++k) shapes.push_back(shp({1, H}));
        if (arity == 0) {
            shapes.push_back(shp({B}));
            shapes.push_back(shp({B}));
        }
        n = int(shapes.size());
        const int n_binary = arity > 0 ? 0 : 2;
        const int64_t E = B * H;
        size_t in_elems = 0;
        for (int j = 0; j < n; ++j) {
            T* p;
            CK(cudaMalloc(&p, vol(shapes[j]) * sizeof(T)));
            init_kernel<<<1024, 256>>>(p, vol(shapes[j]), 77u + 13u * j, j >= n - n_binary);
            in.push_back(p);
            in_elems += vol(shapes[j]);
            T* d;
            CK(cudaMalloc(&d, E * sizeof(T)));
            partials.push_back(d);
            T* a;
            CK(cudaMalloc(&a, vol(shapes[j]) * sizeof(T)));
            adj.push_back(a);
        }
        CK(cudaMalloc(&primal, E * sizeof(T)));
        CK(cudaMalloc(&w, E * sizeof(T)));
        init_kernel<<<1024, 256>>>(w, E, 999u, 0);
        CK(cudaMalloc(&ws, ws_bytes));
        CK(cudaMemset(ws, 0, ws_bytes));
        CK(cudaMalloc(&err, 8));
        CK(cudaMemset(err, 0xff, 8));
        std::string e;
        make_plan(n, shapes.data(), &plan, &e);
        k1_bytes = (in_elems + E + size_t(n) * E) * sizeof(T);
        k2_bytes = (E + size_t(n) * E + in_elems) * sizeof(T);
        step_bytes = k1_bytes + k2_bytes;
        CK(cudaDeviceSynchronize());
    }
};

template <class Body, class T, class Sig>
int fwd(Problem<T>& P, const Tiling* t) {
    std::vector<const void*> in(P.in.begin(), P.in.end());
    void* prim[1] = {P.primal};
    std::vector<void*> parts(P.partials.begin(), P.partials.end());
    FwdArgs a{};
    a.dtype = sizeof(T) == 4 ? BCAD_CU_F32 : BCAD_CU_F64;
    a.in = in.data();
    a.primal = prim;
    a.partials = g_primal_only ? nullptr : parts.data();
    a.stream = g_s;
    a.err = P.err;
    a.plan = &P.plan;
    a.tiling = t;
    std::string e;
    int rc;
    if constexpr (std::is_same_v<Sig, DynSig>) rc = launch_fwd_t<Body, T>(a, &e);
    else rc = launch_fwd_t<Body, T, Sig>(a, &e);
    if (rc) std::fprintf(stderr, "fwd rc %d %s\n", rc, e.c_str());
    return rc;
}

template <class Body, class T, class Sig>
int pull(Problem<T>& P, const Tiling* t) {
    std::vector<const void*> in(P.in.begin(), P.in.end());
    const void* w[1] = {P.w};
    std::vector<const void*> parts(P.partials.begin(), P.partials.end());
    std::vector<void*> adj(P.adj.begin(), P.adj.end());
    PullArgs a{};
    a.dtype = sizeof(T) == 4 ? BCAD_CU_F32 : BCAD_CU_F64;
    a.out_adj = w;
    a.partials = g_recompute ? nullptr : parts.data();
    a.in = in.data();
    a.in_adj = adj.data();
    a.accumulate = nullptr;
    a.workspace = P.ws;
    a.ws_bytes = P.ws_bytes;
    a.stream = g_s;
    a.err = P.err;
    a.plan = &P.plan;
    a.tiling = t;
    std::string e;
    const int rc = launch_pull_t<Body, T, Sig>(a, &e);
    if (rc) std::fprintf(stderr, "pull rc %d %s\n", rc, e.c_str());
    return rc;
}

template <class T>
std::vector<std::vector<T>> snapshot(const std::vector<T*>& ptrs, const std::vector<size_t>& n) {
    CK(cudaStreamSynchronize(g_s));
    std::vector<std::vector<T>> out;
    for (size_t k = 0; k < ptrs.size(); ++k) {
        out.emplace_back(n[k]);
        CK(cudaMemcpy(out.back().data(), ptrs[k], n[k] * sizeof(T), cudaMemcpyDeviceToHost));
    }
    return out;
}

Tiling make_tiling(const Plan& p, int V, int txv, int rpt, int cy) {
    Tiling t;
    t.V = V;
    t.vcols = p.cols / V;
    t.txv = txv;
    t.ty = kThreads / txv;
    t.n_col_tiles = ceil_div(t.vcols, txv);
    t.rpt = rpt;
    t.tile_rows = int64_t(t.ty) * rpt;
    t.n_row_tiles = ceil_div(p.rows, t.tile_rows);
    (void)cy;
    t.n_ctas = t.n_row_tiles * t.n_col_tiles;
    return t;
}

void print_tiling(const char* tag, const char* variant, int64_t B, int64_t H, const Tiling& t, double us, double bytes,
                  bool same) {
    std::printf("{\"exp\": \"%s\", \"variant\": \"%s\", \"B\": %lld, \"H\": %lld, \"txv\": %d, \"ty\": %d, \"rpt\": %d, "
                "\"cy\": %d, \"grid\": [%lld, %lld], \"us\": %.3f, \"GBps\": %.1f, \"bitexact\": %s}\n",
                tag, variant, (long long)B, (long long)H, t.txv, t.ty, t.rpt, 1, (long long)t.n_col_tiles,
                (long long)t.n_row_tiles, us, bytes / (us * 1e-6) / 1e9, same ? "true" : "false");
    std::fflush(stdout);
}

template <class Body, class T, class Sig>
void k1_sweep(const char* tag, bool bias, int64_t B, int64_t H, const std::vector<std::array<int, 2>>& tilings,
              int arity = 0) {
    Problem<T> P(bias, B, H, arity);
    if (g_primal_only) P.k1_bytes -= size_t(P.n) * B * H * sizeof(T);
    constexpr int V = fwd_vec_width<Body, T>();
    const Tiling def = choose_tiling(P.plan, V, ClassMix{}, true);
    fwd<Body, T, Sig>(P, &def);
    std::vector<T*> outs(P.partials.begin(), P.partials.end());
    outs.push_back(P.primal);
    std::vector<size_t> ns(outs.size(), size_t(B * H));
    const auto ref = snapshot(outs, ns);
    double us = time_us([&] { fwd<Body, T, Sig>(P, &def); });
    print_tiling(tag, "default", B, H, def, us, double(P.k1_bytes), true);
    for (auto [txv, rpt] : tilings) {
        const Tiling t = make_tiling(P.plan, V, txv, rpt, 1);
        if (t.n_row_tiles > 65535) continue;
        CK(cudaMemset(P.primal, 0, B * H * sizeof(T)));
        fwd<Body, T, Sig>(P, &t);
        const bool same = snapshot(outs, ns) == ref;
        us = time_us([&] { fwd<Body, T, Sig>(P, &t); });
        print_tiling(tag, "tiled", B, H, t, us, double(P.k1_bytes), same);
    }
    if constexpr (sizeof(T) == 4) {
        if (!bias && arity == 0 && !g_primal_only) {  // memory-only floor of the same access pattern
            float4** d_outs;
            CK(cudaMalloc(&d_outs, 7 * sizeof(float4*)));
            std::vector<float4*> h(7);
            for (int k = 0; k < 6; ++k) h[k] = reinterpret_cast<float4*>(P.partials[k]);
            h[6] = reinterpret_cast<float4*>(P.primal);
            CK(cudaMemcpy(d_outs, h.data(), 7 * sizeof(float4*), cudaMemcpyHostToDevice));
            const size_t nvec = size_t(B * H / 4);
            for (int blocks : {148 * 4, 148 * 8, int((nvec + 255) / 256)}) {
                us = time_us([&] {
                    copy_floor_kernel<<<blocks, 256, 0, g_s>>>(
                        reinterpret_cast<const float4*>(P.in[0]), reinterpret_cast<const float4*>(P.in[1]),
                        reinterpret_cast<const float4*>(P.in[2]), reinterpret_cast<const float4*>(P.in[3]),
                        reinterpret_cast<const float*>(P.in[4]), reinterpret_cast<const float*>(P.in[5]), d_outs,
                        int(H / 4), nvec);
                });
                std::printf("{\"exp\": \"%s\", \"variant\": \"copy_floor\", \"blocks\": %d, \"us\": %.3f, \"GBps\": %.1f}\n",
                            tag, blocks, us, double(P.k1_bytes) / (us * 1e-6) / 1e9);
            }
            const size_t nvec8 = size_t(B * H / 8);
            for (int st256 : {0, 1})
                for (int blocks : {148 * 2, 148 * 4, int((nvec8 + 255) / 256)}) {
                    us = time_us([&] {
                        copy_floor8_kernel<<<blocks, 256, 0, g_s>>>(P.in[0], P.in[1], P.in[2], P.in[3], P.in[4], P.in[5],
                                                                    reinterpret_cast<float* const*>(d_outs), int(H / 8),
                                                                    nvec8, st256);
                    });
                    std::printf("{\"exp\": \"%s\", \"variant\": \"copy_floor_v8%s\", \"blocks\": %d, \"us\": %.3f, "
                                "\"GBps\": %.1f}\n", tag, st256 ? "_st256" : "", blocks, us,
                                double(P.k1_bytes) / (us * 1e-6) / 1e9);
                }
            CK(cudaFree(d_outs));
        }
    }
}

template <class Body, class T, class Sig>
void k2_sweep(const char* tag, bool bias, int64_t B, int64_t H, const std::vector<std::array<int, 3>>& tilings) {
    Problem<T> P(bias, B, H);
    constexpr int V = vec_width<T>();
    const Tiling fdef = choose_tiling(P.plan, V, ClassMix{}, true);
    fwd<Body, T, Sig>(P, &fdef);
    const Tiling def = choose_tiling(P.plan, V, class_mix(P.plan));
    pull<Body, T, Sig>(P, &def);
    std::vector<size_t> ns;
    for (auto& s : P.shapes) ns.push_back(size_t(Problem<T>::vol(s)));
    const auto ref = snapshot(P.adj, ns);
    double us = time_us([&] { pull<Body, T, Sig>(P, &def); });
    print_tiling(tag, "default", B, H, def, us, double(P.k2_bytes), true);
    for (auto [txv, rpt, cy] : tilings) {
        const Tiling t = make_tiling(P.plan, V, txv, rpt, cy);
        if (t.n_row_tiles > 65535) continue;
        for (T* a : P.adj) CK(cudaMemset(a, 0, sizeof(T)));
        CK(cudaMemset(P.ws, 0, P.ws_bytes));  // layouts differ per tiling
        pull<Body, T, Sig>(P, &t);
        const auto got = snapshot(P.adj, ns);
        bool same = true;  // full-shape adjoints bit-exact; reduced ones within 1e-12 relative (other order)
        for (size_t k = 0; k < got.size() && same; ++k)
            for (size_t e = 0; e < got[k].size() && same; ++e) {
                const double x = got[k][e], y = ref[k][e];
                if (ns[k] == size_t(B * H) ? x != y : std::abs(x - y) > 1e-5 * std::max(std::abs(x), std::abs(y)) + 1e-30)
                    same = false;
            }
        us = time_us([&] { pull<Body, T, Sig>(P, &t); });
        print_tiling(tag, "tiled", B, H, t, us, double(P.k2_bytes), same);
    }
}

// Run-to-run bit determinism of K2 under a tiling (reduced adjoints included).
template <class Body, class T, class Sig>
void k2_det(const char* tag, bool bias, int64_t B, int64_t H, int cy_override, int reps) {
    Problem<T> P(bias, B, H);
    constexpr int V = vec_width<T>();
    const Tiling fdef = choose_tiling(P.plan, V, ClassMix{}, true);
    fwd<Body, T, Sig>(P, &fdef);
    Tiling t = choose_tiling(P.plan, V, class_mix(P.plan));
    if (cy_override >= 1) t = make_tiling(P.plan, V, t.txv, t.rpt, cy_override);
    std::vector<size_t> ns;
    for (auto& s : P.shapes) ns.push_back(size_t(Problem<T>::vol(s)));
    pull<Body, T, Sig>(P, &t);
    const auto ref = snapshot(P.adj, ns);
    int bad = 0;
    for (int k = 0; k < reps; ++k) {
        pull<Body, T, Sig>(P, &t);
        if (snapshot(P.adj, ns) != ref) ++bad;
    }
    const double us = time_us([&] { pull<Body, T, Sig>(P, &t); }, 10);
    std::printf("{\"exp\": \"%s\", \"B\": %lld, \"H\": %lld, \"cy\": %d, \"rpt\": %d, \"grid\": [%lld, %lld], "
                "\"nondeterministic_runs\": %d, \"of\": %d, \"us\": %.3f, \"GBps\": %.1f}\n",
                tag, (long long)B, (long long)H, 1, t.rpt, (long long)t.n_col_tiles, (long long)t.n_row_tiles, bad,
                reps, us, double(P.k2_bytes) / (us * 1e-6) / 1e9);
    std::fflush(stdout);
}

// Every reduced adjoint against a host fp64 sum of the rounded terms
// T(w * D_j) (the device's own partials), under a tiling, with the workspace
// poisoned (0xFF = NaN pattern) before the launch and once more re-run.
template <class Body, class T, class Sig>
void k2_check(const char* tag, bool bias, int64_t B, int64_t H, const std::vector<std::array<int, 2>>& tilings) {
    Problem<T> P(bias, B, H);
    constexpr int V = vec_width<T>();
    fwd<Body, T, Sig>(P, nullptr);
    const int64_t E = B * H;
    std::vector<T*> dp(P.partials.begin(), P.partials.end());
    dp.push_back(P.w);
    const auto hp = snapshot(dp, std::vector<size_t>(dp.size(), size_t(E)));
    const auto& hw = hp.back();
    std::vector<std::vector<double>> want(P.n);
    for (int j = 0; j < P.n; ++j) {
        const int64_t v = Problem<T>::vol(P.shapes[j]);
        want[j].assign(size_t(v), 0.0);
        if (v == E) continue;
        const bool col = v == H && P.shapes[j].rank == 2 && P.shapes[j].dims[0] == 1;
        for (int64_t b = 0; b < B; ++b)
            for (int64_t h = 0; h < H; ++h) {
                const size_t e = size_t(b * H + h);
                want[j][size_t(col ? h : b)] += double(T(hw[e] * hp[j][e]));
            }
    }
    std::vector<std::array<int, 2>> all = {{0, 0}};
    all.insert(all.end(), tilings.begin(), tilings.end());
    std::vector<size_t> ns;
    for (auto& s : P.shapes) ns.push_back(size_t(Problem<T>::vol(s)));
    for (auto [txv, rpt] : all) {
        Tiling t = txv == 0 ? choose_tiling(P.plan, V, class_mix(P.plan)) : make_tiling(P.plan, V, txv, rpt, 1);
        if (t.n_row_tiles > 65535) continue;
        CK(cudaMemset(P.ws, 0xff, P.ws_bytes));  // partials poisoned; tickets zero as the C-ABI requires
        const PullLayout L = pull_layout(P.plan, t);
        if (L.n_tickets) CK(cudaMemset(static_cast<char*>(P.ws) + L.ws_tickets, 0, L.n_tickets * 4));
        pull<Body, T, Sig>(P, &t);
        const auto got = snapshot(P.adj, ns);
        CK(cudaMemset(P.ws, 0x00, P.ws_bytes));
        pull<Body, T, Sig>(P, &t);
        const bool rerun_same = snapshot(P.adj, ns) == got;
        double worst = 0.0;
        long long bad = 0;
        int worst_j = -1;
        long long worst_e = -1;
        for (int j = 0; j < P.n; ++j) {
            if (ns[j] == size_t(E)) continue;
            for (size_t e = 0; e < ns[j]; ++e) {
                const double x = got[j][e], y = want[j][e];
                const double r = std::abs(x - y) / (std::abs(y) + 1e-6);
                if (!(r <= 1e-6)) ++bad;
                if (!(r <= worst)) {
                    worst = r;
                    worst_j = j;
                    worst_e = (long long)e;
                }
            }
        }
        std::printf("{\"exp\": \"%s\", \"B\": %lld, \"H\": %lld, \"txv\": %d, \"rpt\": %d, \"grid\": [%lld, %lld], "
                    "\"bad\": %lld, \"worst_rel\": %.3e, \"worst_arg\": %d, \"worst_elem\": %lld, \"rerun_same\": %s}\n",
                    tag, (long long)B, (long long)H, t.txv, t.rpt, (long long)t.n_col_tiles, (long long)t.n_row_tiles,
                    bad, worst, worst_j, worst_e, rerun_same ? "true" : "false");
        std::fflush(stdout);
    }
}

// Pullback time under L2 lookahead distances 0..2, CacheForward and RecomputeReverse.
template <class Body, class T, class Sig>
void k2_prefetch(const char* tag, bool bias, int64_t B, int64_t H) {
    Problem<T> P(bias, B, H);
    fwd<Body, T, Sig>(P, nullptr);
    constexpr int V = vec_width<T>();
    const int64_t E = B * H;
    for (int rec : {0, 1}) {
        g_recompute = rec;
        for (int pf : {0, 1, 2}) {
            Tiling t = choose_tiling(P.plan, V, class_mix(P.plan));
            t.prefetch = pf;
            const double us = time_us([&] { pull<Body, T, Sig>(P, &t); }, 21);
            // recompute streams the 4 full inputs instead of the n partials
            const double bytes = rec ? double(P.k2_bytes) - double(P.n - 4) * E * sizeof(T) : double(P.k2_bytes);
            std::printf("{\"exp\": \"%s\", \"recompute\": %d, \"prefetch\": %d, \"rpt\": %d, \"us\": %.3f, "
                        "\"frac\": %.3f}\n", tag, rec, pf, t.rpt, us, bytes / (us * 1e-6) / 1e9 / 6544.0);
            std::fflush(stdout);
        }
    }
    g_recompute = false;
}

// Whole step (K1 -> K2 [-> K2f], stream launches after an L2 flush) under
// pullback variants: the launcher default, kPipe forced off / on, and given
// (txv, rpt) tilings with and without kPipe. Outputs checked against the
// default's (full-shape adjoints bit-exact; reduced ones bit-exact too when
// the tiling is the default's, else 1e-5 relative).
template <class Body, class T, class Sig>
void step_ab(const char* tag, bool bias, int64_t B, int64_t H, const std::vector<std::array<int, 2>>& tilings) {
    Problem<T> P(bias, B, H);
    constexpr int V = vec_width<T>();
    const Tiling def = choose_tiling(P.plan, V, class_mix(P.plan));
    fwd<Body, T, Sig>(P, nullptr);
    pull<Body, T, Sig>(P, &def);
    std::vector<size_t> ns;
    for (auto& s : P.shapes) ns.push_back(size_t(Problem<T>::vol(s)));
    const auto ref = snapshot(P.adj, ns);
    std::vector<std::pair<std::string, Tiling>> vars;
    vars.push_back({"default", def});
    for (int pipe : {0, 1}) {
        Tiling t = def;
        t.pipe = pipe;
        vars.push_back({pipe ? "default_pipe" : "default_nopipe", t});
    }
    for (auto [txv, rpt] : tilings)
        for (int pipe : {0, 1}) {
            Tiling t = make_tiling(P.plan, V, txv, rpt, 1);
            t.pipe = pipe;
            vars.push_back({pipe ? "tiled_pipe" : "tiled_nopipe", t});
        }
    if (g_skip_finish_variants)
        for (size_t k = 0, n = vars.size(); k < n; ++k) {
            Tiling t = vars[k].second;
            t.combine = 0;  // the separate K2f launch instead of in-kernel tickets
            vars.push_back({vars[k].first + "_k2f", t});
            t.skip_finish = true;  // K2f omitted: the cost of the combination itself
            vars.push_back({vars[k].first + "_nofinish", t});
        }
    for (int rep = 0; rep < 2; ++rep)
        for (auto& [name, t] : vars) {
            for (T* a : P.adj) CK(cudaMemset(a, 0, sizeof(T)));
            CK(cudaMemset(P.ws, 0, P.ws_bytes));
            pull<Body, T, Sig>(P, &t);
            const auto got = snapshot(P.adj, ns);
            const bool same_tiling = t.txv == def.txv && t.rpt == def.rpt && !t.skip_finish;  // same order, bitwise
            bool same = true;
            for (size_t k = 0; k < got.size() && same; ++k)
                for (size_t e = 0; e < got[k].size() && same; ++e) {
                    const double x = got[k][e], y = ref[k][e];
                    if (t.skip_finish && ns[k] != size_t(B * H)) continue;
                    if (ns[k] == size_t(B * H) || same_tiling ? x != y
                                                              : std::abs(x - y) > 1e-5 * std::max(std::abs(x), std::abs(y)) + 1e-30)
                        same = false;
                }
            const double us = time_us([&] {
                fwd<Body, T, Sig>(P, nullptr);
                pull<Body, T, Sig>(P, &t);
            }, 61);
            const double k2 = time_us([&] { pull<Body, T, Sig>(P, &t); }, 61);
            std::printf("{\"exp\": \"%s\", \"rep\": %d, \"variant\": \"%s\", \"txv\": %d, \"rpt\": %d, \"grid\": [%lld, %lld], "
                        "\"pipe\": %d, \"combine\": \"%s\", \"step_us\": %.3f, \"step_frac\": %.3f, \"k2_cold_us\": %.3f, \"same\": %s}\n",
                        tag, rep, name.c_str(), t.txv, t.rpt, (long long)t.n_col_tiles, (long long)t.n_row_tiles,
                        int(pull_pipe(t, g_recompute)), t.skip_finish ? "none" : t.combine == 0 ? "k2f" : "tickets", us,
                        double(P.step_bytes) / (us * 1e-6) / 6538e9, k2, same ? "true" : "false");
            std::fflush(stdout);
        }
}

// Steady-state step time (the bench's method): R rotating problems, K steps
// back to back captured as one CUDA graph, one timed replay (mean over reps).
template <class Body, class T, class Sig>
void step_steady(const char* tag, bool bias, int64_t B, int64_t H, const std::vector<std::array<int, 3>>& variants,
                 const std::vector<std::array<int, 2>>& fwd_variants = {{0, 0}}) {
    constexpr int R = 4, K = 40;
    std::vector<Problem<T>*> P;
    for (int r = 0; r < R; ++r) P.push_back(new Problem<T>(bias, B, H));
    constexpr int V = vec_width<T>();
    for (auto [ftxv, frpt] : fwd_variants)
    for (auto [txv, rpt, pipe] : variants) {
        Tiling t = txv == 0 ? choose_tiling(P[0]->plan, V, class_mix(P[0]->plan)) : make_tiling(P[0]->plan, V, txv, rpt, 1);
        if (pipe >= 0) t.pipe = pipe;
        const Tiling ft = make_tiling(P[0]->plan, V, ftxv ? ftxv : 1, frpt ? frpt : 1, 1);
        const Tiling* ftp = ftxv ? &ft : nullptr;
        for (auto* p : P) CK(cudaMemset(p->ws, 0, p->ws_bytes));
        cudaGraph_t g;
        cudaGraphExec_t ge;
        CK(cudaStreamBeginCapture(g_s, cudaStreamCaptureModeGlobal));
        for (int k = 0; k < K; ++k) {
            fwd<Body, T, Sig>(*P[k % R], ftp);
            pull<Body, T, Sig>(*P[k % R], &t);
        }
        CK(cudaStreamEndCapture(g_s, &g));
        CK(cudaGraphInstantiate(&ge, g, 0));
        std::vector<double> us;
        cudaEvent_t a, b;
        CK(cudaEventCreate(&a));
        CK(cudaEventCreate(&b));
        for (int rep = 0; rep < 9; ++rep) {
            CK(cudaEventRecord(a, g_s));
            CK(cudaGraphLaunch(ge, g_s));
            CK(cudaEventRecord(b, g_s));
            CK(cudaStreamSynchronize(g_s));
            float ms;
            CK(cudaEventElapsedTime(&ms, a, b));
            if (rep > 0) us.push_back(ms * 1e3 / K);
        }
        double m = 0;
        for (double u : us) m += u;
        m /= us.size();
        std::printf("{\"exp\": \"%s\", \"k1\": [%d, %d], \"txv\": %d, \"rpt\": %d, \"pipe\": %d, \"grid\": [%lld, %lld], "
                    "\"step_us\": %.3f, \"step_frac\": %.3f}\n", tag, ftxv, frpt, t.txv, t.rpt, int(pull_pipe(t, g_recompute)),
                    (long long)t.n_col_tiles, (long long)t.n_row_tiles, m, double(P[0]->step_bytes) / (m * 1e-6) / 6538e9);
        std::fflush(stdout);
        CK(cudaGraphExecDestroy(ge));
        CK(cudaGraphDestroy(g));
    }
}

int main(int argc, char** argv) {
    std::string which = argc > 1 ? argv[1] : "all";
    if (which.size() > 2 && which.compare(which.size() - 2, 2, ":r") == 0) {
        g_recompute = true;
        which = which.substr(0, which.size() - 2);
    }
    CK(cudaSetDevice(0));
    CK(cudaStreamCreateWithFlags(&g_s, cudaStreamNonBlocking));
    g_flush = new Flush();
    using namespace bcad_dev;
    if (which == "k1ab") {  // interleaved A/B of K1 rows per thread on small problems
        Problem<float> Pc(false, 1024, 1024), Pb(true, 1024, 1024);
        for (int rep = 0; rep < 6; ++rep)
            for (int rpt : {1, 2, 4}) {
                const Tiling tc = make_tiling(Pc.plan, 4, 256, rpt, 1), tb = make_tiling(Pb.plan, 4, 256, rpt, 1);
                const double uc = time_us([&] { fwd<KHmlstm, float, SigHmlstmCanonical>(Pc, &tc); }, 41);
                const double ub = time_us([&] { fwd<KHmlstmBias, float, SigHmlstmBias>(Pb, &tb); }, 41);
                std::printf("{\"exp\": \"k1ab\", \"rep\": %d, \"rpt\": %d, \"cfg2_us\": %.3f, \"cfg3_us\": %.3f}\n", rep,
                            rpt, uc, ub);
                std::fflush(stdout);
            }
    }
    if (which == "k1small") {  // K1 rows per thread at configs 2 / 3 (means), incl. single-wave rpt = 3
        const std::vector<std::array<int, 2>> t = {{256, 1}, {256, 2}, {256, 3}, {256, 4}, {128, 2}, {128, 3}, {64, 3}};
        k1_sweep<KHmlstm, float, SigHmlstmCanonical>("k1_cfg2", false, 1024, 1024, t);
        k1_sweep<KHmlstmBias, float, SigHmlstmBias>("k1_cfg3", true, 1024, 1024, t);
        step_ab<KHmlstmBias, float, SigHmlstmBias>("step_cfg3", true, 1024, 1024, {{16, 3}, {16, 5}, {32, 3}});
    }
    if (which == "arity32") {  // A = 32 static signature, rows per thread
        const std::vector<std::array<int, 2>> t = {{256, 2}, {256, 4}, {256, 8}, {256, 16}, {256, 32}, {128, 4},
                                                    {128, 8}, {128, 16}, {64, 8}, {64, 16}, {32, 16}};
        k1_sweep<KTanhProduct<32>, float, SigAllFull<32>>("k1_tp32_4096_static", false, 4096, 4096, t, 32);
        k1_sweep<KTanhProduct<1>, float, SigAllFull<1>>("k1_tp1_4096_static", false, 4096, 4096, t, 1);
        k1_sweep<KTanhProduct<4>, float, SigAllFull<4>>("k1_tp4_4096_static", false, 4096, 4096, t, 4);
        k1_sweep<KTanhProduct<4>, float, DynSig>("k1_tp4_4096", false, 4096, 4096, t, 4);
    }
    if (which == "arity") {  // tanh_product_<A> K1 at 4096^2 fp32 (bench extra.arity), rows per thread
        const std::vector<std::array<int, 2>> t = {{256, 4}, {256, 8}, {256, 16}};
        k1_sweep<KTanhProduct<8>, float, DynSig>("k1_tp8_4096", false, 4096, 4096, t, 8);
        k1_sweep<KTanhProduct<16>, float, DynSig>("k1_tp16_4096", false, 4096, 4096, t, 16);
        k1_sweep<KTanhProduct<18>, float, DynSig>("k1_tp18_4096", false, 4096, 4096, t, 18);
        k1_sweep<KTanhProduct<32>, float, DynSig>("k1_tp32_4096", false, 4096, 4096, t, 32);
        k1_sweep<KTanhProduct<8>, float, SigAllFull<8>>("k1_tp8_4096_static", false, 4096, 4096, t, 8);
        k1_sweep<KTanhProduct<16>, float, SigAllFull<16>>("k1_tp16_4096_static", false, 4096, 4096, t, 16);
        k1_sweep<KTanhProduct<18>, float, SigAllFull<18>>("k1_tp18_4096_static", false, 4096, 4096, t, 18);
        k1_sweep<KTanhProduct<32>, float, SigAllFull<32>>("k1_tp32_4096_static", false, 4096, 4096, t, 32);
    }
    if (which == "k2r5") {  // RecomputeReverse pullback alone at config 5 and a mid size (default tilings)
        g_recompute = true;
        k2_sweep<KHmlstmBias, float, SigHmlstmBias>("k2r_cfg5", true, 65536, 4096, {});
        k2_sweep<KHmlstmBias, float, SigHmlstmBias>("k2r_16384x1024", true, 16384, 1024, {});
        k2_sweep<KHmlstm, float, SigHmlstmCanonical>("k2r_canon_65536x4096", false, 65536, 4096, {});
        g_recompute = false;
    }
    if (which == "stepss") {  // steady-state config-3 / config-2 steps under pullback tilings
        step_steady<KHmlstmBias, float, SigHmlstmBias>("ss_cfg3", true, 1024, 1024,
            {{0, 0, -1}, {0, 0, 0}, {16, 2, 0}, {16, 2, 1}, {16, 3, 0}, {16, 4, 0}, {32, 2, 0}, {32, 4, 1}, {8, 4, 1}});
        step_steady<KHmlstm, float, SigHmlstmCanonical>("ss_cfg2", false, 1024, 1024,
            {{0, 0, -1}, {0, 0, 1}, {256, 1, 0}, {256, 4, 0}, {256, 4, 1}, {128, 2, 0}, {128, 4, 1}});
    }
    if (which == "stepss3") {  // config 3 steady state: K1 tilings x a few K2 tilings
        step_steady<KHmlstmBias, float, SigHmlstmBias>("ss3", true, 1024, 1024, {{0, 0, -1}, {16, 2, 0}, {32, 4, 1}},
                                                       {{0, 0}, {128, 3}, {256, 2}, {256, 3}, {128, 2}, {64, 3}, {128, 4}});
    }
    if (which == "stepr") {  // RecomputeReverse steps (K1p + K2r) at the small configs
        g_recompute = true;
        g_primal_only = true;
        step_ab<KHmlstm, float, SigHmlstmCanonical>("stepr_cfg2", false, 1024, 1024, {{256, 2}, {256, 4}, {128, 2}, {128, 4}, {64, 4}});
        step_ab<KHmlstmBias, float, SigHmlstmBias>("stepr_cfg3", true, 1024, 1024, {{16, 2}, {16, 4}, {32, 2}, {32, 4}});
        g_recompute = false;
        g_primal_only = false;
    }
    if (which == "step3") {  // config 3 only, with K2f-less timing variants
        g_skip_finish_variants = true;
        step_ab<KHmlstmBias, float, SigHmlstmBias>("step_cfg3", true, 1024, 1024, {{16, 2}, {32, 2}, {32, 1}, {64, 2}});
        g_skip_finish_variants = false;
    }
    if (which == "step") {
        step_ab<KHmlstmBias, float, SigHmlstmBias>("step_cfg3", true, 1024, 1024,
                                                   {{16, 2}, {16, 4}, {16, 8}, {32, 2}, {32, 4}, {8, 4}, {8, 8}});
        step_ab<KHmlstm, float, SigHmlstmCanonical>("step_cfg2", false, 1024, 1024, {{256, 2}, {256, 4}, {128, 2}});
    }
    if (which == "floor") {
        k1_sweep<KHmlstm, float, SigHmlstmCanonical>("k1_cfg2", false, 1024, 1024, {{256, 1}, {256, 2}});
        k1_sweep<KHmlstm, float, SigHmlstmCanonical>("k1_4096", false, 4096, 1024, {{256, 2}});
    }
    if (which == "all" || which == "k1") {
        const std::vector<std::array<int, 2>> t1 = {{256, 1}, {256, 2}, {128, 1}, {128, 2}, {64, 1}, {64, 2},
                                                     {32, 1}, {32, 2}, {32, 4}};
        k1_sweep<KHmlstm, float, SigHmlstmCanonical>("k1_cfg2", false, 1024, 1024, t1);
        k1_sweep<KHmlstmBias, float, SigHmlstmBias>("k1_cfg3", true, 1024, 1024, t1);
    }
    if (which == "all" || which == "k2") {
        const std::vector<std::array<int, 3>> t2 = {{256, 1, 1}, {256, 2, 1}, {128, 1, 1}, {128, 2, 1},
                                                     {64, 1, 1}, {32, 1, 1}, {32, 2, 1}, {32, 4, 1}};
        k2_sweep<KHmlstm, float, SigHmlstmCanonical>("k2_cfg2", false, 1024, 1024, t2);
        const std::vector<std::array<int, 3>> t3 = {{32, 1, 1}, {32, 2, 1}, {32, 4, 1}, {32, 8, 1},
                                                     {16, 1, 1}, {16, 2, 1}, {16, 4, 1}, {16, 8, 1},
                                                     {8, 1, 1}, {8, 2, 1}, {8, 4, 1}, {8, 8, 1},
                                                     {64, 2, 1}, {64, 4, 1}, {128, 1, 1}, {128, 2, 1}, {256, 1, 1},
                                                     {256, 2, 1}};
        k2_sweep<KHmlstmBias, float, SigHmlstmBias>("k2_cfg3", true, 1024, 1024, t3);
    }
    if (which == "k2b") {  // bias pullback tilings at medium and large batch
        std::vector<std::array<int, 3>> t;
        for (int txv : {8, 16, 32, 64})
            for (int rpt : {1, 2, 4, 8, 16, 32, 64}) t.push_back({txv, rpt, 1});
        k2_sweep<KHmlstmBias, float, SigHmlstmBias>("k2b_4096", true, 4096, 1024, t);
        k2_sweep<KHmlstmBias, float, SigHmlstmBias>("k2b_16384", true, 16384, 1024, t);
        k2_sweep<KHmlstmBias, float, SigHmlstmBias>("k2b_8192x4096", true, 8192, 4096, t);
    }
    if (which == "k1c2time") {  // config-2 K1 alone, repeated (A/B runs)
        Problem<float> P(false, 1024, 1024);
        for (int rep = 0; rep < 5; ++rep) {
            const double us = time_us([&] { fwd<KHmlstm, float, SigHmlstmCanonical>(P, nullptr); }, 41);
            std::printf("{\"exp\": \"k1c2time\", \"rep\": %d, \"us\": %.3f}\n", rep, us);
        }
    }
    if (which == "k1time") {  // default-tiling K1 timings: cfg2, cfg3, cfg5-per-G8-shard, cfg5 sizes
        for (auto [bias, B, H] : {std::tuple<bool, int64_t, int64_t>{false, 1024, 1024}, {true, 1024, 1024},
                                  {true, 8192, 4096}, {true, 65536, 4096}, {false, 8192, 4096}}) {
            if (bias) {
                Problem<float> P(true, B, H);
                const double us = time_us([&] { fwd<KHmlstmBias, float, SigHmlstmBias>(P, nullptr); }, 15);
                std::printf("{\"exp\": \"k1time\", \"bias\": 1, \"B\": %lld, \"H\": %lld, \"us\": %.3f, \"GBps\": %.1f}\n",
                            (long long)B, (long long)H, us, double(P.k1_bytes) / (us * 1e-6) / 1e9);
            } else {
                Problem<float> P(false, B, H);
                const double us = time_us([&] { fwd<KHmlstm, float, SigHmlstmCanonical>(P, nullptr); }, 15);
                std::printf("{\"exp\": \"k1time\", \"bias\": 0, \"B\": %lld, \"H\": %lld, \"us\": %.3f, \"GBps\": %.1f}\n",
                            (long long)B, (long long)H, us, double(P.k1_bytes) / (us * 1e-6) / 1e9);
            }
            std::fflush(stdout);
        }
    }
    if (which == "k1c2") {  // default-tiling config-2 forwards, for ncu
        Problem<float> P(false, 1024, 1024);
        for (int k = 0; k < 3; ++k) fwd<KHmlstm, float, SigHmlstmCanonical>(P, nullptr);
        CK(cudaDeviceSynchronize());
    }
    if (which == "k2c2") {  // default-tiling config-2 pullbacks (ROW reductions), for sanitizers / ncu
        Problem<float> P(false, 1024, 1024);
        fwd<KHmlstm, float, SigHmlstmCanonical>(P, nullptr);
        for (int k = 0; k < 3; ++k) pull<KHmlstm, float, SigHmlstmCanonical>(P, nullptr);
        CK(cudaDeviceSynchronize());
    }
    if (which == "k2tick") {  // config-3 and mixed-layout pullbacks with the in-kernel ticket combine, for sanitizers
        for (auto [B, H] : {std::pair<int64_t, int64_t>{1024, 1024}, {64, 256}, {3000, 1024}}) {
            Problem<float> P(true, B, H);
            fwd<KHmlstmBias, float, SigHmlstmBias>(P, nullptr);
            Tiling t = choose_tiling(P.plan, 4, class_mix(P.plan));
            t.combine = 1;
            for (int k = 0; k < 2; ++k) pull<KHmlstmBias, float, SigHmlstmBias>(P, &t);
            CK(cudaDeviceSynchronize());
        }
    }
    if (which == "k2mix") {  // several reduction layouts in one process: small / tall / wide bias problems
        for (auto [B, H] : {std::pair<int64_t, int64_t>{64, 256}, {4096, 128}, {16, 8192}, {3000, 1024}}) {
            Problem<float> P(true, B, H);
            fwd<KHmlstmBias, float, SigHmlstmBias>(P, nullptr);
            for (int k = 0; k < 2; ++k) pull<KHmlstmBias, float, SigHmlstmBias>(P, nullptr);
            CK(cudaDeviceSynchronize());
        }
    }
    if (which == "k2c3") {  // one default-tiling config-3 pullback, for ncu
        Problem<float> P(true, 1024, 1024);
        const Tiling fdef = choose_tiling(P.plan, 4, ClassMix{}, true);
        fwd<KHmlstmBias, float, SigHmlstmBias>(P, &fdef);
        for (int k = 0; k < 3; ++k) pull<KHmlstmBias, float, SigHmlstmBias>(P, nullptr);
        CK(cudaDeviceSynchronize());
    }
    if (which == "k1b") {  // bias forward tilings ((1,H) loads amortised over rows per thread)
        const std::vector<std::array<int, 2>> t = {{256, 1}, {256, 2}, {256, 4}, {256, 8}, {64, 2}, {64, 4},
                                                    {32, 2}, {32, 4}, {32, 8}};
        for (int64_t B : {256, 1024, 2048, 4096, 16384})
            k1_sweep<KHmlstmBias, float, SigHmlstmBias>(("k1b_" + std::to_string(B)).c_str(), true, B, 1024, t);
        k1_sweep<KHmlstmBias, float, SigHmlstmBias>("k1b_8192x4096", true, 8192, 4096, t);
        k1_sweep<KHmlstm, float, SigHmlstmCanonical>("k1c_4096", false, 4096, 1024, t);
    }
    if (which == "k1rpt") {  // rows per thread of K1 / K1p across body widths
        const std::vector<std::array<int, 2>> t = {{256, 1}, {256, 2}, {256, 4}, {256, 8}, {256, 16}, {256, 32}};
        k1_sweep<KTanhProduct<1>, float, DynSig>("k1_tp1_4096", false, 4096, 4096, t, 1);
        k1_sweep<KTanhProduct<4>, float, DynSig>("k1_tp4_4096", false, 4096, 4096, t, 4);
        k1_sweep<KTanhProduct<16>, float, DynSig>("k1_tp16_4096", false, 4096, 4096, t, 16);
        k1_sweep<KHmlstm, double, SigHmlstmCanonical>("k1_cfg4", false, 8192, 2048, t);
        g_primal_only = true;
        k1_sweep<KHmlstmBias, float, SigHmlstmBias>("k1p_cfg5", true, 65536, 4096, t);
        k1_sweep<KHmlstm, float, SigHmlstmCanonical>("k1p_cfg2", false, 1024, 1024, t);
        g_primal_only = false;
    }
    if (which == "k2pf") {  // pullback L2 lookahead, both policies, several sizes
        k2_prefetch<KHmlstmBias, float, SigHmlstmBias>("k2pf_cfg5", true, 65536, 4096);
        k2_prefetch<KHmlstm, float, SigHmlstmCanonical>("k2pf_cfg2", false, 1024, 1024);
        k2_prefetch<KHmlstmBias, float, SigHmlstmBias>("k2pf_cfg3", true, 1024, 1024);
        k2_prefetch<KHmlstmBias, float, SigHmlstmBias>("k2pf_bias16384", true, 16384, 1024);
        k2_prefetch<KHmlstm, double, SigHmlstmCanonical>("k2pf_cfg4", false, 8192, 2048);
        k2_prefetch<KHmlstm, float, SigHmlstmCanonical>("k2pf_canon65536x4096", false, 65536, 4096);
    }
    if (which == "k5") {  // config-5 size: wave quantisation of the default rpt
        k1_sweep<KHmlstmBias, float, SigHmlstmBias>("k1_cfg5", true, 65536, 4096,
                                                    {{256, 2}, {256, 4}, {256, 8}, {256, 28}, {256, 55}, {256, 56},
                                                     {64, 2}, {64, 4}});
        k2_sweep<KHmlstmBias, float, SigHmlstmBias>("k2_cfg5", true, 65536, 4096,
                                                    {{32, 8, 1}, {32, 16, 1}, {32, 28, 1}, {32, 55, 1}, {32, 56, 1},
                                                     {32, 64, 1}, {16, 16, 1}, {16, 28, 1}, {16, 56, 1}});
    }
    if (which == "k2check") {
        std::vector<std::array<int, 2>> t;
        for (int txv : {8, 16, 32, 64, 128, 256})
            for (int rpt : {1, 2, 4, 16}) t.push_back({txv, rpt});
        k2_check<KHmlstmBias, float, SigHmlstmBias>("k2check_4096", true, 4096, 1024, t);
        k2_check<KHmlstmBias, float, SigHmlstmBias>("k2check_1024", true, 1024, 1024, t);
        k2_check<KHmlstmBias, float, SigHmlstmBias>("k2check_8192x4096", true, 8192, 4096, {{32, 1}, {32, 4}});
        k2_check<KHmlstm, float, SigHmlstmCanonical>("k2check_canon_1024", false, 1024, 1024, t);
        k2_check<KHmlstmBias, double, SigHmlstmBias>("k2check_f64_4096", true, 4096, 1024, {{32, 1}, {16, 4}});
    }
    if (which == "all" || which == "det") {
        k2_det<KHmlstmBias, float, SigHmlstmBias>("det_cfg5", true, 65536, 4096, 0, 4);
        k2_det<KHmlstmBias, float, SigHmlstmBias>("det_cfg3", true, 1024, 1024, 0, 20);
    }
    return 0;
}
