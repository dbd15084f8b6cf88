// The hot-path CUDA kernels (sm_100a), templated on a registered body.
//
//   fwd2d       K1  fused dual-number forward: one visit per output cell,
//                   primal + M*N partials (forward.hpp:98-150) or the primal
//                   only through the real body (broadcast.hpp:102-125).
//                   128-bit vector loads/stores on FULL/COL arguments,
//                   stride-0 scalar loads for ROW/SCALAR ones; no expansion.
//   pull2d      K2  pullback: w (.) D summed over outputs, written elementwise
//                   for FULL arguments and sum-reduced over broadcast axes
//                   for ROW (warp shuffles), COL (CTA shared-memory tiles)
//                   and SCALAR arguments; a reduction spanning several CTAs
//                   leaves fp64 per-tile partials that the last-arriving CTA
//                   of each strip / tile combines in fixed order (completion
//                   tickets in the workspace). No floating-point atomics;
//                   bitwise deterministic run to run. With kRecompute the partials are re-derived
//                   from the inputs in the same pass (RecomputeReverse,
//                   mixed.hpp:75-90) instead of read.
//   pull_finish K2f the same combination as a separate dependent launch, for
//                   callers whose workspace carries no ticket region.
//   fwd_generic / pull_generic   rank-N fallbacks (3+ irreducible axis
//                   groups; odd widths and unaligned views run fwd2d /
//                   pull2d at one cell per thread instead).
#pragma once

#include <cstdint>
#include <type_traits>
#include <cuda_runtime.h>

#include "dual.cuh"
#include "plan.hpp"

namespace bcad_dev {

using bcad_cu_impl::kCol;
using bcad_cu_impl::kFull;
using bcad_cu_impl::kMaxRank;
using bcad_cu_impl::kRow;
using bcad_cu_impl::kScalar;
using bcad_cu_impl::kThreads;
using bcad_cu_impl::kCtasPerSm;
using bcad_cu_impl::kRecomputeCtasPerSm;

// ----------------------------------------------------------- vector I/O
template <class T, int V> struct alignas(sizeof(T) * V) Pack { T x[V]; };

template <class T, int V>
__device__ __forceinline__ Pack<T, V> ld_stream(const T* p) {
    Pack<T, V> r;
    if constexpr (V == 4 && sizeof(T) == 4) {
        const float4 v = __ldcs(reinterpret_cast<const float4*>(p));
        r.x[0] = v.x; r.x[1] = v.y; r.x[2] = v.z; r.x[3] = v.w;
    } else if constexpr (V == 2 && sizeof(T) == 8) {
        const double2 v = __ldcs(reinterpret_cast<const double2*>(p));
        r.x[0] = v.x; r.x[1] = v.y;
    } else if constexpr (V == 2 && sizeof(T) == 4) {
        const float2 v = __ldcs(reinterpret_cast<const float2*>(p));
        r.x[0] = v.x; r.x[1] = v.y;
    } else {
#pragma unroll
        for (int v = 0; v < V; ++v) r.x[v] = __ldcs(p + v);
    }
    return r;
}

// L2 prefetch of a line a later loop iteration reads (no register, no
// scoreboard: the thread does not wait for it)
__device__ __forceinline__ void prefetch_l2(const void* p) { asm volatile("prefetch.global.L2 [%0];" ::"l"(p)); }

template <class T, int V>
__device__ __forceinline__ Pack<T, V> ld_ro(const T* p) {  // read-only, may be re-read (COL args)
    Pack<T, V> r;
    if constexpr (V == 4 && sizeof(T) == 4) {
        const float4 v = __ldg(reinterpret_cast<const float4*>(p));
        r.x[0] = v.x; r.x[1] = v.y; r.x[2] = v.z; r.x[3] = v.w;
    } else if constexpr (V == 2 && sizeof(T) == 8) {
        const double2 v = __ldg(reinterpret_cast<const double2*>(p));
        r.x[0] = v.x; r.x[1] = v.y;
    } else if constexpr (V == 2 && sizeof(T) == 4) {
        const float2 v = __ldg(reinterpret_cast<const float2*>(p));
        r.x[0] = v.x; r.x[1] = v.y;
    } else {
#pragma unroll
        for (int v = 0; v < V; ++v) r.x[v] = __ldg(p + v);
    }
    return r;
}

template <class T, int V>
__device__ __forceinline__ void st_vec(T* p, const Pack<T, V>& r) {
    if constexpr (V == 4 && sizeof(T) == 4) {
        *reinterpret_cast<float4*>(p) = make_float4(r.x[0], r.x[1], r.x[2], r.x[3]);
    } else if constexpr (V == 2 && sizeof(T) == 8) {
        *reinterpret_cast<double2*>(p) = make_double2(r.x[0], r.x[1]);
    } else if constexpr (V == 2 && sizeof(T) == 4) {
        *reinterpret_cast<float2*>(p) = make_float2(r.x[0], r.x[1]);
    } else {
#pragma unroll
        for (int v = 0; v < V; ++v) p[v] = r.x[v];
    }
}

// Load V consecutive cells of argument `cls` at (r, c0).
template <class T, int V>
__device__ __forceinline__ Pack<T, V> ld_arg(const T* base, int cls, int64_t r, int64_t c0, int64_t cols) {
    Pack<T, V> a;
    if (cls == kFull) {
        a = ld_stream<T, V>(base + r * cols + c0);
    } else if (cls == kCol) {
        a = ld_ro<T, V>(base + c0);
    } else {
        const T s = __ldg(base + (cls == kRow ? r : 0));
#pragma unroll
        for (int v = 0; v < V; ++v) a.x[v] = s;
    }
    return a;
}

// Transcendental census (census.cuh; dual.cuh s_tcount): zero this thread's
// tally at kernel entry; at exit add the warp's tallies with one atomic into
// a slot spread by block index (kCountSlots).
__device__ __forceinline__ void count_begin() { s_tcount[threadIdx.x] = 0; }

__device__ __forceinline__ void count_flush(unsigned long long* slots) {
    if (slots == nullptr) return;
    const unsigned mask = __activemask();
    const unsigned c = __reduce_add_sync(mask, s_tcount[threadIdx.x]);
    if (int(threadIdx.x & 31) == __ffs(int(mask)) - 1 && c != 0)
        atomicAdd(slots + ((blockIdx.x + blockIdx.y * 977u) & unsigned(bcad_cu_impl::kCountSlots - 1)),
                  static_cast<unsigned long long>(c));
}

// Device error word: (status << 56) | flat output index; the lowest failing
// cell wins (atomicMin), matching the reference's per-cell annotation.
__device__ __forceinline__ void report_error(unsigned long long* word, int64_t flat) {
    const uint8_t code = s_err_flag[threadIdx.x];
    if (code) {
        atomicMin(word, (static_cast<unsigned long long>(code) << 56) | static_cast<unsigned long long>(flat));
        s_err_flag[threadIdx.x] = 0;
    }
}

// ------------------------------------------------- argument-class signatures
// A signature fixes each argument's stride class at compile time so the
// loads, stores and reductions of the hot kernels are branch-free and the
// broadcast (ROW / COL / SCALAR) loads are hoisted; DynSig reads the class
// from the parameter block (every other shape).
struct DynSig {
    static constexpr bool kStatic = false;
    __host__ __device__ static constexpr int cls(int) { return -1; }
    __host__ __device__ static constexpr bool has(int) { return true; }
};
template <int... C>
struct Sig {
    static constexpr bool kStatic = true;
    static constexpr int kN = sizeof...(C);
    __host__ __device__ static constexpr int cls(int j) {
        constexpr int c[] = {C...};
        return c[j];
    }
    __host__ __device__ static constexpr bool has(int k) {
        constexpr int c[] = {C...};
        for (int j = 0; j < kN; ++j)
            if (c[j] == k) return true;
        return false;
    }
};

// Index of argument j among the arguments of its class: compile-time for a
// static signature when every adjoint is wanted (kDense), else from params.
template <class S, bool kDense>
__device__ __forceinline__ int arg_slot(const int* dyn, int j) {
    if constexpr (S::kStatic && kDense) {
        int n = 0;
        for (int l = 0; l < j; ++l) n += S::cls(l) == S::cls(j);
        return n;
    } else {
        return dyn[j];
    }
}

template <class S>
__device__ __forceinline__ int arg_class(const int* dyn, int j) {
    if constexpr (S::kStatic) return S::cls(j);
    else return dyn[j];
}

// Programmatic dependent launch (PTX griddepcontrol): the dependent kernel
// may be scheduled while its predecessor drains; it waits here before it
// touches any memory, so ordering is exactly stream order.
__device__ __forceinline__ void pdl_wait() { asm volatile("griddepcontrol.wait;" ::: "memory"); }
__device__ __forceinline__ void pdl_trigger() { asm volatile("griddepcontrol.launch_dependents;" ::: "memory"); }

// ------------------------------------------------------ cell evaluation
// True when every branch predicate of the body reads an argument that is
// uniform across a thread's V cells under signature S (ROW / SCALAR class),
// so the V cells can be evaluated as one lane-vector dual (VDual).
template <class Body, class S>
__host__ __device__ constexpr bool vec_eval_ok() {
    if (Body::kPredicateArgs == 0u) return true;
    if (!S::kStatic) return false;
    for (int j = 0; j < Body::kIn; ++j)
        if (((Body::kPredicateArgs >> j) & 1u) && S::cls(j) != kRow && S::cls(j) != kScalar) return false;
    return true;
}

// Arguments that only feed branch predicates (Body::kPredicateOnlyArgs, bit
// j): no arithmetic reads them, so every partial with respect to them is a
// structural zero. The RecomputeReverse pullback skips forming their terms
// (w * 0); the cached pullback reads and sums the stored zeros as the
// reference-faithful byte count requires.
// (-DBCAD_NO_PREDICATE_ONLY=1 disables the skip, for A/B runs.)
template <class Body>
__host__ __device__ constexpr uint32_t predicate_only_args() {
#if defined(BCAD_NO_PREDICATE_ONLY) && BCAD_NO_PREDICATE_ONLY
    return 0u;
#else
    if constexpr (requires { Body::kPredicateOnlyArgs; }) return Body::kPredicateOnlyArgs;
    else return 0u;
#endif
}

// The dual evaluation of one thread's V cells: primals y[M] (nullable) and
// partials d[M*N] from inputs x[N], seeded x_j + e_j (forward.hpp:121-126).
template <class Body, class T, int V, class S>
__device__ __forceinline__ void eval_cells(const Pack<T, V>* x, Pack<T, V>* y, Pack<T, V>* d,
                                           unsigned long long* err, int64_t off) {
    constexpr int N = Body::kIn, M = Body::kOut;
    auto scalar_lane = [&](int v) {
        Dual<T, N> xi[N], yo[M];
#pragma unroll
        for (int j = 0; j < N; ++j) xi[j] = Dual<T, N>::seeded(x[j].x[v], j);
        // a static signature whose predicates vary per cell: the branch-free
        // form, if the body has one
        if constexpr (Body::kSelectForm && S::kStatic && !vec_eval_ok<Body, S>()) Body::template body_select<Dual<T, N>>(xi, yo);
        else Body::template body<Dual<T, N>>(xi, yo);
        if constexpr (Body::kMayRaise) report_error(err, off + v);
#pragma unroll
        for (int i = 0; i < M; ++i) {
            if (y) y[i].x[v] = yo[i].v;
#pragma unroll
            for (int j = 0; j < N; ++j) d[i * N + j].x[v] = yo[i].d[j];
        }
    };
    if constexpr (vec_eval_ok<Body, S>() && V > 1) {
        using VD = VDual<T, N, V>;
        VD xi[N], yo[M];
#pragma unroll
        for (int j = 0; j < N; ++j) {
            xi[j] = VD(T(0));
#pragma unroll
            for (int v = 0; v < V; ++v) xi[j].v[v] = x[j].x[v];
#pragma unroll
            for (int v = 0; v < V; ++v) xi[j].d[j][v] = T(1);
            xi[j].nz = kDenseDuals ? ~0u : (1u << j);
        }
        Body::template body<VD>(xi, yo);
        if constexpr (Body::kMayRaise) {
            if (s_err_flag[threadIdx.x]) {  // rare: find the failing lane(s) in order
                s_err_flag[threadIdx.x] = 0;
#pragma unroll 1
                for (int v = 0; v < V; ++v) scalar_lane(v);
                return;
            }
        }
#pragma unroll
        for (int i = 0; i < M; ++i) {
#pragma unroll
            for (int v = 0; v < V; ++v) {
                if (y) y[i].x[v] = yo[i].v[v];
#pragma unroll
                for (int j = 0; j < N; ++j) d[i * N + j].x[v] = yo[i].d[j][v];
            }
        }
    } else {
#pragma unroll
        for (int v = 0; v < V; ++v) scalar_lane(v);
    }
}

// ------------------------------------------------------------- K1 params
// 2-D grid: blockIdx.x = column tile (txv vector-columns), blockIdx.y = row
// tile (ty thread-rows x rpt rows per thread).
template <int N, int M, class T>
struct Fwd2DParams {
    const T* in[N];
    int cls[N];
    T* primal[M];
    T* partials[M * N];
    int64_t rows, cols;
    int vcols;
    int txv_shift, ty, rpt;
    int64_t tile_rows;
    unsigned long long* err;
};

// K1. kReal: evaluate the real body (primal only). Otherwise the dual body,
// storing whichever of primal / partials pointers are non-null (kDense: all
// of them, no checks). The next row's loads are issued before the current
// row is evaluated, so every thread keeps two rows of loads in flight.
//
// Bodies whose per-cell dual state is wide (tanh_product_<A> at large A) can
// ask for K1 without the next-row register pipeline (Body::kFwdPipeline =
// false) and for a minimum of resident CTAs per SM (Body::kFwdMinBlocks),
// trading the second row of loads in flight for occupancy.
template <class Body>
__host__ __device__ constexpr bool fwd_pipeline() {
    if constexpr (requires { Body::kFwdPipeline; }) return Body::kFwdPipeline;
    else return true;
}
// 0 = no minimum (the compiler's own register heuristic; an explicit 1
// lets ptxas use up to 255 registers, measured 2x slower for A >= 16)
template <class Body>
__host__ __device__ constexpr int fwd_min_blocks() {
    if constexpr (requires { Body::kFwdMinBlocks; }) return Body::kFwdMinBlocks;
    else return 0;
}

template <class Body, class T, int V, bool kReal, class S, bool kDense>
__global__ void __launch_bounds__(kThreads, fwd_min_blocks<Body>()) fwd2d_kernel(const __grid_constant__ Fwd2DParams<Body::kIn, Body::kOut, T> p) {
    constexpr int N = Body::kIn, M = Body::kOut;
    pdl_wait();
    pdl_trigger();
    if constexpr (Body::kMayRaise && !kReal) s_err_flag[threadIdx.x] = 0;
    const int tx = threadIdx.x & ((1 << p.txv_shift) - 1);
    const int ty = threadIdx.x >> p.txv_shift;
    const int vc = (blockIdx.x << p.txv_shift) + tx;
    if (vc >= p.vcols) return;
    const int64_t c0 = int64_t(vc) * V;
    // broadcast loads that do not depend on the row: hoisted
    Pack<T, V> xc[N];
#pragma unroll
    for (int j = 0; j < N; ++j) {
        const int cls = arg_class<S>(p.cls, j);
        if (cls == kCol) xc[j] = ld_ro<T, V>(p.in[j] + c0);
        if (cls == kScalar) {
            const T v0 = __ldg(p.in[j]);
#pragma unroll
            for (int v = 0; v < V; ++v) xc[j].x[v] = v0;
        }
    }
    auto load_row = [&](int64_t r, Pack<T, V>* x) {
        const int64_t off = r * p.cols + c0;
#pragma unroll
        for (int j = 0; j < N; ++j) {
            const int cls = arg_class<S>(p.cls, j);
            if (cls == kFull) {
                x[j] = ld_stream<T, V>(p.in[j] + off);
            } else if (cls == kRow) {
                const T v0 = __ldg(p.in[j] + r);
#pragma unroll
                for (int v = 0; v < V; ++v) x[j].x[v] = v0;
            } else {
                x[j] = xc[j];
            }
        }
    };
    int64_t r = int64_t(blockIdx.y) * p.tile_rows + ty;
    if (r >= p.rows) return;
    constexpr bool kPipe = fwd_pipeline<Body>();
    Pack<T, V> x[N];
    load_row(r, x);
    for (int k = 0; k < p.rpt; ++k) {
        const int64_t rn = r + p.ty;
        const bool has_next = k + 1 < p.rpt && rn < p.rows;
        Pack<T, V> xn[kPipe ? N : 1];
        if constexpr (kPipe)
            if (has_next) load_row(rn, xn);
        const int64_t off = r * p.cols + c0;
        if constexpr (kReal) {
            Pack<T, V> y[M];
#pragma unroll
            for (int v = 0; v < V; ++v) {
                T xi[N], yo[M];
#pragma unroll
                for (int j = 0; j < N; ++j) xi[j] = x[j].x[v];
                if constexpr (Body::kSelectForm && S::kStatic && !vec_eval_ok<Body, S>()) Body::template body_select<T>(xi, yo);
                else Body::template body<T>(xi, yo);
#pragma unroll
                for (int i = 0; i < M; ++i) y[i].x[v] = yo[i];
            }
#pragma unroll
            for (int i = 0; i < M; ++i)
                if (kDense || p.primal[i]) st_vec<T, V>(p.primal[i] + off, y[i]);
        } else {
            Pack<T, V> y[M];
            Pack<T, V> d[M * N];
            eval_cells<Body, T, V, S>(x, y, d, p.err, off);
#pragma unroll
            for (int i = 0; i < M; ++i) {
                if (kDense || p.primal[i]) st_vec<T, V>(p.primal[i] + off, y[i]);
#pragma unroll
                for (int j = 0; j < N; ++j)
                    if (kDense || p.partials[i * N + j]) st_vec<T, V>(p.partials[i * N + j] + off, d[i * N + j]);
            }
        }
        if (!has_next) break;
        if constexpr (kPipe) {
#pragma unroll
            for (int j = 0; j < N; ++j) x[j] = xn[j];
        } else {
            load_row(rn, x);
        }
        r = rn;
    }
}

// ------------------------------------------------------------- K2 params
template <int N, int M, class T>
struct Pull2DParams {
    const T* w[M];        // output adjoints (nullable)
    const T* D[M * N];    // cached partials (CacheForward)
    const T* in[N];       // inputs (RecomputeReverse)
    T* adj[N];            // input adjoint slots (nullable)
    int cls[N];
    int slot[N];          // index among active args of the same reduced class
    int row_j[N], col_j[N], scal_j[N];  // slot -> argument index
    uint32_t acc_mask;    // bit j: add into the existing slot
    int64_t rows, cols;
    int vcols;
    int txv_shift, ty, rpt;
    int prefetch;         // rows ahead whose streams are prefetched into L2 (0 = none)
    int64_t tile_rows;
    int n_row_tiles, n_col_tiles;
    int n_row_args, n_col_args, n_scalar_args;
    double* ws_row;       // [n_row_args][n_col_tiles][rows]
    double* ws_col;       // [n_col_args][n_row_tiles][cols]
    double* ws_scalar;    // [n_scalar_args][n_ctas]
    // Completion tickets of the in-kernel combination ([n_col_tiles] column
    // strips, [n_row_tiles] row tiles, [1] whole grid); null = K2f combines.
    unsigned int* tickets;
    int col_to_ws;        // column sums always leave fp64 partials (fused peer allreduce)
    unsigned long long* err;
};

template <class T>
__device__ __forceinline__ T finish(double s, const T* slot_ptr, bool accumulate) {
    return accumulate ? T(double(*slot_ptr) + s) : T(s);
}

// The cross-CTA combination of one group of up to 32 consecutive reduced
// elements (items [it0, it_end) of the row or column partials): lane =
// element, so every load is coalesced across the warp; the 8 warps split the
// tile partials into 8 contiguous groups whose sums are added in group order.
// Fixed association: bitwise run-to-run deterministic. Called uniformly by
// all threads of a CTA (it synchronises). Loads bypass L1 (__ldcg): inside
// K2 the partials were written by other CTAs of the same grid.
template <int N, int M, class T>
__device__ void combine_group(const Pull2DParams<N, M, T>& p, bool is_row, int64_t it0, int64_t it_end, double* part) {
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const int64_t it = it0 + lane, len = is_row ? p.rows : p.cols;
    const int n = is_row ? p.n_col_tiles : p.n_row_tiles;
    const bool valid = it < it_end;
    const int a = valid ? int(it / len) : 0;
    const int64_t e = valid ? it % len : 0;
    const double* base = (is_row ? p.ws_row : p.ws_col) + size_t(a) * n * len + e;
    const int per = (n + 7) / 8, q0 = warp * per, q1 = min(n, q0 + per);
    double acc = 0.0;
    if (valid) {
        int q = q0;
        for (; q + 8 <= q1; q += 8) {
            double v[8];
#pragma unroll
            for (int u = 0; u < 8; ++u) v[u] = __ldcg(base + size_t(q + u) * len);
#pragma unroll
            for (int u = 0; u < 8; ++u) acc += v[u];
        }
        for (; q < q1; ++q) acc += __ldcg(base + size_t(q) * len);
    }
    __syncthreads();  // part[] may still be read by a previous group
    part[warp * 32 + lane] = acc;
    __syncthreads();
    if (warp == 0 && valid) {
        double sum = 0.0;
#pragma unroll
        for (int g = 0; g < 8; ++g) sum += part[g * 32 + lane];
        const int j = is_row ? p.row_j[a] : p.col_j[a];
        p.adj[j][e] = finish<T>(sum, p.adj[j] + e, (p.acc_mask >> j) & 1u);
    }
}

// One scalar argument's combination over all CTAs' partials (strided sums,
// a fixed-shape tree). Called uniformly by all threads of a CTA.
template <int N, int M, class T>
__device__ void combine_scalar(const Pull2DParams<N, M, T>& p, int a, double* part) {
    const int64_t n_ctas = int64_t(p.n_row_tiles) * p.n_col_tiles;
    double acc = 0.0;
    for (int64_t q = threadIdx.x; q < n_ctas; q += kThreads) acc += __ldcg(p.ws_scalar + size_t(a) * n_ctas + q);
    __syncthreads();
    part[threadIdx.x] = acc;
    __syncthreads();
    for (int stride = kThreads / 2; stride > 0; stride >>= 1) {
        if (threadIdx.x < stride) part[threadIdx.x] += part[threadIdx.x + stride];
        __syncthreads();
    }
    if (threadIdx.x == 0) {
        const int j = p.scal_j[a];
        p.adj[j][0] = finish<T>(part[0], p.adj[j], (p.acc_mask >> j) & 1u);
    }
}

// In-kernel combination of one strip / row tile by its last-arriving CTA:
// the elements e in [e0, e1) of `count` reduced arguments (row or column
// partials), each summed over all n tiles in tile order. The CTA's threads
// work on all elements at once: with few elements, G contiguous tile groups
// per element (thread = (group, element)), the group sums then added in group
// order, so the association depends only on the sizes, never on arrival.
template <int N, int M, class T>
__device__ void combine_set(const Pull2DParams<N, M, T>& p, bool is_row, int count, int64_t e0, int64_t e1,
                            double* part) {
    const int64_t len = is_row ? p.rows : p.cols;
    const int n = is_row ? p.n_col_tiles : p.n_row_tiles;
    const int width = int(e1 - e0), n_el = count * width;
    int w = 1;
    while (w < n_el && w < kThreads) w <<= 1;
    const int G = min(kThreads / w, n);  // tile groups per element
    const int per = (n + G - 1) / G;
    for (int base = 0; base < n_el; base += w) {
        const int g = threadIdx.x / w, el = base + int(threadIdx.x % w);
        const bool valid = g < G && el < n_el;
        double acc = 0.0;
        int a = 0;
        int64_t e = 0;
        if (valid) {
            a = el / width;
            e = e0 + el % width;
            const double* src = (is_row ? p.ws_row : p.ws_col) + size_t(a) * n * len + e;
            const int q0 = g * per, q1 = min(n, q0 + per);
            int q = q0;
            for (; q + 8 <= q1; q += 8) {
                double v[8];
#pragma unroll
                for (int u = 0; u < 8; ++u) v[u] = __ldcg(src + size_t(q + u) * len);
#pragma unroll
                for (int u = 0; u < 8; ++u) acc += v[u];
            }
            for (; q < q1; ++q) acc += __ldcg(src + size_t(q) * len);
        }
        __syncthreads();
        if (valid) part[g * w + int(threadIdx.x % w)] = acc;
        __syncthreads();
        if (g == 0 && valid) {
            double sum = 0.0;
            for (int k = 0; k < G; ++k) sum += part[k * w + int(threadIdx.x % w)];
            const int j = is_row ? p.row_j[a] : p.col_j[a];
            p.adj[j][e] = finish<T>(sum, p.adj[j] + e, (p.acc_mask >> j) & 1u);
        }
    }
}

// Shared-memory layout of K2 (dynamic, doubles):
//   col_acc [n_col_args][kThreads][V]      per-thread column partials
//   row_acc [n_row_args][rpt*ty][wpr]      per-(row, warp) row partials
//   scal_acc[n_scalar_args][kThreads]      per-thread scalar partials
__host__ __device__ inline size_t pull_smem_doubles(int n_col, int n_row, int n_scal, int V, int rpt, int ty, int wpr) {
    return size_t(n_col) * kThreads * V + size_t(n_row) * rpt * ty * wpr + size_t(n_scal) * kThreads;
}

// K2: terms w_i * D_ij rounded to T exactly like backprop_diag's tensor_zip
// (mixed.hpp:34-38); FULL slots get the reference's element arithmetic,
// reduced slots an fp64 sum of those terms in a fixed order.
//
// kPipe (small grids, at most two CTAs per SM): the next row's streams are
// loaded into registers before the current row is reduced, so every thread
// keeps two rows of loads in flight (as K1 does); up to 128 registers, which
// costs no occupancy when the grid cannot fill more than two CTAs per SM.
// Reduction order is unchanged, so results are bit-identical to kPipe=false.
template <class Body, class T, int V, bool kRecompute, class S, bool kDense, bool kPipe = false>
__global__ void __launch_bounds__(kThreads, kPipe ? 2 : (kRecompute ? kRecomputeCtasPerSm : kCtasPerSm)) pull2d_kernel(const __grid_constant__ Pull2DParams<Body::kIn, Body::kOut, T> p) {
    constexpr int N = Body::kIn, M = Body::kOut;
    constexpr bool kAnyRow = !S::kStatic || S::has(kRow);
    constexpr bool kAnyCol = !S::kStatic || S::has(kCol);
    constexpr bool kAnyScal = !S::kStatic || S::has(kScalar);
    constexpr uint32_t kZeroPartials = kRecompute ? predicate_only_args<Body>() : 0u;
    extern __shared__ double smem[];
    pdl_wait();
    pdl_trigger();  // lets the finisher (if any) be scheduled; it waits for this grid to complete
    if constexpr (Body::kMayRaise && kRecompute) s_err_flag[threadIdx.x] = 0;

    const int tid = threadIdx.x;
    const int txv = 1 << p.txv_shift;
    const int tx = tid & (txv - 1);
    const int ty = tid >> p.txv_shift;
    const int lanes = txv < 32 ? txv : 32;          // lanes sharing a row in one warp
    const int wpr = txv > 32 ? txv >> 5 : 1;         // warps per row
    const int wir = (tid & (txv - 1)) >> 5;          // warp index within its row
    const int ct = blockIdx.x, rt = blockIdx.y;
    const int vc = (ct << p.txv_shift) + tx;
    const bool active = vc < p.vcols;
    const int64_t c0 = int64_t(vc) * V;
    const int trows = p.rpt * p.ty;                  // rows of this tile
    const int row_base = ty * wpr + wir;             // this thread's row_acc column

    double* col_acc = smem;
    double* row_acc = col_acc + size_t(p.n_col_args) * kThreads * V;
    double* scal_acc = row_acc + size_t(p.n_row_args) * trows * wpr;
    if constexpr (kAnyCol)  // each thread zeroes exactly the partials it accumulates (no barrier needed)
        for (int a = 0; a < p.n_col_args; ++a)
#pragma unroll
            for (int v = 0; v < V; ++v) col_acc[(size_t(a) * kThreads + tid) * V + v] = 0.0;
    if constexpr (kAnyScal)
        for (int a = 0; a < p.n_scalar_args; ++a) scal_acc[a * kThreads + tid] = 0.0;

    // broadcast inputs that do not depend on the row (recompute only)
    Pack<T, V> xc[N];
    if constexpr (kRecompute) {
#pragma unroll
        for (int j = 0; j < N; ++j) {
            const int cls = arg_class<S>(p.cls, j);
            if (active && cls == kCol) xc[j] = ld_ro<T, V>(p.in[j] + c0);
            if (cls == kScalar) {
                const T v0 = __ldg(p.in[j]);
#pragma unroll
                for (int v = 0; v < V; ++v) xc[j].x[v] = v0;
            }
        }
    }
    // One row's streamed operands: the output adjoints w_i and either the
    // cached partials D_ij or (recompute) the inputs x_j.
    constexpr int kStreams = kRecompute ? N : M * N;
    auto load_row = [&](int64_t r, Pack<T, V>* w, Pack<T, V>* q) {
        const int64_t off = r * p.cols + c0;
#pragma unroll
        for (int i = 0; i < M; ++i)
            if (kDense || p.w[i]) w[i] = ld_stream<T, V>(p.w[i] + off);
        if constexpr (kRecompute) {
#pragma unroll
            for (int j = 0; j < N; ++j) {
                const int cls = arg_class<S>(p.cls, j);
                if (cls == kFull) {
                    q[j] = ld_stream<T, V>(p.in[j] + off);
                } else if (cls == kRow) {
                    const T v0 = __ldg(p.in[j] + r);
#pragma unroll
                    for (int v = 0; v < V; ++v) q[j].x[v] = v0;
                } else {
                    q[j] = xc[j];
                }
            }
        } else {
#pragma unroll
            for (int i = 0; i < M; ++i)
#pragma unroll
                for (int j = 0; j < N; ++j)
                    if (kDense || (p.w[i] && p.adj[j])) q[i * N + j] = ld_stream<T, V>(p.D[i * N + j] + off);
        }
    };

    // L2 prefetch of a later row's streams (register-free lookahead; a
    // register double buffer would push the kernel below its resident CTAs)
    auto prefetch_row = [&](int64_t r) {
        const int64_t off = r * p.cols + c0;
#pragma unroll
        for (int i = 0; i < M; ++i)
            if (kDense || p.w[i]) prefetch_l2(p.w[i] + off);
        if constexpr (kRecompute) {
#pragma unroll
            for (int j = 0; j < N; ++j)
                if (arg_class<S>(p.cls, j) == kFull) prefetch_l2(p.in[j] + off);
        } else {
#pragma unroll
            for (int i = 0; i < M; ++i)
#pragma unroll
                for (int j = 0; j < N; ++j)
                    if (kDense || (p.w[i] && p.adj[j])) prefetch_l2(p.D[i * N + j] + off);
        }
    };

    // Compiled into the RecomputeReverse pullback of the registered signatures
    // only: in the cached pullback it gains at most 1% and its addresses spill
    // the all-FULL (divergence) signatures at 64 registers; the select-form
    // (per-cell branch) recompute has no registers to spare for them either.
    constexpr bool kPrefetch = kRecompute && S::kStatic && !(Body::kSelectForm && !vec_eval_ok<Body, S>());
    const int64_t r0 = int64_t(rt) * p.tile_rows + ty;
    Pack<T, V> wn[kPipe ? M : 1], qn[kPipe ? kStreams : 1];
    if constexpr (kPipe)
        if (active && r0 < p.rows) load_row(r0, wn, qn);
    // Every lane runs the same rpt iterations (rows past the end are masked),
    // so the ROW shuffles always see complete lane groups.
    for (int k = 0; k < p.rpt; ++k) {
        const int64_t r = r0 + int64_t(k) * p.ty;
        const bool live = active && r < p.rows;

        Pack<T, V> w[M], q[kStreams];
        if constexpr (kPipe) {
#pragma unroll
            for (int i = 0; i < M; ++i) w[i] = wn[i];
#pragma unroll
            for (int t = 0; t < kStreams; ++t) q[t] = qn[t];
            const int64_t rn = r + p.ty;
            if (active && k + 1 < p.rpt && rn < p.rows) load_row(rn, wn, qn);
        } else {
            if (live) load_row(r, w, q);
        }
        if (kPrefetch && k == 0 && active)  // behind the first row's loads
            for (int kk = 1; kk <= p.prefetch && kk < p.rpt; ++kk)
                if (r0 + int64_t(kk) * p.ty < p.rows) prefetch_row(r0 + int64_t(kk) * p.ty);
        const int64_t off = r * p.cols + c0;
        Pack<T, V> D[M * N];
        if constexpr (kRecompute) {
            if (live) eval_cells<Body, T, V, S>(q, static_cast<Pack<T, V>*>(nullptr), D, p.err, off);
        } else {
#pragma unroll
            for (int t = 0; t < M * N; ++t) D[t] = q[t];
        }
#pragma unroll
        for (int j = 0; j < N; ++j) {
            if (!kDense && !p.adj[j]) continue;
            const int cls = arg_class<S>(p.cls, j);
            const bool acc = !kDense && ((p.acc_mask >> j) & 1u);
            // RecomputeReverse: an argument that only feeds branch predicates
            // has structurally zero partials, so its terms are exact zeros and
            // are not formed (compile-time per unrolled j)
            const bool zero_d = (kZeroPartials >> j) & 1u;
            if (cls == kFull) {
                if (!live) continue;
                T* dst = p.adj[j] + off;
                Pack<T, V> out;
                if (acc) out = ld_stream<T, V>(dst);
#pragma unroll
                for (int v = 0; v < V; ++v) {
                    T a = acc ? out.x[v] : T(0);
                    if (!zero_d)
#pragma unroll
                        for (int i = 0; i < M; ++i)
                            if (kDense || p.w[i]) a = a + w[i].x[v] * D[i * N + j].x[v];
                    out.x[v] = a;
                }
                st_vec<T, V>(dst, out);
                continue;
            }
            if (zero_d) {  // reduced class, all terms zero: the row sum is 0, column / scalar sums unchanged
                if constexpr (kAnyRow)
                    if (cls == kRow && (tid & (lanes - 1)) == 0)
                        row_acc[(arg_slot<S, kDense>(p.slot, j) * trows + k * p.ty) * wpr + row_base] = 0.0;
                continue;
            }
            // reduced classes: fp64 sum of the rounded terms. A dead row adds
            // nothing to column / scalar partials (skipped: adding +0.0 to a
            // sum that starts at +0.0 changes no bit); row sums need the zero
            // for the lane shuffle. Each cell's sum starts from its first term
            // rather than 0.0 + term: every sum these feed starts from +0.0,
            // so the results are bit-identical and the adds are saved.
            if (cls != kRow && !live) continue;
            double s[V];
#pragma unroll
            for (int v = 0; v < V; ++v) {
                s[v] = 0.0;
                bool first = true;
#pragma unroll
                for (int i = 0; i < M; ++i)
                    if (kDense || p.w[i]) {
                        const double t = double(T(w[i].x[v] * D[i * N + j].x[v]));
                        s[v] = first ? t : s[v] + t;
                        first = false;
                    }
                if (cls == kRow && !live) s[v] = 0.0;
            }
            if (cls == kCol) {
                if constexpr (kAnyCol) {
                    double* ca = col_acc + (size_t(arg_slot<S, kDense>(p.slot, j)) * kThreads + tid) * V;
#pragma unroll
                    for (int v = 0; v < V; ++v) ca[v] += s[v];
                }
            } else if (cls == kScalar) {
                if constexpr (kAnyScal) {
                    double t = 0.0;
#pragma unroll
                    for (int v = 0; v < V; ++v) t += s[v];
                    scal_acc[arg_slot<S, kDense>(p.slot, j) * kThreads + tid] += t;
                }
            } else if constexpr (kAnyRow) {  // kRow: lanes of this row in this warp
                double t = 0.0;
#pragma unroll
                for (int v = 0; v < V; ++v) t += s[v];
                // xor offsets below `lanes` stay inside the row's aligned lane
                // group; unrolled with a warp-uniform predicate (no loop)
#pragma unroll
                for (int o = 16; o > 0; o >>= 1)
                    if (o < lanes) t += __shfl_xor_sync(0xffffffffu, t, o);
                if ((tid & (lanes - 1)) == 0)
                    row_acc[(arg_slot<S, kDense>(p.slot, j) * trows + k * p.ty) * wpr + row_base] = t;
            }
        }
        // issued after this row's registers are retired (fewest live values)
        if (kPrefetch && p.prefetch > 0 && active && k + 1 + p.prefetch < p.rpt) {
            const int64_t rp = r + int64_t(1 + p.prefetch) * p.ty;
            if (rp < p.rows) prefetch_row(rp);
        }
    }
    if constexpr (!kAnyRow && !kAnyCol && !kAnyScal) return;
    else {
        __syncthreads();
        const int64_t n_ctas = int64_t(p.n_row_tiles) * p.n_col_tiles;
        // ---- CTA-level combination (fixed order)
        if constexpr (kAnyRow) {
            for (int item = tid; item < p.n_row_args * trows; item += kThreads) {
                const int a = item / trows, lr = item % trows;
                const int kk = lr / p.ty, yy = lr % p.ty;
                const int64_t r = int64_t(rt) * p.tile_rows + yy + int64_t(kk) * p.ty;
                if (r >= p.rows) continue;
                double sacc = 0.0;
                for (int q = 0; q < wpr; ++q) sacc += row_acc[(size_t(a) * trows + lr) * wpr + q];
                const int j = p.row_j[a];
                if (p.n_col_tiles == 1) p.adj[j][r] = finish<T>(sacc, p.adj[j] + r, (p.acc_mask >> j) & 1u);
                else p.ws_row[(size_t(a) * p.n_col_tiles + ct) * p.rows + r] = sacc;
            }
        }
        const int ccols = txv * V;
        if constexpr (kAnyCol) {
            for (int item = tid; item < p.n_col_args * ccols; item += kThreads) {
                const int a = item / ccols, cc = item % ccols;
                const int txi = cc / V, v = cc % V;
                const int64_t c = int64_t(ct) * ccols + cc;
                if (c >= p.cols) continue;
                double sacc = 0.0;
                for (int y = 0; y < p.ty; ++y) sacc += col_acc[(size_t(a) * kThreads + (y << p.txv_shift) + txi) * V + v];
                const int j = p.col_j[a];
                if (p.n_row_tiles == 1 && !p.col_to_ws) p.adj[j][c] = finish<T>(sacc, p.adj[j] + c, (p.acc_mask >> j) & 1u);
                else p.ws_col[(size_t(a) * p.n_row_tiles + rt) * p.cols + c] = sacc;
            }
        }
        if constexpr (kAnyScal) {
            for (int a = 0; a < p.n_scalar_args; ++a) {
                __syncthreads();
                for (int stride = kThreads / 2; stride > 0; stride >>= 1) {
                    if (tid < stride) scal_acc[a * kThreads + tid] += scal_acc[a * kThreads + tid + stride];
                    __syncthreads();
                }
                if (tid == 0) {
                    const double sacc = scal_acc[a * kThreads];
                    const int j = p.scal_j[a];
                    if (n_ctas == 1) p.adj[j][0] = finish<T>(sacc, p.adj[j], (p.acc_mask >> j) & 1u);
                    else p.ws_scalar[size_t(a) * n_ctas + size_t(rt) * p.n_col_tiles + ct] = sacc;
                }
            }
        }
        // ---- cross-CTA combination inside K2 (distributed completion
        // tickets): the last CTA of each column strip combines the strip's
        // column partials over all row tiles, the last CTA of each row tile
        // the tile's row partials over all column tiles, the last CTA of the
        // grid the scalar partials; each resets its ticket to zero for the
        // next pullback on this workspace. Writers publish with a fence
        // before their ticket; the summation order is fixed by tile index,
        // not by arrival, so results are bitwise deterministic.
        if (p.tickets) {
            __shared__ unsigned int s_last[3];
            __shared__ double part[kThreads];
            const bool col_x = kAnyCol && p.n_row_tiles > 1 && p.n_col_args > 0;
            const bool row_x = kAnyRow && p.n_col_tiles > 1 && p.n_row_args > 0;
            const bool scal_x = kAnyScal && n_ctas > 1 && p.n_scalar_args > 0;
            __syncthreads();  // every partial of this CTA is written
            if (tid == 0) {
                __threadfence();
                s_last[0] = col_x && atomicAdd(p.tickets + ct, 1u) == unsigned(p.n_row_tiles - 1);
                s_last[1] = row_x && atomicAdd(p.tickets + p.n_col_tiles + rt, 1u) == unsigned(p.n_col_tiles - 1);
                s_last[2] = scal_x && atomicAdd(p.tickets + p.n_col_tiles + p.n_row_tiles, 1u) == unsigned(n_ctas - 1);
                if (s_last[0] | s_last[1] | s_last[2]) __threadfence();
            }
            __syncthreads();
            if (s_last[0]) {
                const int64_t c0 = int64_t(ct) * ccols;
                combine_set(p, false, p.n_col_args, c0, min(p.cols, c0 + ccols), part);
                if (tid == 0) p.tickets[ct] = 0u;
            }
            if (s_last[1]) {
                const int64_t r0t = int64_t(rt) * p.tile_rows;
                combine_set(p, true, p.n_row_args, r0t, min(p.rows, r0t + p.tile_rows), part);
                if (tid == 0) p.tickets[p.n_col_tiles + rt] = 0u;
            }
            if (s_last[2]) {
                for (int a = 0; a < p.n_scalar_args; ++a) combine_scalar(p, a, part);
                if (tid == 0) p.tickets[p.n_col_tiles + p.n_row_tiles] = 0u;
            }
        }
    }
}

// K2f: the same cross-CTA combination as a separate, programmatically
// dependent launch (it waits for K2's grid, so K2 needs no tickets): one CTA
// per group of 32 reduced elements, one per scalar argument. Used when the
// caller's workspace has no ticket region (pull_layout, tickets = false).
template <int N, int M, class T>
__global__ void __launch_bounds__(kThreads) pull_finish_kernel(const __grid_constant__ Pull2DParams<N, M, T> p) {
    pdl_wait();
    __shared__ double part[kThreads];
    const int64_t row_items = p.n_col_tiles > 1 ? int64_t(p.n_row_args) * p.rows : 0;
    const int64_t col_items = p.n_row_tiles > 1 ? int64_t(p.n_col_args) * p.cols : 0;
    const int64_t row_blocks = (row_items + 31) / 32, col_blocks = (col_items + 31) / 32;
    const int64_t b = blockIdx.x;
    if (b >= row_blocks + col_blocks) {
        combine_scalar(p, int(b - row_blocks - col_blocks), part);
        return;
    }
    const bool is_row = b < row_blocks;
    combine_group(p, is_row, (is_row ? b : b - row_blocks) * 32, is_row ? row_items : col_items, part);
}

// ------------------------------------------------ fused peer allreduce
__device__ __forceinline__ unsigned long long ld_acquire_sys(const unsigned long long* p) {
    unsigned long long v;
    asm volatile("ld.acquire.sys.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
    return v;
}
__device__ __forceinline__ void st_release_sys(unsigned long long* p, unsigned long long v) {
    asm volatile("st.release.sys.global.u64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}
__device__ __forceinline__ unsigned long long global_ns() {
    unsigned long long t;
    asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
    return t;
}

// K2f-AR: K2's cross-CTA combination fused with the allreduce of the
// batch-broadcast (column-class) adjoints over a peer-memory group, in place
// of K2f + ncclAllReduce. Row-class groups are combined locally as in K2f.
// Each column group's CTA sums its 32 elements' tile partials (fp64, fixed
// order) and stores them straight into slot `rank` of EVERY rank's buffer
// (NVLink peer stores; the buffers were exchanged once by CUDA IPC). The last
// arriving CTA publishes a step-counter flag to every rank (release, system
// scope), waits for every rank's flag (acquire), then adds the world's slots
// in rank order — identical bits on every rank — and writes the adjoints
// (one fp32 rounding of the fp64 world sum). Double-buffered by step parity:
// a rank can run at most one step ahead of another, so a fast rank's next
// stores never land in the slots being read. A peer that never arrives traps
// after 30 s instead of hanging the device.
template <int N, int M, class T>
__global__ void __launch_bounds__(kThreads) pull_finish_ar_kernel(const __grid_constant__ Pull2DParams<N, M, T> p,
                                                                  const __grid_constant__ bcad_cu_impl::PeerParams q) {
    pdl_wait();
    __shared__ double part[kThreads];
    __shared__ unsigned long long s_epoch;
    __shared__ int s_last;
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const int64_t row_items = p.n_col_tiles > 1 ? int64_t(p.n_row_args) * p.rows : 0;
    const int64_t col_items = int64_t(p.n_col_args) * p.cols;
    const int64_t row_blocks = (row_items + 31) / 32, col_blocks = (col_items + 31) / 32;
    const int64_t b = blockIdx.x;
    if (b < row_blocks) {
        combine_group(p, true, b * 32, row_items, part);
        return;
    }
    if (threadIdx.x == 0) s_epoch = *reinterpret_cast<volatile unsigned long long*>(q.epoch);
    // local fp64 sums of this group's 32 column elements (combine_group's order)
    const int64_t it = (b - row_blocks) * 32 + lane;
    const bool valid = it < col_items;
    const int a = valid ? int(it / p.cols) : 0;
    const int64_t e = valid ? it % p.cols : 0;
    const int n = p.n_row_tiles;
    const double* base = p.ws_col + size_t(a) * n * p.cols + e;
    const int per = (n + 7) / 8, q0 = warp * per, q1 = min(n, q0 + per);
    double acc = 0.0;
    if (valid)
        for (int k = q0; k < q1; ++k) acc += base[size_t(k) * p.cols];
    part[warp * 32 + lane] = acc;
    __syncthreads();
    const unsigned long long next = s_epoch + 1;
    const size_t par = size_t(next & 1u);
    if (warp == 0 && valid) {
        double sum = 0.0;
#pragma unroll
        for (int g = 0; g < 8; ++g) sum += part[g * 32 + lane];
        for (int k = 0; k < q.world; ++k) q.slots[k][(par * q.world + q.rank) * size_t(q.n) + it] = sum;
        __threadfence_system();
    }
    __syncthreads();
    if (threadIdx.x == 0) s_last = atomicAdd(q.arrive, 1u) == unsigned(col_blocks - 1);
    __syncthreads();
    if (!s_last) return;
    // the last CTA of this rank: publish, wait for every rank, add in rank order
    if (threadIdx.x == 0) __threadfence_system();
    __syncthreads();
    if (threadIdx.x < q.world) {
        st_release_sys(q.flags[threadIdx.x] + q.rank, next);
        const unsigned long long t0 = global_ns();
        while (ld_acquire_sys(q.flags[q.rank] + threadIdx.x) < next)
            if (global_ns() - t0 > 30000000000ull) __trap();  // a peer never arrived
    }
    __syncthreads();
    const double* mine = q.slots[q.rank] + par * q.world * size_t(q.n);
    for (int64_t i = threadIdx.x; i < col_items; i += kThreads) {
        double sum = 0.0;
        for (int k = 0; k < q.world; ++k) sum += __ldcv(mine + size_t(k) * q.n + i);
        const int aa = int(i / p.cols);
        const int64_t c = i % p.cols;
        const int j = p.col_j[aa];
        p.adj[j][c] = finish<T>(sum, p.adj[j] + c, (p.acc_mask >> j) & 1u);
    }
    __syncthreads();
    if (threadIdx.x == 0) {
        *q.arrive = 0u;
        *reinterpret_cast<volatile unsigned long long*>(q.epoch) = next;
    }
}

// Blocks of pull_finish_kernel for a tiling (0 = nothing to combine).
inline int64_t pull_finish_blocks(int64_t rows, int64_t cols, int n_row_tiles, int n_col_tiles, int n_row_args,
                                  int n_col_args, int n_scalar_args) {
    const int64_t ri = n_col_tiles > 1 ? int64_t(n_row_args) * rows : 0;
    const int64_t ci = n_row_tiles > 1 ? int64_t(n_col_args) * cols : 0;
    const int64_t si = int64_t(n_row_tiles) * n_col_tiles > 1 ? n_scalar_args : 0;
    return (ri + 31) / 32 + (ci + 31) / 32 + si;
}

// ------------------------------------------------------- generic kernels
template <int N, int M, class T>
struct GenParams {
    const T* in[N];
    int64_t strides[N][kMaxRank];
    int64_t arg_vol[N];
    int out_rank;
    int64_t out_dims[kMaxRank];
    int64_t vol;
    T* primal[M];
    T* partials[M * N];
    // pullback
    const T* w[M];
    const T* D[M * N];
    T* adj[N];
    uint32_t acc_mask;
    int64_t adj_offset[N + 1];  // prefix sums of arg volumes over active adj
    // segmented reductions (pull_generic_seg_kernel): segments per element of
    // argument j (0 = not segmented), prefix sums of arg_vol[j] * segs[j],
    // and the fp64 partials [item][segment]
    int segs[N];
    int64_t seg_offset[N + 1];
    double* seg_ws;
    // column-mode segmented arguments (full along the last axis): a CTA per
    // (kThreads consecutive elements, segment); first CTA of each argument
    uint32_t seg_col_mask;
    int64_t seg_block[N + 1];
    unsigned long long* err;
    unsigned long long* tcount;  // census kernel: transcendental counter slots
};

template <int N, int M, class T>
__device__ __forceinline__ void decode_offsets(const GenParams<N, M, T>& p, int64_t flat, int64_t* off) {
#pragma unroll
    for (int j = 0; j < N; ++j) off[j] = 0;
    if (p.vol <= 0xffffffffll) {  // 32-bit index arithmetic (64-bit division costs ~4x the instructions)
        uint32_t f = uint32_t(flat);
        for (int k = p.out_rank - 1; k >= 0; --k) {
            const uint32_t len = uint32_t(p.out_dims[k]);
            const uint32_t c = f % len;
            f /= len;
#pragma unroll
            for (int j = 0; j < N; ++j) off[j] += int64_t(c) * p.strides[j][k];
        }
        return;
    }
    for (int k = p.out_rank - 1; k >= 0; --k) {
        const int64_t len = p.out_dims[k];
        const int64_t c = flat % len;
        flat /= len;
#pragma unroll
        for (int j = 0; j < N; ++j) off[j] += c * p.strides[j][k];
    }
}

template <class Body, class T, bool kReal>
__global__ void __launch_bounds__(kThreads) fwd_generic_kernel(const __grid_constant__ GenParams<Body::kIn, Body::kOut, T> p) {
    constexpr int N = Body::kIn, M = Body::kOut;
    if constexpr (Body::kMayRaise && !kReal) s_err_flag[threadIdx.x] = 0;
    for (int64_t cell = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; cell < p.vol;
         cell += int64_t(gridDim.x) * blockDim.x) {
        int64_t off[N];
        decode_offsets<N, M, T>(p, cell, off);
        if constexpr (kReal) {
            T xi[N], yo[M];
#pragma unroll
            for (int j = 0; j < N; ++j) xi[j] = p.in[j][off[j]];
            Body::template body<T>(xi, yo);
#pragma unroll
            for (int i = 0; i < M; ++i)
                if (p.primal[i]) p.primal[i][cell] = yo[i];
        } else {
            Dual<T, N> xi[N], yo[M];
#pragma unroll
            for (int j = 0; j < N; ++j) {
                xi[j] = Dual<T, N>::seeded(p.in[j][off[j]], j);
            }
            Body::template body<Dual<T, N>>(xi, yo);
            if constexpr (Body::kMayRaise) report_error(p.err, cell);
#pragma unroll
            for (int i = 0; i < M; ++i) {
                if (p.primal[i]) p.primal[i][cell] = yo[i].v;
#pragma unroll
                for (int j = 0; j < N; ++j)
                    if (p.partials[i * N + j]) p.partials[i * N + j][cell] = yo[i].d[j];
            }
        }
    }
}

// Generic forward, V cells per thread along the output's last axis (when
// its length is a multiple of V and every argument is contiguous or
// broadcast along it): one offset decode per V cells, 128-bit loads of the
// arguments full along the last axis (read-only loads for those re-read
// through broadcasting), 128-bit stores of the primal and the partials.
template <class Body, class T, int V, bool kReal>
__global__ void __launch_bounds__(kThreads) fwd_generic_vec_kernel(const __grid_constant__ GenParams<Body::kIn, Body::kOut, T> p) {
    constexpr int N = Body::kIn, M = Body::kOut;
    if constexpr (Body::kMayRaise && !kReal) s_err_flag[threadIdx.x] = 0;
    const int last = p.out_rank - 1;
    const int64_t nv = p.vol / V;
    for (int64_t v = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; v < nv; v += int64_t(gridDim.x) * blockDim.x) {
        const int64_t cell = v * V;
        int64_t off[N];
        decode_offsets<N, M, T>(p, cell, off);
        Pack<T, V> x[N];
#pragma unroll
        for (int j = 0; j < N; ++j) {
            if (p.strides[j][last] == 0) {
                const T s = __ldg(p.in[j] + off[j]);
#pragma unroll
                for (int u = 0; u < V; ++u) x[j].x[u] = s;
            } else if (p.arg_vol[j] == p.vol) {
                x[j] = ld_stream<T, V>(p.in[j] + off[j]);
            } else {
                x[j] = ld_ro<T, V>(p.in[j] + off[j]);
            }
        }
        if constexpr (kReal) {
            Pack<T, V> y[M];
#pragma unroll
            for (int u = 0; u < V; ++u) {
                T xi[N], yo[M];
#pragma unroll
                for (int j = 0; j < N; ++j) xi[j] = x[j].x[u];
                Body::template body<T>(xi, yo);
#pragma unroll
                for (int i = 0; i < M; ++i) y[i].x[u] = yo[i];
            }
#pragma unroll
            for (int i = 0; i < M; ++i)
                if (p.primal[i]) st_vec<T, V>(p.primal[i] + cell, y[i]);
        } else {
            Pack<T, V> y[M], d[M * N];
            eval_cells<Body, T, V, DynSig>(x, y, d, p.err, cell);
#pragma unroll
            for (int i = 0; i < M; ++i) {
                if (p.primal[i]) st_vec<T, V>(p.primal[i] + cell, y[i]);
#pragma unroll
                for (int j = 0; j < N; ++j)
                    if (p.partials[i * N + j]) st_vec<T, V>(p.partials[i * N + j] + cell, d[i * N + j]);
            }
        }
    }
}

// Generic pullback of the arguments of the output's full shape (p.adj set
// for exactly those): their adjoint is elementwise, sum_i w_i (.) D_ij in
// the element type in output order, as the thread-per-element kernel forms
// it (cnt = 1), V cells per thread, each output's seed read once for all of
// them. RecomputeReverse re-evaluates D as fwd_generic_vec_kernel does.
template <class Body, class T, int V, bool kRecompute>
__global__ void __launch_bounds__(kThreads) pull_generic_full_kernel(const __grid_constant__ GenParams<Body::kIn, Body::kOut, T> p) {
    constexpr int N = Body::kIn, M = Body::kOut;
    if constexpr (Body::kMayRaise && kRecompute) s_err_flag[threadIdx.x] = 0;
    const int last = p.out_rank - 1;
    const int64_t nv = p.vol / V;
    for (int64_t v = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; v < nv; v += int64_t(gridDim.x) * blockDim.x) {
        const int64_t cell = v * V;
        Pack<T, V> w[M];
#pragma unroll
        for (int i = 0; i < M; ++i)
            if (p.w[i]) w[i] = ld_stream<T, V>(p.w[i] + cell);
        Pack<T, V> d[M * N];
        if constexpr (kRecompute) {
            int64_t off[N];
            decode_offsets<N, M, T>(p, cell, off);
            Pack<T, V> x[N];
#pragma unroll
            for (int j = 0; j < N; ++j) {
                if (p.strides[j][last] == 0) {
                    const T s = __ldg(p.in[j] + off[j]);
#pragma unroll
                    for (int u = 0; u < V; ++u) x[j].x[u] = s;
                } else if (p.arg_vol[j] == p.vol) {
                    x[j] = ld_stream<T, V>(p.in[j] + off[j]);
                } else {
                    x[j] = ld_ro<T, V>(p.in[j] + off[j]);
                }
            }
            eval_cells<Body, T, V, DynSig>(x, static_cast<Pack<T, V>*>(nullptr), d, p.err, cell);
        }
#pragma unroll
        for (int j = 0; j < N; ++j) {
            if (!p.adj[j]) continue;
            Pack<T, V> out;
            if ((p.acc_mask >> j) & 1u) out = ld_stream<T, V>(p.adj[j] + cell);
            else
#pragma unroll
                for (int u = 0; u < V; ++u) out.x[u] = T(0);
#pragma unroll
            for (int i = 0; i < M; ++i) {
                if (!p.w[i]) continue;
                Pack<T, V> dj;
                if constexpr (kRecompute) dj = d[i * N + j];
                else dj = ld_stream<T, V>(p.D[i * N + j] + cell);
#pragma unroll
                for (int u = 0; u < V; ++u) out.x[u] = out.x[u] + T(w[i].x[u] * dj.x[u]);
            }
            st_vec<T, V>(p.adj[j] + cell, out);
        }
    }
}

// Generic pullback. kWarp = false: one thread per element e of each input j
// walks the output cells that map onto e (the broadcast axes of j,
// row-major) and sums the terms. kWarp = true (arguments reduced over >= 32
// cells): one warp per element, lanes take every 32nd cell, fixed-order
// butterfly — the same fp64 sum of the same rounded terms, in parallel.
template <class Body, class T, bool kRecompute, bool kWarp>
__global__ void __launch_bounds__(kThreads) pull_generic_kernel(const __grid_constant__ GenParams<Body::kIn, Body::kOut, T> p) {
    constexpr int N = Body::kIn, M = Body::kOut;
    if constexpr (Body::kMayRaise && kRecompute) s_err_flag[threadIdx.x] = 0;
    const int64_t total = p.adj_offset[N];
    const int lane = threadIdx.x & 31;
    const int64_t first = kWarp ? (blockIdx.x * int64_t(blockDim.x) + threadIdx.x) / 32
                                : blockIdx.x * int64_t(blockDim.x) + threadIdx.x;
    const int64_t step = kWarp ? int64_t(gridDim.x) * blockDim.x / 32 : int64_t(gridDim.x) * blockDim.x;
    for (int64_t g = first; g < total; g += step) {
        int j = 0;
        while (j + 1 < N && g >= p.adj_offset[j + 1]) ++j;
        const int64_t e = g - p.adj_offset[j];
        // arg coordinates of e on the output axes; broadcast axes enumerate
        int64_t base[kMaxRank], cnt = 1;
        int nb = 0;
        int bax[kMaxRank];
        {
            int64_t rem = e;
            for (int k = p.out_rank - 1; k >= 0; --k) {
                if (p.strides[j][k] != 0) {
                    const int64_t len = p.out_dims[k];
                    base[k] = rem % len;
                    rem /= len;
                } else {
                    base[k] = 0;
                }
            }
            for (int k = 0; k < p.out_rank; ++k)
                if (p.strides[j][k] == 0 && p.out_dims[k] > 1) {
                    bax[nb++] = k;
                    cnt *= p.out_dims[k];
                }
        }
        // sum over outputs of the rounded terms w_i * D_ij at output cell `flat`
        auto cell_terms = [&](int64_t flat, T* exact_out) -> double {
            T dj[M];
            if constexpr (kRecompute) {
                int64_t off[N];
                decode_offsets<N, M, T>(p, flat, off);
                Dual<T, N> xi[N], yo[M];
#pragma unroll
                for (int jj = 0; jj < N; ++jj) xi[jj] = Dual<T, N>::seeded(p.in[jj][off[jj]], jj);
                Body::template body<Dual<T, N>>(xi, yo);
                if constexpr (Body::kMayRaise) report_error(p.err, flat);
#pragma unroll
                for (int i = 0; i < M; ++i) {
                    T v = T(0);
#pragma unroll
                    for (int jj = 0; jj < N; ++jj)
                        if (jj == j) v = yo[i].d[jj];
                    dj[i] = v;
                }
            } else {
#pragma unroll
                for (int i = 0; i < M; ++i) dj[i] = p.w[i] ? p.D[i * N + j][flat] : T(0);
            }
            double sum = 0.0;
#pragma unroll
            for (int i = 0; i < M; ++i) {
                if (!p.w[i]) continue;
                const T term = p.w[i][flat] * dj[i];
                if (exact_out) *exact_out = *exact_out + term;
                else sum += double(term);
            }
            return sum;
        };
        const bool acc = (p.acc_mask >> j) & 1u;
        int64_t coord[kMaxRank];
        for (int k = 0; k < p.out_rank; ++k) coord[k] = base[k];
        if constexpr (kWarp) {
            double sum = 0.0;
            for (int64_t q = lane; q < cnt; q += 32) {
                int64_t rem = q;  // q -> coordinates on the broadcast axes, last fastest
                for (int b2 = nb - 1; b2 >= 0; --b2) {
                    const int k = bax[b2];
                    coord[k] = rem % p.out_dims[k];
                    rem /= p.out_dims[k];
                }
                int64_t flat = 0;
                for (int k = 0; k < p.out_rank; ++k) flat = flat * p.out_dims[k] + coord[k];
                sum += cell_terms(flat, nullptr);
            }
#pragma unroll
            for (int o = 16; o > 0; o >>= 1) sum += __shfl_xor_sync(0xffffffffu, sum, o);
            if (lane == 0) p.adj[j][e] = acc ? T(double(p.adj[j][e]) + sum) : T(sum);
        } else {
            T exact = acc ? p.adj[j][e] : T(0);
            double sum = 0.0;
            for (int64_t q = 0; q < cnt; ++q) {
                int64_t flat = 0;
                for (int k = 0; k < p.out_rank; ++k) flat = flat * p.out_dims[k] + coord[k];
                sum += cell_terms(flat, cnt == 1 ? &exact : nullptr);
                // odometer over the broadcast axes, last axis fastest
                for (int b2 = nb - 1; b2 >= 0; --b2) {
                    const int k = bax[b2];
                    if (++coord[k] < p.out_dims[k]) break;
                    coord[k] = 0;
                }
            }
            if (cnt == 1) p.adj[j][e] = exact;
            else p.adj[j][e] = acc ? T(double(p.adj[j][e]) + sum) : T(sum);
        }
    }
}

// Generic pullback, arguments reduced over many output cells, cut into
// `segs` contiguous segments of each element's broadcast cells (row-major,
// last broadcast axis fastest) whose fp64 partials pull_generic_seg_finish
// adds in segment order. Two CTA shapes, chosen per argument:
//  - row mode (reduced along the last axis, >= kSegMinCells cells): one CTA
//    per (element, segment); threads stride the segment, so warps read
//    consecutive cells; then a fixed-shape shared-memory tree;
//  - column mode (full along the last axis): one CTA per (kThreads
//    consecutive elements, segment); each thread walks its element's segment
//    in order, so warps read consecutive elements of the same broadcast cell.
// Either way a fixed association of the same rounded terms; bitwise
// run-to-run deterministic.
template <class Body, class T, bool kRecompute>
__device__ __forceinline__ double generic_cell_term(const GenParams<Body::kIn, Body::kOut, T>& p, int j, int64_t flat) {
    constexpr int N = Body::kIn, M = Body::kOut;
    T dj[M];
    if constexpr (kRecompute) {
        int64_t off[N];
        decode_offsets<N, M, T>(p, flat, off);
        Dual<T, N> xi[N], yo[M];
#pragma unroll
        for (int jj = 0; jj < N; ++jj) xi[jj] = Dual<T, N>::seeded(p.in[jj][off[jj]], jj);
        Body::template body<Dual<T, N>>(xi, yo);
        if constexpr (Body::kMayRaise) report_error(p.err, flat);
#pragma unroll
        for (int i = 0; i < M; ++i) {
            T v = T(0);
#pragma unroll
            for (int jj = 0; jj < N; ++jj)
                if (jj == j) v = yo[i].d[jj];
            dj[i] = v;
        }
    } else {
#pragma unroll
        for (int i = 0; i < M; ++i) dj[i] = p.w[i] ? p.D[i * N + j][flat] : T(0);
    }
    double sum = 0.0;
#pragma unroll
    for (int i = 0; i < M; ++i)
        if (p.w[i]) sum += double(T(p.w[i][flat] * dj[i]));
    return sum;
}

template <class Body, class T, bool kRecompute>
__global__ void __launch_bounds__(kThreads) pull_generic_seg_kernel(const __grid_constant__ GenParams<Body::kIn, Body::kOut, T> p) {
    constexpr int N = Body::kIn;
    if constexpr (Body::kMayRaise && kRecompute) s_err_flag[threadIdx.x] = 0;
    __shared__ double part[kThreads];
    const int64_t b = blockIdx.x;
    int j = 0;
    while (j + 1 < N && b >= p.seg_block[j + 1]) ++j;
    const int S = p.segs[j];
    const bool column = (p.seg_col_mask >> j) & 1u;
    const int64_t local = b - p.seg_block[j];
    int64_t e;
    int seg;
    if (column) {
        seg = int(local % S);
        e = (local / S) * kThreads + threadIdx.x;
        if (e >= p.arg_vol[j]) return;  // no CTA-wide sync below in column mode
    } else {
        e = local / S;
        seg = int(local % S);
    }
    // the element's coordinates on the axes where argument j is full, and the
    // broadcast axes it is summed over
    int64_t coord[kMaxRank], ostride[kMaxRank];
    int bax[kMaxRank];
    int nb = 0;
    int64_t cnt = 1, flat0 = 0;
    {
        int64_t rem = e, os = 1;
        for (int k = p.out_rank - 1; k >= 0; --k) {
            ostride[k] = os;
            os *= p.out_dims[k];
            if (p.strides[j][k] != 0) {
                coord[k] = rem % p.out_dims[k];
                rem /= p.out_dims[k];
            } else {
                coord[k] = 0;
            }
            flat0 += coord[k] * ostride[k];
        }
        for (int k = 0; k < p.out_rank; ++k)
            if (p.strides[j][k] == 0 && p.out_dims[k] > 1) {
                bax[nb++] = k;
                cnt *= p.out_dims[k];
            }
    }
    const int64_t q0 = cnt * seg / S, q1 = cnt * (seg + 1) / S;
    double sum = 0.0;
    if (column) {
        // odometer over the broadcast axes from cell q0, the flat index kept
        // incrementally; four cells' loads in flight before they are summed
        int64_t c[kMaxRank];
        int64_t flat = flat0;
        {
            int64_t rem = q0;
            for (int b2 = nb - 1; b2 >= 0; --b2) {
                const int k = bax[b2];
                c[k] = rem % p.out_dims[k];
                rem /= p.out_dims[k];
                flat += c[k] * ostride[k];
            }
        }
        auto advance = [&]() {
            for (int b2 = nb - 1; b2 >= 0; --b2) {
                const int k = bax[b2];
                flat += ostride[k];
                if (++c[k] < p.out_dims[k]) return;
                flat -= c[k] * ostride[k];
                c[k] = 0;
            }
        };
        int64_t q = q0;
        for (; q + 4 <= q1; q += 4) {
            int64_t f[4];
#pragma unroll
            for (int u = 0; u < 4; ++u) {
                f[u] = flat;
                advance();
            }
            double t[4];
#pragma unroll
            for (int u = 0; u < 4; ++u) t[u] = generic_cell_term<Body, T, kRecompute>(p, j, f[u]);
#pragma unroll
            for (int u = 0; u < 4; ++u) sum += t[u];
        }
        for (; q < q1; ++q) {
            sum += generic_cell_term<Body, T, kRecompute>(p, j, flat);
            advance();
        }
        p.seg_ws[p.seg_offset[j] + e * S + seg] = sum;
            return;
    }
    {
        // threads stride the segment by kThreads cells: the odometer advances
        // by kThreads with a division only when an axis wraps; four cells'
        // loads in flight before they are summed (in q order)
        int64_t c[kMaxRank];
        int64_t flat = flat0;
        {
            int64_t rem = q0 + threadIdx.x;
            for (int b2 = nb - 1; b2 >= 0; --b2) {
                const int k = bax[b2];
                c[k] = rem % p.out_dims[k];
                rem /= p.out_dims[k];
                flat += c[k] * ostride[k];
            }
        }
        auto advance = [&]() {
            int64_t step = kThreads;
            for (int b2 = nb - 1; b2 >= 0 && step; --b2) {
                const int k = bax[b2];
                const int64_t len = p.out_dims[k];
                int64_t cn = c[k] + step;
                step = 0;
                if (cn >= len) {
                    step = cn / len;
                    cn -= step * len;
                }
                flat += (cn - c[k]) * ostride[k];
                c[k] = cn;
            }
        };
        int64_t q = q0 + threadIdx.x;
        for (; q + 3 * kThreads < q1; q += 4 * kThreads) {
            int64_t f[4];
#pragma unroll
            for (int u = 0; u < 4; ++u) {
                f[u] = flat;
                advance();
            }
            double t[4];
#pragma unroll
            for (int u = 0; u < 4; ++u) t[u] = generic_cell_term<Body, T, kRecompute>(p, j, f[u]);
#pragma unroll
            for (int u = 0; u < 4; ++u) sum += t[u];
        }
        for (; q < q1; q += kThreads) {
            sum += generic_cell_term<Body, T, kRecompute>(p, j, flat);
            advance();
        }
    }
    part[threadIdx.x] = sum;
    __syncthreads();
    for (int stride = kThreads / 2; stride > 0; stride >>= 1) {
        if (threadIdx.x < stride) part[threadIdx.x] += part[threadIdx.x + stride];
        __syncthreads();
    }
    if (threadIdx.x == 0) p.seg_ws[p.seg_offset[j] + e * S + seg] = part[0];
}

template <int N, int M, class T>
__global__ void __launch_bounds__(kThreads) pull_generic_seg_finish(const __grid_constant__ GenParams<N, M, T> p) {
    const int64_t g = blockIdx.x * int64_t(blockDim.x) + threadIdx.x;  // over segmented elements
    int j = 0;
    int64_t base = 0;  // first element index of argument j among segmented elements
    for (; j < N; ++j) {
        const int64_t n = p.segs[j] > 0 ? p.arg_vol[j] : 0;
        if (g < base + n) break;
        base += n;
    }
    if (j >= N) return;
    const int64_t e = g - base;
    const int S = p.segs[j];
    double sum = 0.0;
    for (int k = 0; k < S; ++k) sum += p.seg_ws[p.seg_offset[j] + e * S + k];
    const bool acc = (p.acc_mask >> j) & 1u;
    p.adj[j][e] = acc ? T(double(p.adj[j][e]) + sum) : T(sum);
}

// ------------------------------------------------- transcendental census
// Tally<T>: a real that counts its exp / log / sin / cos / tanh / sigmoid
// evaluations (the reference's counting wrappers, dual.hpp:55-60, 280-320)
// into this thread's s_tcount slot. Primal values are computed exactly as the
// production kernels compute them (same d_* calls, same operation order under
// --fmad=false), so every branch a body takes on Tally is the branch the
// production kernel took on that cell.
template <class T>
struct Tally {
    T v;
    BCAD_HD Tally() : v(T(0)) {}
    BCAD_HD Tally(T x) : v(x) {}  // NOLINT: bodies mix reals and literals
    template <class U, class = std::enable_if_t<std::is_arithmetic_v<U> && !std::is_same_v<U, T>>>
    BCAD_HD Tally(U x) : v(T(x)) {}  // NOLINT
};
__device__ __forceinline__ void tally_one() { s_tcount[threadIdx.x] += 1u; }
#define BCAD_TALLY_BIN(OP)                                                                                    \
    template <class T> BCAD_HD Tally<T> operator OP(const Tally<T>& a, const Tally<T>& b) { return Tally<T>(a.v OP b.v); } \
    template <class T> BCAD_HD Tally<T> operator OP(const Tally<T>& a, double b) { return Tally<T>(a.v OP T(b)); }       \
    template <class T> BCAD_HD Tally<T> operator OP(double a, const Tally<T>& b) { return Tally<T>(T(a) OP b.v); }
BCAD_TALLY_BIN(+)
BCAD_TALLY_BIN(-)
BCAD_TALLY_BIN(*)
BCAD_TALLY_BIN(/)
#undef BCAD_TALLY_BIN
#define BCAD_TALLY_CMP(OP)                                                                                    \
    template <class T> BCAD_HD bool operator OP(const Tally<T>& a, const Tally<T>& b) { return a.v OP b.v; }            \
    template <class T> BCAD_HD bool operator OP(const Tally<T>& a, double b) { return a.v OP T(b); }                    \
    template <class T> BCAD_HD bool operator OP(double a, const Tally<T>& b) { return T(a) OP b.v; }
BCAD_TALLY_CMP(<)
BCAD_TALLY_CMP(>)
BCAD_TALLY_CMP(<=)
BCAD_TALLY_CMP(>=)
BCAD_TALLY_CMP(==)
BCAD_TALLY_CMP(!=)
#undef BCAD_TALLY_CMP
template <class T> BCAD_HD Tally<T> operator-(const Tally<T>& a) { return Tally<T>(-a.v); }
template <class T> __device__ Tally<T> sigmoid(const Tally<T>& a) { tally_one(); return Tally<T>(raw_sigmoid(a.v)); }
template <class T> __device__ Tally<T> tanh(const Tally<T>& a) { tally_one(); return Tally<T>(d_tanh(a.v)); }
template <class T> __device__ Tally<T> exp(const Tally<T>& a) { tally_one(); return Tally<T>(d_exp(a.v)); }
template <class T> __device__ Tally<T> log(const Tally<T>& a) { tally_one(); return Tally<T>(d_log(a.v)); }
template <class T> __device__ Tally<T> sin(const Tally<T>& a) { tally_one(); return Tally<T>(d_sin(a.v)); }
template <class T> __device__ Tally<T> cos(const Tally<T>& a) { tally_one(); return Tally<T>(d_cos(a.v)); }
template <class T> __device__ Tally<T> sqrt(const Tally<T>& a) { return Tally<T>(d_sqrt(a.v)); }
template <class T> __device__ Tally<T> abs(const Tally<T>& a) { return Tally<T>(a.v < T(0) ? -a.v : a.v); }
template <class T> __device__ Tally<T> pow(const Tally<T>& a, double c) { return Tally<T>(d_pow(a.v, T(c))); }
template <class T> struct scalar_of<Tally<T>> { using type = T; };

// One census pass over the output cells of a launch that just ran: the body
// on Tally scalars per cell (kSelect: the branch-free select form, which the
// production kernels use when the boundary bits vary per cell), tallies
// flushed once per warp. Only launched while the census is armed.
template <class Body, class T, bool kSelect>
__global__ void __launch_bounds__(kThreads) census_kernel(const __grid_constant__ GenParams<Body::kIn, Body::kOut, T> p) {
    constexpr int N = Body::kIn, M = Body::kOut;
    count_begin();
    for (int64_t cell = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; cell < p.vol;
         cell += int64_t(gridDim.x) * blockDim.x) {
        int64_t off[N];
        decode_offsets<N, M, T>(p, cell, off);
        Tally<T> xi[N], yo[M];
#pragma unroll
        for (int j = 0; j < N; ++j) xi[j] = Tally<T>(p.in[j][off[j]]);
        if constexpr (kSelect) Body::template body_select<Tally<T>>(xi, yo);
        else Body::template body<Tally<T>>(xi, yo);
    }
    count_flush(p.tcount);
}

}  // namespace bcad_dev
