// Host launchers: pick the 2-D vectorised kernels (with a compile-time
// argument-class signature when one is registered for the body, else the
// runtime-class variant) or the generic rank-N fallback, fill the by-value
// parameter block and launch on the caller's stream with programmatic
// dependent launch enabled. Included once per registration TU.
#pragma once

#include <cstdint>
#include <mutex>
#include <string>
#include <unordered_map>
#include <utility>

#include "kernels.cuh"
#include "registry.hpp"

namespace bcad_cu_impl {

using bcad_dev::DynSig;
using bcad_dev::Sig;

inline bool aligned16(const void* p) { return (reinterpret_cast<uintptr_t>(p) & 15u) == 0; }

inline int cuda_status(cudaError_t e, std::string* err) {
    if (e == cudaSuccess) return BCAD_CU_OK;
    *err = std::string("CUDA error: ") + cudaGetErrorString(e);
    return BCAD_CU_ERR_CUDA;
}

inline int generic_grid(int64_t work) {
    const int64_t blocks = ceil_div(work, kThreads);
    const int64_t cap = int64_t(sm_count()) * 16;
    return int(blocks < 1 ? 1 : (blocks > cap ? cap : blocks));
}

// cudaLaunchKernelEx with cudaLaunchAttributeProgrammaticStreamSerialization:
// the kernel may be scheduled while the previous kernel on the stream drains
// and blocks in griddepcontrol.wait until it has completed.
template <class Params>
cudaError_t launch_pdl(void (*kern)(Params), dim3 grid, size_t smem, cudaStream_t stream, const Params& p) {
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = grid;
    cfg.blockDim = dim3(kThreads);
    cfg.dynamicSmemBytes = smem;
    cfg.stream = stream;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    attr[0].val.programmaticStreamSerializationAllowed = 1;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    return cudaLaunchKernelEx(&cfg, kern, p);
}

// Resident 256-thread CTAs per SM of a kernel (occupancy API, cached per
// kernel; kCtasPerSm if the query fails, e.g. without a device).
inline std::mutex& occupancy_mutex() {
    static std::mutex m;
    return m;
}
inline std::unordered_map<const void*, int>& occupancy_cache() {
    static std::unordered_map<const void*, int> c;
    return c;
}
template <class Params>
int ctas_per_sm(void (*kern)(Params)) {
    const void* key = reinterpret_cast<const void*>(kern);
    {
        std::lock_guard<std::mutex> lock(occupancy_mutex());
        auto it = occupancy_cache().find(key);
        if (it != occupancy_cache().end()) return it->second;
    }
    int n = 0;
    if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&n, kern, kThreads, 0) != cudaSuccess || n < 1) {
        (void)cudaGetLastError();
        return kCtasPerSm;
    }
    std::lock_guard<std::mutex> lock(occupancy_mutex());
    occupancy_cache()[key] = n;
    return n;
}

template <class S>
bool sig_matches(const Plan& plan) {
    if (S::kN != plan.n) return false;
    for (int j = 0; j < plan.n; ++j)
        if (S::cls(j) != plan.cls[j]) return false;
    return true;
}

template <class F>
int with_sig(const Plan&, F&& f) {
    return f(DynSig{});
}
template <class S0, class... Rest, class F>
int with_sig(const Plan& plan, F&& f) {
    if (sig_matches<S0>(plan)) return f(S0{});
    return with_sig<Rest...>(plan, f);
}

template <int N, int M, class T>
void fill_generic(bcad_dev::GenParams<N, M, T>& g, const Plan& plan) {
    g.out_rank = plan.out_rank;
    for (int k = 0; k < kMaxRank; ++k) g.out_dims[k] = k < plan.out_rank ? plan.out_dims[k] : 1;
    g.vol = plan.vol;
    for (int j = 0; j < N; ++j) {
        for (int k = 0; k < kMaxRank; ++k) g.strides[j][k] = plan.strides[j][k];
        g.arg_vol[j] = plan.arg_vol[j];
    }
}

// The transcendental census (kernels.cuh census_kernel): one launch after a
// body-evaluating launch, only while counting is armed (FwdArgs / PullArgs
// tcount non-null). kSelect mirrors the production kernel's choice of the
// branch-free select form (static signature whose predicates vary per cell).
template <class Body, class S>
constexpr bool census_select() {
    if constexpr (S::kStatic) return Body::kSelectForm && !bcad_dev::vec_eval_ok<Body, S>();
    else return false;
}
template <class Body, class T>
int launch_census(const Plan& plan, const void* const* in, unsigned long long* tcount, bool select, cudaStream_t s,
                  std::string* err) {
    constexpr int N = Body::kIn, M = Body::kOut;
    bcad_dev::GenParams<N, M, T> g{};
    fill_generic(g, plan);
    for (int j = 0; j < N; ++j) g.in[j] = static_cast<const T*>(in[j]);
    g.tcount = tcount;
    const int grid = generic_grid(plan.vol);
    bool launched = false;
    if constexpr (Body::kSelectForm)  // only bodies with a select form instantiate it
        if (select) {
            bcad_dev::census_kernel<Body, T, true><<<grid, kThreads, 0, s>>>(g);
            launched = true;
        }
    if (!launched) bcad_dev::census_kernel<Body, T, false><<<grid, kThreads, 0, s>>>(g);
    return cuda_status(cudaGetLastError(), err);
}

// ---------------------------------------------------------------- forward
// K1's cells per thread: one 128-bit vector, unless the body caps it
// (Body::kMaxVec) because its dual state per cell is wide enough that V
// cells would not fit in registers (tanh_product_<A> for large A: every
// partial of the product is structurally nonzero).
template <class Body, class T>
constexpr int fwd_vec_width() {
    constexpr int v = vec_width<T>();
    if constexpr (requires { Body::kMaxVec; }) return Body::kMaxVec < v ? Body::kMaxVec : v;
    else return v;
}

// Generic kernels' cells per thread along the output's last axis: one
// 128-bit vector for bodies whose per-cell dual state is small (N*M <= 18),
// when the last axis is a multiple of it and every argument is contiguous
// (stride 1) or broadcast (stride 0) along it.
template <class Body, class T>
constexpr int generic_vec_width() {
    return Body::kIn * Body::kOut <= 18 ? fwd_vec_width<Body, T>() : 1;
}
inline bool generic_vec_ok(const Plan& plan, int V) {
    const int last = plan.out_rank - 1;
    if (last < 0 || plan.out_dims[last] % V != 0) return false;
    for (int j = 0; j < plan.n; ++j)
        if (plan.strides[j][last] != 0 && plan.strides[j][last] != 1) return false;
    return true;
}

// K1's rows per thread on large problems (more than two waves of CTAs):
// short CTAs, unless the body asks for more (Body::kFwdRows). The
// primal-only K1p moves 5 tensors per cell instead of 1 + N + M*N and wants
// longer CTAs. Measured (scripts/lab k1rpt / k5, fraction of the copy peak):
// HM-LSTM bias 65536 x 4096 fp32 K1 2 rows 1.02, 4 rows 1.00, 55 rows 0.94;
// fp64 8192 x 2048 K1 2 rows 1.00, 8 rows 0.96; K1p 65536 x 4096 2 rows 0.88,
// 16 rows 1.00; tanh_product_4 4096^2 2 rows 0.83, 8 rows 0.87;
// tanh_product_16 2 rows 0.66, 16 rows 0.71.
constexpr int kFwdRows = 2, kFwdRowsPrimalOnly = 16;
template <class Body>
constexpr int fwd_rows() {
    if constexpr (requires { Body::kFwdRows; }) return Body::kFwdRows;
    else return kFwdRows;
}

// The tiled 2-D forward at VV cells per thread (the body's vector width, or
// 1 for widths / pointers that do not allow vectors).
template <class Body, class T, int VV, class... Sigs>
int launch_fwd2d(const FwdArgs& a, std::string* err) {
    constexpr int N = Body::kIn, M = Body::kOut;
    const Plan& plan = *a.plan;
    const bool real = a.partials == nullptr;
    bcad_dev::Fwd2DParams<N, M, T> p{};
    for (int j = 0; j < N; ++j) {
        p.in[j] = static_cast<const T*>(a.in[j]);
        p.cls[j] = plan.cls[j];
    }
    for (int i = 0; i < M; ++i) {
        p.primal[i] = a.primal ? static_cast<T*>(a.primal[i]) : nullptr;
        for (int j = 0; j < N; ++j) p.partials[i * N + j] = a.partials ? static_cast<T*>(a.partials[i * N + j]) : nullptr;
    }
    p.rows = plan.rows;
    p.cols = plan.cols;
    p.err = a.err;
    bool dense = true;  // every output pointer present: no per-store checks
    for (int i = 0; i < M; ++i) {
        dense = dense && p.primal[i];
        for (int j = 0; j < N && !real; ++j) dense = dense && p.partials[i * N + j];
    }
    return with_sig<Sigs...>(plan, [&](auto sig) {
        using S = decltype(sig);
        void (*kern)(bcad_dev::Fwd2DParams<N, M, T>);
        if constexpr (S::kStatic) {
            if (dense) kern = real ? &bcad_dev::fwd2d_kernel<Body, T, VV, true, S, true> : &bcad_dev::fwd2d_kernel<Body, T, VV, false, S, true>;
            else kern = real ? &bcad_dev::fwd2d_kernel<Body, T, VV, true, S, false> : &bcad_dev::fwd2d_kernel<Body, T, VV, false, S, false>;
        } else {
            kern = real ? &bcad_dev::fwd2d_kernel<Body, T, VV, true, S, false> : &bcad_dev::fwd2d_kernel<Body, T, VV, false, S, false>;
        }
        // no reductions in K1: wide row tiles, one wave of this kernel's
        // resident CTAs on small problems
        const Tiling t = a.tiling ? *a.tiling
                                  : choose_tiling(plan, VV, ClassMix{}, /*fine=*/true,
                                                  real ? kFwdRowsPrimalOnly : fwd_rows<Body>(), ctas_per_sm(kern));
        p.vcols = int(t.vcols);
        p.txv_shift = __builtin_ctz(unsigned(t.txv));
        p.ty = t.ty;
        p.rpt = t.rpt;
        p.tile_rows = t.tile_rows;
        const dim3 grid(unsigned(t.n_col_tiles), unsigned(t.n_row_tiles));
        if (const int rc = cuda_status(launch_pdl(kern, grid, 0, a.stream, p), err)) return rc;
        if (a.tcount) return launch_census<Body, T>(plan, a.in, a.tcount, census_select<Body, S>(), a.stream, err);
        return int(BCAD_CU_OK);
    });
}

template <class Body, class T, class... Sigs>
int launch_fwd_t(const FwdArgs& a, std::string* err) {
    constexpr int N = Body::kIn, M = Body::kOut, V = fwd_vec_width<Body, T>();
    const Plan& plan = *a.plan;
    const bool real = a.partials == nullptr;
    bool vec = plan.is2d && plan.cols % V == 0;
    for (int j = 0; j < N && vec; ++j)
        if ((plan.cls[j] == kFull || plan.cls[j] == kCol) && !aligned16(a.in[j])) vec = false;
    for (int i = 0; i < M && vec; ++i) {
        if (a.primal && a.primal[i] && !aligned16(a.primal[i])) vec = false;
        for (int j = 0; j < N && a.partials && vec; ++j)
            if (a.partials[i * N + j] && !aligned16(a.partials[i * N + j])) vec = false;
    }
    if (vec) return launch_fwd2d<Body, T, V, Sigs...>(a, err);
    // odd widths / unaligned views of a 2-D problem: the same tiled kernel, one cell per thread
    if constexpr (V > 1)
        if (plan.is2d) return launch_fwd2d<Body, T, 1>(a, err);
    bcad_dev::GenParams<N, M, T> g{};
    fill_generic(g, plan);
    for (int j = 0; j < N; ++j) g.in[j] = static_cast<const T*>(a.in[j]);
    for (int i = 0; i < M; ++i) {
        g.primal[i] = a.primal ? static_cast<T*>(a.primal[i]) : nullptr;
        for (int j = 0; j < N; ++j) g.partials[i * N + j] = a.partials ? static_cast<T*>(a.partials[i * N + j]) : nullptr;
    }
    g.err = a.err;
    if constexpr (generic_vec_width<Body, T>() > 1) {
        constexpr int GV = generic_vec_width<Body, T>();
        bool gvec = generic_vec_ok(plan, GV);
        for (int j = 0; j < N && gvec; ++j)
            if (plan.strides[j][plan.out_rank - 1] != 0 && !aligned16(a.in[j])) gvec = false;
        for (int i = 0; i < M && gvec; ++i) {
            if (a.primal && a.primal[i] && !aligned16(a.primal[i])) gvec = false;
            for (int j = 0; j < N && a.partials && gvec; ++j)
                if (a.partials[i * N + j] && !aligned16(a.partials[i * N + j])) gvec = false;
        }
        if (gvec) {
            const int grid = generic_grid(plan.vol / GV);
            if (real) bcad_dev::fwd_generic_vec_kernel<Body, T, GV, true><<<grid, kThreads, 0, a.stream>>>(g);
            else bcad_dev::fwd_generic_vec_kernel<Body, T, GV, false><<<grid, kThreads, 0, a.stream>>>(g);
            if (const int rc = cuda_status(cudaGetLastError(), err)) return rc;
            return a.tcount ? launch_census<Body, T>(plan, a.in, a.tcount, false, a.stream, err) : BCAD_CU_OK;
        }
    }
    const int grid = generic_grid(plan.vol);
    if (real) bcad_dev::fwd_generic_kernel<Body, T, true><<<grid, kThreads, 0, a.stream>>>(g);
    else bcad_dev::fwd_generic_kernel<Body, T, false><<<grid, kThreads, 0, a.stream>>>(g);
    if (const int rc = cuda_status(cudaGetLastError(), err)) return rc;
    return a.tcount ? launch_census<Body, T>(plan, a.in, a.tcount, false, a.stream, err) : BCAD_CU_OK;
}

// --------------------------------------------------------------- pullback
// Pullback L2 lookahead (RecomputeReverse kernels only, kernels.cuh): the
// streams of a thread's next row are prefetched into L2 while it evaluates
// the current one. Measured (scripts/lab k2pf, fraction of the copy peak,
// lookahead 0 -> 1): config 5 0.80 -> 0.92, fp64 config 4 0.82 -> 0.92,
// canonical 65536 x 4096 0.95 -> 1.00, bias 16384 x 1024 0.61 -> 0.66;
// neutral at config 3, off at two rows per thread (config 2: nothing to
// overlap). Two rows ahead is slower everywhere.
inline int pull_prefetch_rows(bool recompute, const Tiling& t) {
    if (t.prefetch >= 0) return t.prefetch;
    return recompute && t.rpt >= 3 ? 1 : 0;
}

// Register double buffer of the pullback (kPipe): on small, latency-bound
// grids, and only with at least two rows per thread to overlap. Measured
// (scripts/lab step / stepr, profiles/r02/lab_step_pipe.jsonl,
// lab_stepr_pipe.jsonl), config-sized steps with stream launches:
//   cached    config 3 (256 CTAs) 33.9 -> 29.6 us; config 2 (512 CTAs) 19.4 -> 20.1 us (worse: not used)
//   recompute config 2 (512 CTAs) 21.1 -> 19.4 us; config 3 (256 CTAs) 30.9 -> 27.6 us
// The recompute pullback already runs at three CTAs per SM (80 registers),
// so dropping to two costs it less than it costs the cached one at four.
inline bool pull_pipe(const Tiling& t, bool recompute) {
    if (t.pipe >= 0) return t.pipe > 0;
    return t.rpt >= 2 && t.n_ctas <= (recompute ? 4 : 2) * int64_t(sm_count());
}

// The tiled 2-D pullback at VV cells per thread (VV = the 128-bit width, or
// 1 for widths / pointers that do not allow vectors) with signature
// dispatch over Sigs (none: runtime classes only).
template <class Body, class T, int VV, class... Sigs>
int launch_pull2d(const PullArgs& a, std::string* err) {
    constexpr int N = Body::kIn, M = Body::kOut;
    const Plan& plan = *a.plan;
    const bool recompute = a.partials == nullptr;
    const Tiling t = a.tiling ? *a.tiling : choose_tiling(plan, VV, class_mix(plan));
    const PullLayout L = pull_layout(plan, t);  // offsets sized for every argument
    if (a.ws_bytes < L.total || (L.total > 0 && !a.workspace)) {
        *err = "pullback workspace too small: need " + std::to_string(L.total) + " bytes";
        return BCAD_CU_ERR_CONFIG;
    }
    bcad_dev::Pull2DParams<N, M, T> p{};
    int nr = 0, nc = 0, ns = 0;
    for (int j = 0; j < N; ++j) {
        p.in[j] = a.in ? static_cast<const T*>(a.in[j]) : nullptr;
        p.adj[j] = static_cast<T*>(a.in_adj[j]);
        p.cls[j] = plan.cls[j];
        p.slot[j] = -1;
        if (a.accumulate && a.accumulate[j]) p.acc_mask |= 1u << j;
        if (!p.adj[j]) continue;
        if (plan.cls[j] == kRow) { p.row_j[nr] = j; p.slot[j] = nr++; }
        if (plan.cls[j] == kCol) { p.col_j[nc] = j; p.slot[j] = nc++; }
        if (plan.cls[j] == kScalar) { p.scal_j[ns] = j; p.slot[j] = ns++; }
    }
    for (int i = 0; i < M; ++i) {
        p.w[i] = static_cast<const T*>(a.out_adj[i]);
        for (int j = 0; j < N; ++j) p.D[i * N + j] = recompute ? nullptr : static_cast<const T*>(a.partials[i * N + j]);
    }
    p.rows = plan.rows;
    p.cols = plan.cols;
    p.vcols = int(t.vcols);
    p.txv_shift = __builtin_ctz(unsigned(t.txv));
    p.ty = t.ty;
    p.rpt = t.rpt;
    p.prefetch = pull_prefetch_rows(recompute, t);
    p.tile_rows = t.tile_rows;
    p.n_col_tiles = int(t.n_col_tiles);
    p.n_row_tiles = int(t.n_row_tiles);
    p.n_row_args = nr;
    p.n_col_args = nc;
    p.n_scalar_args = ns;
    char* ws = static_cast<char*>(a.workspace);
    p.ws_row = reinterpret_cast<double*>(ws + L.ws_row);
    p.ws_col = reinterpret_cast<double*>(ws + L.ws_col);
    p.ws_scalar = reinterpret_cast<double*>(ws + L.ws_scalar);
    p.err = a.err;
    int64_t fin_blocks = bcad_dev::pull_finish_blocks(plan.rows, plan.cols, p.n_row_tiles, p.n_col_tiles, nr, nc, ns);
    // cross-CTA reductions combined inside K2 (completion tickets) unless the
    // tiling asks for the separate K2f launch
    if (fin_blocks > 0 && pull_combine_in_kernel(t, nr, nc, ns) && !a.peer) {
        p.tickets = reinterpret_cast<unsigned int*>(ws + L.ws_tickets);
        fin_blocks = 0;
    }
    // fused allreduce over a peer group: column sums always leave fp64
    // partials, and K2f-AR replaces K2f (+ the collective)
    int64_t ar_blocks = 0;
    if (a.peer) {
        if (nc == 0 || (ns > 0 && t.n_ctas > 1)) {
            *err = "fused peer allreduce: the problem needs (1,H)-class (column) reductions and no scalar ones";
            return BCAD_CU_ERR_CONFIG;
        }
        if (int64_t(nc) * plan.cols > a.peer->n) {
            *err = "fused peer allreduce: " + std::to_string(int64_t(nc) * plan.cols) +
                   " reduced elements exceed the peer group's " + std::to_string(a.peer->n);
            return BCAD_CU_ERR_CONFIG;
        }
        p.col_to_ws = 1;
        ar_blocks = (t.n_col_tiles > 1 && nr > 0 ? (int64_t(nr) * plan.rows + 31) / 32 : 0) +
                    (int64_t(nc) * plan.cols + 31) / 32;
        fin_blocks = 0;
    }
    const size_t smem = pull_smem_bytes(nc, nr, ns, t);
    const dim3 grid(unsigned(t.n_col_tiles), unsigned(t.n_row_tiles));
    bool dense = p.acc_mask == 0;  // every w and adjoint present, nothing accumulated
    for (int i = 0; i < M; ++i) dense = dense && p.w[i];
    for (int j = 0; j < N; ++j) dense = dense && p.adj[j];
    const bool pipe = pull_pipe(t, recompute);
    return with_sig<Sigs...>(plan, [&](auto sig) {
        using S = decltype(sig);
        void (*kern)(bcad_dev::Pull2DParams<N, M, T>);
        if constexpr (S::kStatic) {
            if (dense && pipe)
                kern = recompute ? &bcad_dev::pull2d_kernel<Body, T, VV, true, S, true, true>
                                 : &bcad_dev::pull2d_kernel<Body, T, VV, false, S, true, true>;
            else if (dense) kern = recompute ? &bcad_dev::pull2d_kernel<Body, T, VV, true, S, true> : &bcad_dev::pull2d_kernel<Body, T, VV, false, S, true>;
            else kern = recompute ? &bcad_dev::pull2d_kernel<Body, T, VV, true, S, false> : &bcad_dev::pull2d_kernel<Body, T, VV, false, S, false>;
        } else {
            kern = recompute ? &bcad_dev::pull2d_kernel<Body, T, VV, true, S, false> : &bcad_dev::pull2d_kernel<Body, T, VV, false, S, false>;
        }
        if (smem > 48 * 1024) {
            const cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem));
            if (e != cudaSuccess) return cuda_status(e, err);
        }
        int rc = cuda_status(launch_pdl(kern, grid, smem, a.stream, p), err);
        if (rc) return rc;
        if (recompute && a.tcount)  // K2r re-evaluated every cell's body
            if ((rc = launch_census<Body, T>(plan, a.in, a.tcount, census_select<Body, S>(), a.stream, err))) return rc;
        if (ar_blocks > 0) {
            cudaLaunchConfig_t cfg = {};
            cfg.gridDim = dim3(unsigned(ar_blocks));
            cfg.blockDim = dim3(kThreads);
            cfg.stream = a.stream;
            cudaLaunchAttribute attr[1];
            attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
            attr[0].val.programmaticStreamSerializationAllowed = 1;
            cfg.attrs = attr;
            cfg.numAttrs = 1;
            return cuda_status(cudaLaunchKernelEx(&cfg, &bcad_dev::pull_finish_ar_kernel<N, M, T>, p, *a.peer), err);
        }
        if (fin_blocks == 0 || t.skip_finish) return rc;
        return cuda_status(launch_pdl(&bcad_dev::pull_finish_kernel<N, M, T>, dim3(unsigned(fin_blocks)), 0,
                                      a.stream, p), err);
    });
}

template <class Body, class T, class... Sigs>
int launch_pull_t(const PullArgs& a, std::string* err) {
    constexpr int N = Body::kIn, M = Body::kOut, V = vec_width<T>();
    const Plan& plan = *a.plan;
    const bool recompute = a.partials == nullptr;
    bool vec = pull_vec_shape_ok<T>(plan);
    for (int i = 0; i < M && vec; ++i)
        if (a.out_adj[i] && !aligned16(a.out_adj[i])) vec = false;
    for (int j = 0; j < N && vec; ++j) {
        if (!a.in_adj[j]) continue;
        if (plan.cls[j] == kFull && !aligned16(a.in_adj[j])) vec = false;
        for (int i = 0; i < M && !recompute && vec; ++i)
            if (a.out_adj[i] && !aligned16(a.partials[i * N + j])) vec = false;
    }
    for (int j = 0; j < N && recompute && vec; ++j)
        if ((plan.cls[j] == kFull || plan.cls[j] == kCol) && !aligned16(a.in[j])) vec = false;
    if (vec) return launch_pull2d<Body, T, V, Sigs...>(a, err);
    if (a.peer && !pull_scalar2d_ok<T>(plan)) {
        *err = "fused peer allreduce needs a 2-D (rows x cols) problem";
        return BCAD_CU_ERR_CONFIG;
    }
    // odd widths / unaligned views of a 2-D problem: the same tiled kernel, one
    // cell per thread (when the caller's workspace fits that layout)
    if (pull_scalar2d_ok<T>(plan) &&
        a.ws_bytes >= pull_layout(plan, choose_tiling(plan, 1, class_mix(plan))).total)
        return launch_pull2d<Body, T, 1>(a, err);
    // generic rank-N pullback: a thread per element (coalesced when the
    // argument is full along the last axis; its reduction cut into segments
    // when that leaves too few threads), a warp per element for arguments
    // reduced over >= 32 cells including the last axis, segments over CTAs
    // when those are >= 4096 cells
    bcad_dev::GenParams<N, M, T> g{};
    fill_generic(g, plan);
    for (int j = 0; j < N; ++j) g.in[j] = a.in ? static_cast<const T*>(a.in[j]) : nullptr;
    for (int j = 0; j < N; ++j)
        if (a.accumulate && a.accumulate[j]) g.acc_mask |= 1u << j;
    for (int i = 0; i < M; ++i) {
        g.w[i] = static_cast<const T*>(a.out_adj[i]);
        for (int j = 0; j < N; ++j) g.D[i * N + j] = recompute ? nullptr : static_cast<const T*>(a.partials[i * N + j]);
    }
    g.err = a.err;
    bcad_dev::GenParams<N, M, T> gw = g, gs = g, gf = g;
    bool any_full = false;
    // arguments reduced over many cells per element: segmented (needs the
    // workspace bcad_cu_pullback_workspace sizes for the generic path)
    const size_t seg_bytes = generic_seg_ws(plan);
    const bool can_seg = seg_bytes > 0 && a.workspace && a.ws_bytes >= seg_bytes;
    int64_t off = 0, offw = 0, segoff = 0, seg_items = 0, segblk = 0;
    for (int j = 0; j < N; ++j) {
        const int S = can_seg && a.in_adj[j] ? generic_segments(plan, j) : 0;
        const bool col = S && generic_column_mode(plan, j);
        if (col) gs.seg_col_mask |= 1u << j;
        gs.seg_block[j] = segblk;
        segblk += col ? ceil_div(plan.arg_vol[j], kThreads) * S : plan.arg_vol[j] * S;
        const bool wide = a.in_adj[j] && S == 0 && reduced_along_last_axis(plan, j) &&
                          plan.vol / (plan.arg_vol[j] > 0 ? plan.arg_vol[j] : 1) >= 32;
        const bool full = a.in_adj[j] && plan.arg_vol[j] == plan.vol;
        any_full |= full;
        gf.adj[j] = full ? static_cast<T*>(a.in_adj[j]) : nullptr;
        g.adj[j] = wide || S || full ? nullptr : static_cast<T*>(a.in_adj[j]);
        gw.adj[j] = wide ? static_cast<T*>(a.in_adj[j]) : nullptr;
        gs.adj[j] = S ? static_cast<T*>(a.in_adj[j]) : nullptr;
        gs.segs[j] = S;
        gs.seg_offset[j] = segoff;
        segoff += plan.arg_vol[j] * S;
        if (S) seg_items += plan.arg_vol[j];
        g.adj_offset[j] = off;
        gw.adj_offset[j] = offw;
        if (g.adj[j]) off += plan.arg_vol[j];
        if (gw.adj[j]) offw += plan.arg_vol[j];
    }
    g.adj_offset[N] = off;
    gw.adj_offset[N] = offw;
    gs.seg_offset[N] = segoff;
    gs.seg_block[N] = segblk;
    gs.seg_ws = static_cast<double*>(a.workspace);
    if (segoff > 0) {
        if (recompute) bcad_dev::pull_generic_seg_kernel<Body, T, true><<<unsigned(segblk), kThreads, 0, a.stream>>>(gs);
        else bcad_dev::pull_generic_seg_kernel<Body, T, false><<<unsigned(segblk), kThreads, 0, a.stream>>>(gs);
        if (const int rc = cuda_status(cudaGetLastError(), err)) return rc;
        bcad_dev::pull_generic_seg_finish<N, M, T><<<unsigned(ceil_div(seg_items, kThreads)), kThreads, 0, a.stream>>>(gs);
        if (const int rc = cuda_status(cudaGetLastError(), err)) return rc;
    }
    if (any_full) {  // arguments of the output's shape: elementwise
        constexpr int GV = generic_vec_width<Body, T>();
        bool gvec = GV > 1 && generic_vec_ok(plan, GV);
        for (int i = 0; i < M && gvec; ++i) {
            if (gf.w[i] && !aligned16(gf.w[i])) gvec = false;
            for (int j = 0; j < N && gvec; ++j)
                if (gf.w[i] && gf.adj[j] && !recompute && !aligned16(gf.D[i * N + j])) gvec = false;
        }
        for (int j = 0; j < N && gvec; ++j) {
            if (gf.adj[j] && !aligned16(gf.adj[j])) gvec = false;
            if (recompute && plan.strides[j][plan.out_rank - 1] != 0 && !aligned16(gf.in[j])) gvec = false;
        }
        if (gvec) {
            const int grid = generic_grid(plan.vol / GV);
            if (recompute) bcad_dev::pull_generic_full_kernel<Body, T, GV, true><<<grid, kThreads, 0, a.stream>>>(gf);
            else bcad_dev::pull_generic_full_kernel<Body, T, GV, false><<<grid, kThreads, 0, a.stream>>>(gf);
        } else {
            const int grid = generic_grid(plan.vol);
            if (recompute) bcad_dev::pull_generic_full_kernel<Body, T, 1, true><<<grid, kThreads, 0, a.stream>>>(gf);
            else bcad_dev::pull_generic_full_kernel<Body, T, 1, false><<<grid, kThreads, 0, a.stream>>>(gf);
        }
        if (const int rc = cuda_status(cudaGetLastError(), err)) return rc;
    }
    if (off > 0) {
        const int grid = generic_grid(off);
        if (recompute) bcad_dev::pull_generic_kernel<Body, T, true, false><<<grid, kThreads, 0, a.stream>>>(g);
        else bcad_dev::pull_generic_kernel<Body, T, false, false><<<grid, kThreads, 0, a.stream>>>(g);
        if (const int rc = cuda_status(cudaGetLastError(), err)) return rc;
    }
    if (offw > 0) {
        const int grid = generic_grid(offw * 32);
        if (recompute) bcad_dev::pull_generic_kernel<Body, T, true, true><<<grid, kThreads, 0, a.stream>>>(gw);
        else bcad_dev::pull_generic_kernel<Body, T, false, true><<<grid, kThreads, 0, a.stream>>>(gw);
        if (const int rc = cuda_status(cudaGetLastError(), err)) return rc;
    }
    if (recompute && a.tcount) {
        // the generic RecomputeReverse kernels re-evaluate every cell once for
        // the full-shape arguments together and once per reduced argument
        int passes = any_full ? 1 : 0;
        for (int j = 0; j < N; ++j) passes += a.in_adj[j] && plan.arg_vol[j] != plan.vol;
        for (int k = 0; k < passes; ++k)
            if (const int rc = launch_census<Body, T>(plan, a.in, a.tcount, false, a.stream, err)) return rc;
    }
    return BCAD_CU_OK;
}

template <class Body, class... Sigs>
int launch_fwd_any(const FwdArgs& a, std::string* err) {
    return a.dtype == BCAD_CU_F32 ? launch_fwd_t<Body, float, Sigs...>(a, err)
                                  : launch_fwd_t<Body, double, Sigs...>(a, err);
}
template <class Body, class... Sigs>
int launch_pull_any(const PullArgs& a, std::string* err) {
    return a.dtype == BCAD_CU_F32 ? launch_pull_t<Body, float, Sigs...>(a, err)
                                  : launch_pull_t<Body, double, Sigs...>(a, err);
}

// Argument-class signatures of the HM-LSTM workloads:
// canonical (B,H)x4 + (B)x2; divergence (B,H)x6; bias (B,H)x4 + (1,H)x3 + (B)x2.
using SigHmlstmCanonical = Sig<kFull, kFull, kFull, kFull, kRow, kRow>;
using SigHmlstmDivergence = Sig<kFull, kFull, kFull, kFull, kFull, kFull>;
using SigHmlstmBias = Sig<kFull, kFull, kFull, kFull, kCol, kCol, kCol, kRow, kRow>;
// Every argument full-shape (an elementwise problem, e.g. the arity workload):
// compile-time classes drop the per-argument class branches and, with every
// output wanted, the per-store null checks.
template <int N, class Seq = std::make_integer_sequence<int, N>>
struct SigAllFullT;
template <int N, int... I>
struct SigAllFullT<N, std::integer_sequence<int, I...>> {
    using type = Sig<((void)I, int(kFull))...>;
};
template <int N>
using SigAllFull = typename SigAllFullT<N>::type;
// The arguments in PRED broadcast along the last axis ((B)-shaped, ROW), the
// others full-shape: the layout of a body branching on per-row flags (the
// HM-LSTM boundary bits), whose cells then evaluate as lane vectors.
template <int N, uint32_t PRED, class Seq = std::make_integer_sequence<int, N>>
struct SigPredRowT;
template <int N, uint32_t PRED, int... I>
struct SigPredRowT<N, PRED, std::integer_sequence<int, I...>> {
    using type = Sig<(((PRED >> I) & 1u) ? int(kRow) : int(kFull))...>;
};
template <int N, uint32_t PRED>
using SigPredRow = typename SigPredRowT<N, PRED>::type;

}  // namespace bcad_cu_impl

#define BCAD_ENTRY(Body, ...)                                                                          \
    bcad_cu_kernel_entry {                                                                             \
        Body::kName, Body::kIn, Body::kOut, Body::kMayRaise,                                           \
            &bcad_cu_impl::launch_fwd_any<Body __VA_OPT__(, ) __VA_ARGS__>,                             \
            &bcad_cu_impl::launch_pull_any<Body __VA_OPT__(, ) __VA_ARGS__>                             \
    }

// A registered body whose forward also gets signature S but whose pullback
// dispatches on runtime classes only (wide bodies: their static pullback
// instantiations dominate compile time for no benchmarked use).
#define BCAD_ENTRY_FWD_SIG(Body, S)                                                                    \
    bcad_cu_kernel_entry {                                                                             \
        Body::kName, Body::kIn, Body::kOut, Body::kMayRaise, &bcad_cu_impl::launch_fwd_any<Body, S>,    \
            &bcad_cu_impl::launch_pull_any<Body>                                                       \
    }
