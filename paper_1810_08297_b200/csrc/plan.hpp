// Host-side broadcast planning for the device kernels.
//
// The reference walks output cells with a per-argument stride table and an
// odometer (BroadcastPlan, proj/include/bcad/broadcast.hpp:19-88). On the
// GPU the same first-axis broadcast is first canonicalised: length-1 output
// axes are dropped and adjacent axes on which every argument has the same
// full/broadcast pattern are merged. What remains is almost always a 2-D
// (rows x cols) problem in which every argument is one of four stride
// classes — FULL (r*cols + c), ROW ((B) against (B,H): r), COL ((1,H): c) or
// SCALAR (0) — served by the vectorised tiled kernels. Anything with three
// or more irreducible axis groups uses the generic rank-N kernels.
#pragma once

#include <cstdint>
#include <cstring>
#include <string>

#include "bcad_cu.h"

namespace bcad_cu_impl {

constexpr int kMaxRank = BCAD_CU_MAX_RANK;
constexpr int kMaxIn = BCAD_CU_MAX_INPUTS;
constexpr int kMaxOut = BCAD_CU_MAX_OUTPUTS;
constexpr int kThreads = 256;

enum ArgClass : int { kFull = 0, kRow = 1, kCol = 2, kScalar = 3 };

struct Plan {
    int n = 0;
    // Output shape (reference semantics) and its volume.
    int out_rank = 0;
    int64_t out_dims[kMaxRank] = {};
    int64_t vol = 1;
    // Generic path: element strides of each argument over the output axes
    // (0 where the argument is broadcast), and each argument's volume.
    int64_t strides[kMaxIn][kMaxRank] = {};
    int64_t arg_vol[kMaxIn] = {};
    // 2-D canonical form (valid when is2d).
    bool is2d = false;
    int64_t rows = 1, cols = 1;
    int cls[kMaxIn] = {};
};

inline int64_t dim_of(const bcad_cu_shape& s, int k) { return k < s.rank ? s.dims[k] : 1; }

// Returns BCAD_CU_OK or BCAD_CU_ERR_SHAPE_MISMATCH with a reference-style message.
inline int make_plan(int n, const bcad_cu_shape* shapes, Plan* p, std::string* err) {
    *p = Plan{};
    p->n = n;
    for (int j = 0; j < n; ++j) {
        if (shapes[j].rank < 0 || shapes[j].rank > kMaxRank) {
            *err = "shape rank " + std::to_string(shapes[j].rank) + " outside [0, 8]";
            return BCAD_CU_ERR_SHAPE_MISMATCH;
        }
        int64_t v = 1;
        for (int k = 0; k < shapes[j].rank; ++k) {
            if (shapes[j].dims[k] < 1) {
                *err = "shape dimensions must be >= 1";
                return BCAD_CU_ERR_SHAPE_MISMATCH;
            }
            v *= shapes[j].dims[k];
        }
        p->arg_vol[j] = v;
        if (shapes[j].rank > p->out_rank) p->out_rank = shapes[j].rank;
    }
    // broadcast_shape (shape.hpp:70-90)
    for (int k = 0; k < p->out_rank; ++k) {
        int64_t len = 1;
        for (int j = 0; j < n; ++j) {
            const int64_t d = dim_of(shapes[j], k);
            if (d == 1) continue;
            if (len == 1) {
                len = d;
            } else if (d != len) {
                *err = "broadcast shape mismatch at dim " + std::to_string(k) + ": lengths " +
                       std::to_string(len) + " vs " + std::to_string(d);
                return BCAD_CU_ERR_SHAPE_MISMATCH;
            }
        }
        p->out_dims[k] = len;
        p->vol *= len;
    }
    // make_broadcast_plan strides (broadcast.hpp:25-41)
    for (int j = 0; j < n; ++j) {
        int64_t running = 1;
        for (int k = shapes[j].rank - 1; k >= 0; --k) {
            p->strides[j][k] = shapes[j].dims[k] == 1 ? 0 : running;
            running *= shapes[j].dims[k];
        }
    }
    // Canonicalise: drop length-1 output axes, merge equal-pattern neighbours.
    int64_t glen[kMaxRank];
    uint32_t gpat[kMaxRank];  // bit j set = argument j is full on the group
    int g = 0;
    for (int k = 0; k < p->out_rank; ++k) {
        if (p->out_dims[k] == 1) continue;
        uint32_t pat = 0;
        for (int j = 0; j < n; ++j)
            if (dim_of(shapes[j], k) != 1) pat |= 1u << j;
        if (g > 0 && gpat[g - 1] == pat) {
            glen[g - 1] *= p->out_dims[k];
        } else {
            glen[g] = p->out_dims[k];
            gpat[g] = pat;
            ++g;
        }
    }
    bool elementwise = true;  // every argument FULL or SCALAR
    for (int j = 0; j < n && elementwise; ++j) {
        const bool full = p->arg_vol[j] == p->vol, scalar = p->arg_vol[j] == 1;
        if (!full && !scalar) elementwise = false;
    }
    if (elementwise) {
        // Pure elementwise: any (rows, cols) factorisation of vol is valid.
        p->is2d = true;
        int64_t cols = 1;
        for (int64_t c = 4096; c >= 1; c >>= 1)
            if (p->vol % c == 0) { cols = c; break; }
        p->cols = cols;
        p->rows = p->vol / cols;
        for (int j = 0; j < n; ++j) p->cls[j] = (p->arg_vol[j] == p->vol && p->vol > 1) ? kFull : kScalar;
        if (p->vol == 1)
            for (int j = 0; j < n; ++j) p->cls[j] = kScalar;
        return BCAD_CU_OK;
    }
    if (g == 2) {
        p->is2d = true;
        p->rows = glen[0];
        p->cols = glen[1];
        for (int j = 0; j < n; ++j) {
            const bool fr = gpat[0] >> j & 1u, fc = gpat[1] >> j & 1u;
            p->cls[j] = fr ? (fc ? kFull : kRow) : (fc ? kCol : kScalar);
        }
    }
    return BCAD_CU_OK;
}

// Tile geometry of the 2-D kernels: 256 threads as (txv vector-columns) x
// (ty thread-rows); each thread walks `rpt` rows of its tile.
struct Tiling {
    int V = 1;         // elements per vector access
    int64_t vcols = 0; // cols / V
    int txv = 32, ty = 8, rpt = 1;
    int64_t tile_rows = 8, n_row_tiles = 1, n_col_tiles = 1, n_ctas = 1;
};

constexpr int kSmCount = 148;

inline int64_t ceil_div(int64_t a, int64_t b) { return (a + b - 1) / b; }

inline Tiling choose_tiling(const Plan& p, int V, bool has_col_reduction) {
    Tiling t;
    t.V = V;
    t.vcols = p.cols / V;
    int txv = 1;
    while (txv < 32 && txv < t.vcols) txv <<= 1;
    t.txv = txv;
    t.ty = kThreads / txv;
    t.n_col_tiles = ceil_div(t.vcols, txv);
    const int64_t tiles1 = ceil_div(p.rows, t.ty);  // row tiles at rpt = 1
    // Aim for ~8 resident 256-thread CTAs on each of the 148 SMs, times a few
    // waves, before growing the per-thread row count; column reductions
    // favour fewer row tiles (each adds one fp64 partial row to combine).
    const int64_t target = int64_t(kSmCount) * 8 * (has_col_reduction ? 2 : 4);
    int64_t rpt = (tiles1 * t.n_col_tiles) / target;
    if (rpt < 1) rpt = 1;
    if (rpt > 64) rpt = 64;
    t.rpt = int(rpt);
    t.tile_rows = int64_t(t.ty) * t.rpt;
    t.n_row_tiles = ceil_div(p.rows, t.tile_rows);
    t.n_ctas = t.n_row_tiles * t.n_col_tiles;
    return t;
}

// Workspace layout of the 2-D pullback (all offsets in bytes, 256-aligned).
struct PullLayout {
    int n_row_args = 0, n_col_args = 0, n_scalar_args = 0;
    size_t ws_row = 0, ws_col = 0, ws_scalar = 0, counters = 0, total = 0;
    size_t smem = 0;
};

inline size_t align256(size_t x) { return (x + 255) & ~size_t(255); }

inline PullLayout pull_layout(const Plan& p, const Tiling& t) {
    PullLayout L;
    for (int j = 0; j < p.n; ++j) {
        if (p.cls[j] == kRow) ++L.n_row_args;
        if (p.cls[j] == kCol) ++L.n_col_args;
        if (p.cls[j] == kScalar) ++L.n_scalar_args;
    }
    size_t off = 0;
    L.ws_row = off;
    if (t.n_col_tiles > 1) off += align256(size_t(L.n_row_args) * t.n_col_tiles * p.rows * 8);
    L.ws_col = off;
    if (t.n_row_tiles > 1) off += align256(size_t(L.n_col_args) * t.n_row_tiles * p.cols * 8);
    L.ws_scalar = off;
    if (t.n_ctas > 1) off += align256(size_t(L.n_scalar_args) * t.n_ctas * 8);
    L.counters = off;
    off += align256(size_t(t.n_row_tiles + t.n_col_tiles + 1) * 4);
    L.total = off;
    L.smem = size_t(L.n_col_args) * kThreads * t.V * 8 + size_t(L.n_scalar_args) * kThreads * 8;
    return L;
}

constexpr size_t kMaxPullSmem = 160 * 1024;

template <class T>
constexpr int vec_width() { return 16 / int(sizeof(T)); }

template <class T>
bool pull_vec_shape_ok(const Plan& plan) {
    constexpr int V = vec_width<T>();
    if (!plan.is2d || plan.cols % V != 0) return false;
    const Tiling t = choose_tiling(plan, V, true);
    return pull_layout(plan, t).smem <= kMaxPullSmem;
}

template <class T>
size_t pull_ws_t(const Plan& plan) {
    constexpr int V = vec_width<T>();
    if (!pull_vec_shape_ok<T>(plan)) return 256;
    bool has_col = false;
    for (int j = 0; j < plan.n; ++j) has_col |= plan.cls[j] == kCol;
    return pull_layout(plan, choose_tiling(plan, V, has_col)).total;
}


}  // namespace bcad_cu_impl
