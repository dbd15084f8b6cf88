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

#include <algorithm>
#include <atomic>
#include <cstdint>
#include <cstring>
#include <string>

#include <cuda_runtime.h>

#include "bcad_cu.h"

namespace bcad_cu_impl {

constexpr int kMaxRank = BCAD_CU_MAX_RANK;
constexpr int kMaxIn = BCAD_CU_MAX_INPUTS;
constexpr int kMaxOut = BCAD_CU_MAX_OUTPUTS;
constexpr int kThreads = 256;
// Device transcendental-evaluation counter slots (one atomic per warp into
// slot blockIdx % kCountSlots; the host sums them, abi.cu)
constexpr int kCountSlots = 1024;

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
// (ty thread-rows); each thread walks `rpt` rows of its tile. The grid is
// (n_col_tiles, n_row_tiles).
struct Tiling {
    int V = 1;          // elements per vector access
    int64_t vcols = 0;  // cols / V
    int txv = 32, ty = 8, rpt = 1;
    int64_t tile_rows = 8;
    int64_t n_row_tiles = 1, n_col_tiles = 1, n_ctas = 1;
    int prefetch = -1;  // pullback: rows ahead prefetched into L2 (-1 = the launcher's default)
    int pipe = -1;      // pullback: next row loaded into registers (kPipe; -1 = the launcher's default)
    bool skip_finish = false;  // lab timing only: omit K2f (reduced adjoints left incomplete)
    int combine = -1;   // cross-CTA reductions: -1 / 1 in K2 (tickets), 0 the separate K2f launch
};

// SM count of the current device (cached per ordinal; 148 on B200, and the
// fallback when no device is visible, so host-only workspace queries still
// answer). Workspace sizes follow the tiling, so a workspace must be queried
// with the device it will run on current.
constexpr int kDefaultSmCount = 148;
inline int sm_count() {
    static std::atomic<int> cache[64] = {};
    int dev = 0;
    if (cudaGetDevice(&dev) != cudaSuccess || dev < 0 || dev >= 64) {
        (void)cudaGetLastError();
        return kDefaultSmCount;
    }
    int n = cache[dev].load(std::memory_order_relaxed);
    if (n > 0) return n;
    if (cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, dev) != cudaSuccess || n < 1) {
        (void)cudaGetLastError();
        n = kDefaultSmCount;
    }
    cache[dev].store(n, std::memory_order_relaxed);
    return n;
}
constexpr int kCtasPerSm = 4;  // 256-thread CTAs at <= 64 registers per thread
// RecomputeReverse pullback (duals re-derived in registers): three CTAs per
// SM (<= 80 registers; the registered HM-LSTM signatures fit without spills).
// Same cells per thread and tiling as the cached pullback, so both policies
// reduce in the same order and agree bit for bit (mixed.hpp:103-130).
constexpr int kRecomputeCtasPerSm = 3;
constexpr int64_t kMaxGridY = 65535;

inline int64_t ceil_div(int64_t a, int64_t b) { return (a + b - 1) / b; }

struct ClassMix {
    bool row = false, col = false, scalar = false;
};

inline ClassMix class_mix(const Plan& p) {
    ClassMix m;
    for (int j = 0; j < p.n; ++j) {
        m.row |= p.cls[j] == kRow;
        m.col |= p.cls[j] == kCol;
        m.scalar |= p.cls[j] == kScalar && p.vol > 1;
    }
    return m;
}

// Shape of the tile by reduction mix:
//  * column reductions ((1,H) args) use one warp per row segment (txv = 32,
//    128 fp32 columns) and tall tiles, balancing the per-column fp64 partials
//    (cols x row tiles) against the per-row ones (rows x column tiles);
//  * otherwise a CTA spans up to 256 vector-columns of one row, so (B)-arg
//    reductions finish inside the CTA (shuffles + one shared-memory pass).
// Rows per thread: one wave of CTAs for small problems (latency-bound); short
// CTAs for large ones (K1 `fine_rows`, the pullback about eight waves and at
// most 16 rows), never more than 65535 row tiles.
// Small problems (at most two waves at one row per thread) run as one wave:
// config-2 K1 at two rows per thread 12.3 us against 14.3 us at one
// (interleaved A/B, scripts/lab k1ab; config 3 unchanged).
//
// K1 (fine) passes the kernel's own resident CTAs per SM (fwd_ctas_per_sm,
// from the occupancy API) so a small problem really is ONE wave, and keeps
// rows at most 128 vector-columns wide there. Measured at config 3 (bias K1,
// 74 registers, 3 CTAs per SM; scripts/lab k1small, means): 256 x 2 rows
// (512 CTAs, 1.15 waves) 15.9 us, 256 x 3 (342 CTAs) 15.1 us, 128 x 3 14.5 us;
// config 2 (4 CTAs per SM): 256 x 2 12.6 us, 128 x 2 12.5 us.
inline Tiling choose_tiling(const Plan& p, int V, const ClassMix& mix, bool fine = false, int fine_rows = 2,
                            int fwd_ctas_per_sm = kCtasPerSm) {
    Tiling t;
    t.V = V;
    t.vcols = p.cols / V;
    const int sms = sm_count();
    const int64_t slots = int64_t(sms) * (fine ? fwd_ctas_per_sm : kCtasPerSm);
    // K1 runs small problems (up to three rows per thread) as one wave
    const bool fine_small = fine && ceil_div(p.rows * std::max<int64_t>(t.vcols, 1), 256) <= 3 * slots;
    int cap = mix.col ? 32 : fine_small ? 128 : 256;
    int txv = 1;
    while (txv < cap && txv < t.vcols) txv <<= 1;
    // Column reductions ((1,H) arguments): at least 4 rows per thread, which
    // amortises each CTA's shared-memory setup and combine; small problems
    // also take 16-lane column tiles (64 fp32 columns) and about two CTAs per
    // SM, balancing the fp64 tile partials per column against those per row.
    // Measured (lab, bias variant) against the former 32 lanes x 1..6 rows:
    // B x H = 1024 x 1024 -18%, 4096 x 1024 -14%, 16384 x 1024 -4%; larger
    // problems keep 32 lanes (half the per-row partials, within 2%).
    const bool col_small = mix.col && !fine && txv == 32 && t.vcols >= 256 &&
                           ceil_div(p.rows, kThreads / 32) * ceil_div(t.vcols, 32) <= 2 * slots;
    if (col_small) txv = 16;
    t.txv = txv;
    t.ty = kThreads / txv;
    t.n_col_tiles = ceil_div(t.vcols, txv);
    const int64_t tiles1 = ceil_div(p.rows, t.ty);  // row tiles at rpt = 1
    const int64_t work = tiles1 * t.n_col_tiles;     // CTAs at rpt = 1
    // Large problems: short CTAs, many waves. K1 (fine, no reductions) takes
    // `fine_rows` rows per thread (launch.cuh fwd_rows); the pullback about
    // eight waves, at most 16 rows per thread. Measured at config 5 (lab k5,
    // bias 65536 x 4096 fp32): K1 55 -> 2 rows 0.94 -> 1.02 of the copy peak,
    // K2 55 -> 16 rows 0.94 -> 0.97.
    int64_t rpt = (fine ? fine_small : work <= 2 * slots) ? ceil_div(work, slots)
                                                           : (fine ? fine_rows : work / (8 * slots));
    if (col_small) rpt = ceil_div(work, 2 * sms);
    else if (mix.col && !fine && rpt < 4) rpt = 4;
    if (rpt < 1) rpt = 1;
    if (!fine && rpt > 16) rpt = 16;
    // keep the per-tile row partials in shared memory small
    if (mix.row)
        while (rpt > 1 && rpt * t.ty * (txv > 32 ? txv / 32 : 1) > 4096) rpt >>= 1;
    while (ceil_div(p.rows, int64_t(t.ty) * rpt) > kMaxGridY) rpt <<= 1;
    t.rpt = int(rpt);
    t.tile_rows = int64_t(t.ty) * t.rpt;
    t.n_row_tiles = ceil_div(p.rows, t.tile_rows);
    t.n_ctas = t.n_row_tiles * t.n_col_tiles;
    return t;
}

// Workspace (global: fp64 tile partials of reductions that span CTAs, then
// the completion tickets of their in-kernel combination) and dynamic shared
// memory of the 2-D pullback. Offsets are sized for every argument of a
// class, so a workspace queried once serves any subset of wanted adjoints.
// Every partial is written before it is read; the tickets must be zero before
// the first pullback (bcad_cu_pullback_workspace_init zero-fills the
// workspace) and every pullback leaves them zero again.
struct PullLayout {
    int n_row_args = 0, n_col_args = 0, n_scalar_args = 0;
    size_t ws_row = 0, ws_col = 0, ws_scalar = 0, ws_tickets = 0, n_tickets = 0, total = 0;
    size_t smem = 0;
};

inline size_t align256(size_t x) { return (x + 255) & ~size_t(255); }

inline size_t pull_smem_bytes(int n_col, int n_row, int n_scal, const Tiling& t) {
    const int wpr = t.txv > 32 ? t.txv / 32 : 1;
    return 8 * (size_t(n_col) * kThreads * t.V + size_t(n_row) * t.rpt * t.ty * wpr + size_t(n_scal) * kThreads);
}

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
    // (one tile row too: the fused peer allreduce reads fp64 column partials)
    if (L.n_col_args > 0) off += align256(size_t(L.n_col_args) * t.n_row_tiles * p.cols * 8);
    L.ws_scalar = off;
    if (t.n_ctas > 1) off += align256(size_t(L.n_scalar_args) * t.n_ctas * 8);
    L.ws_tickets = off;
    if (off > 0) {  // some reduction spans CTAs
        L.n_tickets = size_t(t.n_col_tiles + t.n_row_tiles + 1);
        off += align256(L.n_tickets * 4);
    }
    L.total = off;
    L.smem = pull_smem_bytes(L.n_col_args, L.n_row_args, L.n_scalar_args, t);
    return L;
}

constexpr size_t kMaxPullSmem = 160 * 1024;

// Peer-memory group of the fused pullback allreduce (abi.cu
// bcad_cu_peer_group_*, kernels.cuh pull_finish_ar_kernel): every rank's
// buffer holds, per parity of the step counter, [world][n] fp64 slots (rank
// k's local column sums land in slot k of every rank), then [world] arrival
// flags, the local step counter and the local CTA arrival counter.
constexpr int kMaxPeers = 8;
struct PeerParams {
    double* slots[kMaxPeers];                // rank k's slot region [2][world][n]
    unsigned long long* flags[kMaxPeers];    // rank k's flags [world]
    unsigned long long* epoch;               // this rank's step counter
    unsigned int* arrive;                    // this rank's CTA arrival counter
    int rank, world;
    int64_t n;                               // elements per slot (max_elems of the group)
};

template <class T>
constexpr int vec_width() { return 16 / int(sizeof(T)); }

template <class T>
bool pull_vec_shape_ok(const Plan& plan) {
    constexpr int V = vec_width<T>();
    if (!plan.is2d || plan.cols % V != 0) return false;
    return pull_layout(plan, choose_tiling(plan, V, class_mix(plan))).smem <= kMaxPullSmem;
}

// The tiled pullback at one cell per thread (odd widths, unaligned views).
template <class T>
bool pull_scalar2d_ok(const Plan& plan) {
    return plan.is2d && pull_layout(plan, choose_tiling(plan, 1, class_mix(plan))).smem <= kMaxPullSmem;
}

// Generic (rank-N) pullback: an argument reduced over at least kSegMinCells
// output cells per element is summed in segments of about kSegCells cells,
// one CTA each, into fp64 partials the finisher adds in segment order.
constexpr int64_t kSegMinCells = 4096, kSegCells = 4096;
constexpr int kMaxSegs = 256;
// True when argument j is broadcast along the output's last (fastest) axis:
// its reduced cells then include consecutive addresses, so lanes striding
// the reduction read coalesced; otherwise neighbouring ELEMENTS are
// neighbouring addresses and a thread per element reads coalesced.
inline bool reduced_along_last_axis(const Plan& plan, int j) {
    const int last = plan.out_rank - 1;
    return last >= 0 && plan.out_dims[last] > 1 && plan.strides[j][last] == 0;
}
// Arguments full along the last axis but reduced over kColMinCells or more
// cells per element (e.g. (B,1,H) under a (B,T,H) output): a thread per
// element, as above, but the reduction is also cut into segments over the
// grid's y dimension until about kColThreads threads are in flight (a thread
// walking all its cells alone leaves the SMs latency-bound when the argument
// is small), at least kColSegCells cells per segment.
constexpr int64_t kColMinCells = 64, kColSegCells = 16, kColThreads = int64_t(1) << 18;
inline bool generic_column_mode(const Plan& plan, int j) { return !reduced_along_last_axis(plan, j); }
inline int generic_segments(const Plan& plan, int j) {
    const int64_t av = plan.arg_vol[j] > 0 ? plan.arg_vol[j] : 1;
    const int64_t cnt = plan.vol / av;
    if (generic_column_mode(plan, j)) {
        if (cnt < kColMinCells) return 0;
        const int64_t s = std::min<int64_t>({kMaxSegs, cnt / kColSegCells, ceil_div(kColThreads, av)});
        return s > 1 ? int(s) : 0;
    }
    if (cnt < kSegMinCells) return 0;
    return int(std::min<int64_t>(kMaxSegs, ceil_div(cnt, kSegCells)));
}
inline size_t generic_seg_ws(const Plan& plan) {
    size_t b = 0;
    for (int j = 0; j < plan.n; ++j) b += size_t(plan.arg_vol[j]) * size_t(generic_segments(plan, j)) * 8;
    return b;
}

// Workspace of the tiled variant the width selects: vectors when the width
// allows them, else one cell per thread. (A vector-width problem handed
// unaligned views at launch uses the one-cell variant only if this
// workspace also fits its layout, else the generic kernel.)
template <class T>
size_t pull_ws_t(const Plan& plan) {
    constexpr int V = vec_width<T>();
    size_t ws = 256;
    if (pull_vec_shape_ok<T>(plan)) ws = std::max(ws, pull_layout(plan, choose_tiling(plan, V, class_mix(plan))).total);
    else if (pull_scalar2d_ok<T>(plan)) ws = std::max(ws, pull_layout(plan, choose_tiling(plan, 1, class_mix(plan))).total);
    else ws = std::max(ws, align256(generic_seg_ws(plan)));  // generic: segmented reductions
    return ws;
}

// Where the cross-CTA reductions are combined: by default in the finisher
// launch K2f (programmatically dependent: its CTAs are scheduled while K2
// drains); with Tiling::combine = 1 inside K2 by the last-arriving CTA of
// each strip / row tile (completion tickets). Measured at config 3
// (scripts/lab step3, profiles/r02/lab_step3_combine.jsonl): step 29.7 us
// with K2f, 31.7 us with tickets (every CTA pays a fence and two ticket
// atomics at its end, and the last CTA's combine sits on the tail), 26.6 us
// with no combination at all — so K2f stays the default and tickets an option.
inline bool pull_combine_in_kernel(const Tiling& t, int nr, int nc, int ns) {
    (void)nr;
    (void)nc;
    (void)ns;
    return t.combine > 0;
}

// Kernel launches of one pullback on the tiled path with aligned pointers:
// K2, plus the finisher K2f when a reduction spans CTAs and is not combined
// inside K2 (mirrors launch_pull2d). 0 when the problem takes the generic path.
template <class T>
int pull_launches_t(const Plan& plan) {
    int V = vec_width<T>();
    if (!pull_vec_shape_ok<T>(plan)) {
        if (!pull_scalar2d_ok<T>(plan)) {
            // generic rank-N: elementwise (full-shape arguments), segmented
            // reductions (+ finisher), thread- and warp-per-element kernels,
            // each launched when some input uses it
            bool full = false, seg = false, thread = false, warp = false;
            for (int j = 0; j < plan.n; ++j) {
                const int64_t cnt = plan.vol / (plan.arg_vol[j] > 0 ? plan.arg_vol[j] : 1);
                if (plan.arg_vol[j] == plan.vol) full = true;
                else if (generic_segments(plan, j)) seg = true;
                else if (reduced_along_last_axis(plan, j) && cnt >= 32) warp = true;
                else thread = true;
            }
            return full + 2 * seg + thread + warp;
        }
        V = 1;
    }
    const Tiling t = choose_tiling(plan, V, class_mix(plan));
    int nr = 0, nc = 0, ns = 0;
    for (int j = 0; j < plan.n; ++j) {
        nr += plan.cls[j] == kRow;
        nc += plan.cls[j] == kCol;
        ns += plan.cls[j] == kScalar;
    }
    const bool fin = (t.n_col_tiles > 1 && nr > 0) || (t.n_row_tiles > 1 && nc > 0) || (t.n_ctas > 1 && ns > 0);
    return fin && !pull_combine_in_kernel(t, nr, nc, ns) ? 2 : 1;
}

}  // namespace bcad_cu_impl
