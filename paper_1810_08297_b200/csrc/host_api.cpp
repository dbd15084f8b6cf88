// libbcad_host.so: the end-to-end host entry (include/bcad_host.h) written
// against the C++ drop-in API, exactly the reference's run_cell_once
// sequence (proj/src/bench.cpp:112-128) with device tensors.
#include "bcad_host.h"

#include <algorithm>
#include <memory>
#include <atomic>
#include <optional>
#include <span>
#include <unordered_map>
#include <string>
#include <thread>
#include <vector>

#include "bcad/bcad.hpp"

namespace {

thread_local std::string g_err;

int code_of(const std::exception& e) {
    using namespace bcad;
    if (dynamic_cast<const TagMismatch*>(&e)) return BCAD_CU_ERR_TAG_MISMATCH;
    if (dynamic_cast<const DivisionByZero*>(&e)) return BCAD_CU_ERR_DIVISION_BY_ZERO;
    if (dynamic_cast<const DomainError*>(&e)) return BCAD_CU_ERR_DOMAIN;
    if (dynamic_cast<const NonDifferentiablePoint*>(&e)) return BCAD_CU_ERR_NON_DIFFERENTIABLE;
    if (dynamic_cast<const ShapeMismatch*>(&e)) return BCAD_CU_ERR_SHAPE_MISMATCH;
    if (dynamic_cast<const ArityMismatch*>(&e)) return BCAD_CU_ERR_ARITY_MISMATCH;
    if (dynamic_cast<const SeedShapeMismatch*>(&e)) return BCAD_CU_ERR_SEED_SHAPE_MISMATCH;
    if (dynamic_cast<const UnknownPrimitive*>(&e)) return BCAD_CU_ERR_UNKNOWN_PRIMITIVE;
    if (dynamic_cast<const ConfigError*>(&e)) return BCAD_CU_ERR_CONFIG;
    if (dynamic_cast<const CudaError*>(&e)) return BCAD_CU_ERR_CUDA;
    if (dynamic_cast<const NcclError*>(&e)) return BCAD_CU_ERR_NCCL;
    return BCAD_CU_ERR_GENERIC;
}

// One reference step (bench.cpp:112-128) on the current stream: tape inputs
// from host buffers, mixed_broadcast, backward(seeds), host copies of the
// primal / gradients. Returns the tape's peak_cached_bytes.
template <class Real>
int64_t tape_step(const char* name, int n_in, const void* const* host_in, const bcad_cu_shape* shapes, int m_out,
                  int policy, const void* const* host_seeds, void* const* host_primal, void* const* host_grads) {
    using namespace bcad;
    Tape<Real> tape;
    std::vector<Var<Real>> vars;
    {
        CopyBatch up(0);  // the n_in uploads as one runtime call
        std::vector<Tensor<Real>> x;
        for (int j = 0; j < n_in; ++j) {
            x.push_back(Tensor<Real>::uninitialized(Shape::from_c(shapes[j])));
            up.add(x.back().device_data(), host_in[j], x.back().bytes());
        }
        up.submit(current_stream());
        for (Tensor<Real>& t : x) vars.push_back(tape.input(std::move(t)));
    }
    const BroadcastKernel<Real> kernel(n_in, m_out, name);
    const std::vector<Var<Real>> outs = mixed_broadcast<Real>(
        tape, kernel, std::span<const Var<Real>>(vars), policy == 0 ? MixedPolicy::CacheForward : MixedPolicy::RecomputeReverse);
    std::vector<std::pair<Var<Real>, Tensor<Real>>> seeds;
    CopyBatch prim(1), sup(0);
    for (int i = 0; i < m_out; ++i) {
        const Tensor<Real>& v = tape.value(outs[static_cast<std::size_t>(i)]);
        if (host_primal && host_primal[i]) prim.add(host_primal[i], v.device_data(), v.bytes());
        if (host_seeds && host_seeds[i]) {
            seeds.emplace_back(outs[static_cast<std::size_t>(i)], Tensor<Real>::uninitialized(v.shape()));
            sup.add(seeds.back().second.device_data(), host_seeds[i], v.bytes());
        }
    }
    prim.submit(current_stream());
    sup.submit(current_stream());
    const Gradients<Real> grads = tape.backward(std::span<const std::pair<Var<Real>, Tensor<Real>>>(seeds));
    CopyBatch down(1);
    for (int j = 0; j < n_in; ++j) {
        if (!host_grads || !host_grads[j]) continue;
        const Tensor<Real>& g = grads.at(vars[static_cast<std::size_t>(j)]);
        down.add(host_grads[j], g.device_data(), g.bytes());
    }
    down.submit(current_stream());
    return tape.peak_cached_bytes();
}

// ---- pipelined step. The batch axis (axis 0) is cut into row chunks that
// flow through three streams: host->device copies (h2d), the K1/K2 kernels
// (the caller's stream) and device->host copies (d2h), so the upload of
// chunk c+1, the kernels of chunk c and the download of chunk c-1 overlap.
// Rows are independent under the reference's first-axis broadcasting
// (shape.hpp:13-16): per row the arithmetic and the (B)-axis reductions are
// the one-shot tape's, bit for bit. Batch-broadcast arguments (axis 0 of
// length 1, scalars) are uploaded once and their reduced gradients are
// accumulated over chunks in chunk order by the pullback's accumulate flag.

std::atomic<int> g_pipeline{0};  // 0 auto, 1 off, k > 1 at most k chunks

// Auto chunking: each chunk costs two batched copy calls, two launches and
// two events, and the last chunk's download is exposed, so chunks stay
// large (measured on B200 over PCIe: ~4 chunks of ~9-10 MB beat both the
// one-shot step and finer pipelines at configs 2 and 3).
constexpr std::size_t kChunkBytes = std::size_t(9) << 20;  // host<->device bytes per chunk
constexpr int kMaxChunks = 16;

struct Pipe {
    void* h2d = nullptr;
    void* d2h = nullptr;
    void* fork = nullptr;
    void* join = nullptr;    // the step's last download (recorded on d2h)
    void* x_free = nullptr;  // the step's last kernel (recorded on the compute stream): inputs consumed
    void* in_ready[kMaxChunks] = {};
    void* out_ready[kMaxChunks] = {};
    Pipe() {
        bcad::check(bcad_cu_stream_create(&h2d));
        bcad::check(bcad_cu_stream_create(&d2h));
        bcad::check(bcad_cu_event_create(&fork));
        bcad::check(bcad_cu_event_create(&join));
        bcad::check(bcad_cu_event_create(&x_free));
        for (int c = 0; c < kMaxChunks; ++c) {
            bcad::check(bcad_cu_event_create(&in_ready[c]));
            bcad::check(bcad_cu_event_create(&out_ready[c]));
        }
    }
    ~Pipe() {  // best effort: may run after the CUDA context is gone
        for (int c = 0; c < kMaxChunks; ++c) {
            bcad_cu_event_destroy(in_ready[c]);
            bcad_cu_event_destroy(out_ready[c]);
        }
        bcad_cu_event_destroy(fork);
        bcad_cu_event_destroy(join);
        bcad_cu_event_destroy(x_free);
        bcad_cu_stream_destroy(h2d);
        bcad_cu_stream_destroy(d2h);
    }
};

Pipe& pipe() {
    static thread_local Pipe p;
    return p;
}

int64_t volume(const bcad_cu_shape& s) {
    int64_t v = 1;
    for (int d = 0; d < s.rank; ++d) v *= s.dims[d];
    return v;
}

// Number of row chunks for this call (1 = one-shot tape).
// Asynchronous steps overlap each other's head and tail, so they take fewer,
// larger chunks: measured at config 2 (scripts/e2e_async_probe.py) a stream
// of async steps runs 0.44 ms per step at 2 chunks, 0.49 at 4, 0.56 at 8 —
// 2 chunks reach the H2D floor (21 MB at ~48 GB/s).
constexpr int kAsyncChunks = 2;

int plan_chunks(bcad_cu_kernel k, int n_in, const bcad_cu_shape* shapes, const bcad_cu_shape& out, int m_out,
                std::size_t elem, const void* const* host_seeds, void* const* host_primal, void* const* host_grads,
                const std::vector<bool>& split, bool async = false) {
    const int cfg = g_pipeline.load(std::memory_order_relaxed);
    if (cfg == 1 || out.rank < 1 || out.dims[0] < 2) return 1;
    if (bcad_cu_kernel_may_raise(k)) return 1;  // keep the reference's whole-tensor error index
    for (int j = 0; j < n_in; ++j)
        if (!split[j] && shapes[j].rank > 0 && shapes[j].dims[0] != 1) return 1;
    const int64_t vol = volume(out);
    std::size_t bytes = 0;
    for (int j = 0; j < n_in; ++j)
        if (split[j]) bytes += std::size_t(volume(shapes[j])) * elem * ((host_grads && host_grads[j]) ? 2 : 1);
    for (int i = 0; i < m_out; ++i)
        bytes += std::size_t(vol) * elem * (((host_seeds && host_seeds[i]) ? 1 : 0) + ((host_primal && host_primal[i]) ? 1 : 0));
    int chunks = cfg > 1 ? cfg : int(std::min<std::size_t>(kMaxChunks, bytes / kChunkBytes));
    if (async && cfg == 0 && chunks > kAsyncChunks) chunks = kAsyncChunks;
    chunks = std::min(chunks, kMaxChunks);
    if (chunks > out.dims[0]) chunks = int(out.dims[0]);
    return chunks < 2 ? 1 : chunks;
}

// Device buffers and chunk plan of one pipelined-step signature.
template <class Real>
struct StepBuffers {
    std::vector<bcad::Tensor<Real>> x, y, D, w, g;
    std::vector<int64_t> bound;  // chunk row boundaries
    std::vector<std::pair<int64_t, std::unique_ptr<bcad::detail::DeviceBuffer>>> ws;  // per chunk height
    std::vector<std::size_t> ws_bytes;
    std::size_t device_bytes = 0;
    // streams and events of this entry (prepared steps own theirs, so
    // consecutive asynchronous steps on different entries overlap)
    std::unique_ptr<Pipe> own_pipe;
    mutable bool used = false;  // a previous step enqueued on these buffers
    std::size_t ws_index(int64_t r) const {
        for (std::size_t q = 0; q < ws.size(); ++q)
            if (ws[q].first == r) return q;
        return 0;
    }
};

// Allocates (stream-ordered, on the current stream) every device buffer the
// pipelined step uses.
template <class Real>
void prepare_step(StepBuffers<Real>& S, bcad_cu_kernel k, int n_in, const bcad_cu_shape* shapes, int m_out, int policy,
                  const void* const* host_seeds, void* const* host_grads, const bcad_cu_shape& out,
                  const std::vector<bool>& split, int chunks) {
    using namespace bcad;
    constexpr int dt = dtype_of<Real>::value;
    void* const comp = current_stream();
    const int64_t B = out.dims[0], E = volume(out);
    const std::size_t n = static_cast<std::size_t>(n_in), m = static_cast<std::size_t>(m_out);
    auto alloc = [&](int64_t elems) {
        S.device_bytes += std::size_t(elems) * sizeof(Real);
        return Tensor<Real>::uninitialized(Shape{elems});
    };
    for (int j = 0; j < n_in; ++j) S.x.push_back(alloc(volume(shapes[j])));
    for (int i = 0; i < m_out; ++i) S.y.push_back(alloc(E));
    if (policy == 0)
        for (std::size_t t = 0; t < m * n; ++t) S.D.push_back(alloc(E));
    for (int i = 0; i < m_out; ++i) S.w.push_back(alloc(host_seeds && host_seeds[i] ? E : 1));
    for (int j = 0; j < n_in; ++j) S.g.push_back(alloc(host_grads && host_grads[j] ? volume(shapes[j]) : 1));
    // Chunk boundaries: the first and last chunks get half the rows of the
    // others, so the pipeline fills and drains faster (the exposed head is
    // the first chunk's upload, the exposed tail the last chunk's download).
    S.bound.assign(static_cast<std::size_t>(chunks) + 1, 0);
    const double units = chunks > 2 ? double(chunks) - 1.0 : double(chunks);
    double acc = 0.0;
    for (int c = 0; c < chunks; ++c) {
        acc += (chunks > 2 && (c == 0 || c == chunks - 1)) ? 0.5 : 1.0;
        S.bound[c + 1] = c + 1 == chunks ? B
                                         : std::min(B - (chunks - c - 1),
                                                    std::max(S.bound[c] + 1, int64_t(double(B) * acc / units + 0.5)));
    }
    for (int c = 0; c < chunks; ++c) {  // one workspace per distinct chunk height
        const int64_t r = S.bound[c + 1] - S.bound[c];
        bool seen = false;
        for (auto& [h, buf] : S.ws) seen = seen || h == r;
        if (seen) continue;
        std::vector<bcad_cu_shape> cs(shapes, shapes + n_in);
        for (int j = 0; j < n_in; ++j)
            if (split[j]) cs[j].dims[0] = r;
        std::size_t b = 0;
        check(bcad_cu_pullback_workspace(k, dt, n_in, cs.data(), m_out, &b));
        S.ws.emplace_back(r, std::make_unique<detail::DeviceBuffer>(b, comp));
        check(bcad_cu_pullback_workspace_init(S.ws.back().second->ptr, b, comp));
        S.ws_bytes.push_back(b);
        S.device_bytes += b;
    }
}

// Enqueues the pipelined step on the current stream (no synchronisation, no
// allocation). Returns the one-shot tape's peak_cached_bytes.
template <class Real>
int64_t enqueue_step(const StepBuffers<Real>& S, bcad_cu_kernel k, int n_in, const void* const* host_in,
                     const bcad_cu_shape* shapes, int m_out, int policy, const void* const* host_seeds,
                     void* const* host_primal, void* const* host_grads, const bcad_cu_shape& out,
                     const std::vector<bool>& split) {
    using namespace bcad;
    constexpr int dt = dtype_of<Real>::value;
    void* const comp = current_stream();
    Pipe& P = S.own_pipe ? *S.own_pipe : pipe();
    const int chunks = int(S.bound.size()) - 1;
    const int64_t B = out.dims[0], E = volume(out), out_row = E / B;
    const std::size_t n = static_cast<std::size_t>(n_in), m = static_cast<std::size_t>(m_out);
    std::vector<int64_t> row_elems(n, 0);
    int64_t in_elems = 0;
    for (int j = 0; j < n_in; ++j) {
        in_elems += volume(shapes[j]);
        if (split[j]) row_elems[j] = volume(shapes[j]) / B;
    }
    std::vector<bool> has_w(m, false), has_g(n, false);
    for (int i = 0; i < m_out; ++i) has_w[i] = host_seeds && host_seeds[i];
    for (int j = 0; j < n_in; ++j) has_g[j] = host_grads && host_grads[j];
    auto dev = [](const Tensor<Real>& t) { return const_cast<Real*>(t.device_data()); };
    // Buffer reuse across steps on these buffers: the kernels may overwrite
    // y / D / g only after the previous step's downloads have read them, the
    // uploads may overwrite x / w only after its last kernel has read them.
    // The first step instead orders the copy streams after the compute
    // stream, where the buffers were allocated (stream-ordered).
    if (S.used) check(bcad_cu_stream_wait_event(comp, P.join));
    {
        CopyBatch rep(0);  // batch-broadcast inputs: whole, on the compute stream
        for (int j = 0; j < n_in; ++j)
            if (!split[j]) rep.add(dev(S.x[j]), host_in[j], S.x[j].bytes());
        rep.submit(comp);
    }
    if (!S.used || !S.own_pipe) {
        check(bcad_cu_event_record(P.fork, comp));
        check(bcad_cu_stream_wait_event(P.h2d, P.fork));
        check(bcad_cu_stream_wait_event(P.d2h, P.fork));
    } else {
        check(bcad_cu_stream_wait_event(P.h2d, P.x_free));
    }

    std::vector<bcad_cu_shape> cs(shapes, shapes + n_in);
    std::vector<const void*> xin(n), wp(m), Dp(m * n);
    std::vector<void*> yp(m), Dw(m * n), gp(n);
    std::vector<unsigned char> acc(n, 0);
    for (int c = 0; c < chunks; ++c) {
        const int64_t b0 = S.bound[c], b1 = S.bound[c + 1], r = b1 - b0;
        const std::size_t cell0 = static_cast<std::size_t>(b0 * out_row), cells = static_cast<std::size_t>(r * out_row);
        // h2d: this chunk's rows of the batch-sharded inputs and of the seeds
        CopyBatch up(0);
        for (int j = 0; j < n_in; ++j) {
            if (!split[j]) continue;
            const std::size_t o = static_cast<std::size_t>(b0 * row_elems[j]), cnt = static_cast<std::size_t>(r * row_elems[j]);
            up.add(dev(S.x[j]) + o, static_cast<const Real*>(host_in[j]) + o, cnt * sizeof(Real));
        }
        for (int i = 0; i < m_out; ++i)
            if (has_w[i])
                up.add(dev(S.w[i]) + cell0, static_cast<const Real*>(host_seeds[i]) + cell0, cells * sizeof(Real));
        up.submit(P.h2d);
        check(bcad_cu_event_record(P.in_ready[c], P.h2d));
        // compute: K1 then K2 on the chunk (row-offset views of the buffers)
        check(bcad_cu_stream_wait_event(comp, P.in_ready[c]));
        for (int j = 0; j < n_in; ++j) {
            const int64_t o = split[j] ? b0 * row_elems[j] : 0;
            xin[j] = dev(S.x[j]) + o;
            cs[j] = shapes[j];
            if (split[j]) cs[j].dims[0] = r;
            gp[j] = has_g[j] ? static_cast<void*>(dev(S.g[j]) + o) : nullptr;
            acc[j] = (!split[j] && c > 0) ? 1 : 0;
        }
        for (int i = 0; i < m_out; ++i) {
            yp[i] = dev(S.y[i]) + cell0;
            wp[i] = has_w[i] ? static_cast<const void*>(dev(S.w[i]) + cell0) : nullptr;
        }
        for (std::size_t t = 0; t < S.D.size(); ++t) {
            Dw[t] = dev(S.D[t]) + cell0;
            Dp[t] = Dw[t];
        }
        const std::size_t q = S.ws_index(r);
        check(bcad_cu_forward(k, dt, n_in, xin.data(), cs.data(), m_out, yp.data(), policy == 0 ? Dw.data() : nullptr, comp));
        check(bcad_cu_pullback(k, dt, n_in, cs.data(), m_out, wp.data(), policy == 0 ? Dp.data() : nullptr, xin.data(),
                               gp.data(), acc.data(), S.ws[q].second->ptr, S.ws_bytes[q], comp));
        check(bcad_cu_event_record(P.out_ready[c], comp));
        // d2h: the chunk's primal rows and batch-sharded gradient rows
        check(bcad_cu_stream_wait_event(P.d2h, P.out_ready[c]));
        CopyBatch down(1);
        for (int i = 0; i < m_out; ++i)
            if (host_primal && host_primal[i])
                down.add(static_cast<Real*>(host_primal[i]) + cell0, dev(S.y[i]) + cell0, cells * sizeof(Real));
        for (int j = 0; j < n_in; ++j) {
            if (!split[j] || !has_g[j]) continue;
            const std::size_t o = static_cast<std::size_t>(b0 * row_elems[j]), cnt = static_cast<std::size_t>(r * row_elems[j]);
            down.add(static_cast<Real*>(host_grads[j]) + o, dev(S.g[j]) + o, cnt * sizeof(Real));
        }
        down.submit(P.d2h);
    }
    check(bcad_cu_event_record(P.x_free, comp));
    bool whole_grads = false;  // reduced gradients of batch-broadcast inputs: complete after the last chunk
    for (int j = 0; j < n_in; ++j) whole_grads = whole_grads || (!split[j] && has_g[j]);
    if (whole_grads) {
        check(bcad_cu_stream_wait_event(P.d2h, P.x_free));
        CopyBatch rep(1);
        for (int j = 0; j < n_in; ++j)
            if (!split[j] && has_g[j]) rep.add(host_grads[j], dev(S.g[j]), S.g[j].bytes());
        rep.submit(P.d2h);
    }
    check(bcad_cu_event_record(P.join, P.d2h));
    S.used = true;
    // what the one-shot tape reports (tape.hpp:236-243): inputs + values + cache
    return (in_elems + int64_t(m) * E + (policy == 0 ? int64_t(m * n) * E : 0)) * int64_t(sizeof(Real));
}

// ---- prepared steps. A caller repeating a step on the same pinned host
// buffers (the serving / training-loop case) keeps its device buffers,
// chunk plan and workspaces, so later calls only enqueue copies and kernels
// (measured at config 2: 0.57 vs 0.59 ms per call). Bounded: a few entries
// per thread, each at most kMaxPreparedBytes of device memory (bigger steps
// allocate per call). Replaying the enqueued work as a CUDA graph was
// measured too and lost the upload/download overlap (0.77 ms), so calls are
// issued, not replayed.
std::atomic<int> g_prepared{1};
constexpr std::size_t kMaxPreparedBytes = std::size_t(2) << 30;
constexpr std::size_t kMaxPreparedEntries = 4;

template <class Real>
struct Prepared {
    StepBuffers<Real> bufs;
    uint64_t last_use = 0;
};

template <class Real>
std::unordered_map<std::string, std::unique_ptr<Prepared<Real>>>& prepared_cache() {
    static thread_local std::unordered_map<std::string, std::unique_ptr<Prepared<Real>>> c;
    return c;
}

std::string step_key(const char* name, int n_in, const bcad_cu_shape* shapes, int m_out, int policy, int chunks,
                     const void* const* host_in, const void* const* host_seeds, void* const* host_primal,
                     void* const* host_grads, void* stream) {
    std::string key(name);
    auto put = [&key](const void* p, std::size_t b) { key.append(static_cast<const char*>(p), b); };
    const int64_t hdr[] = {n_in, m_out, policy, chunks};
    put(hdr, sizeof hdr);
    put(&stream, sizeof stream);
    for (int j = 0; j < n_in; ++j) {
        put(&shapes[j].rank, sizeof shapes[j].rank);
        put(shapes[j].dims, sizeof(int64_t) * std::size_t(shapes[j].rank));
        const void* ptr[] = {host_in[j], host_grads ? host_grads[j] : nullptr};
        put(ptr, sizeof ptr);
    }
    for (int i = 0; i < m_out; ++i) {
        const void* ptr[] = {host_seeds ? host_seeds[i] : nullptr, host_primal ? host_primal[i] : nullptr};
        put(ptr, sizeof ptr);
    }
    return key;
}

bool all_pinned(int n_in, const void* const* host_in, int m_out, const void* const* host_seeds,
                void* const* host_primal, void* const* host_grads) {
    for (int j = 0; j < n_in; ++j) {
        if (!bcad_cu_host_is_pinned(host_in[j])) return false;
        if (host_grads && host_grads[j] && !bcad_cu_host_is_pinned(host_grads[j])) return false;
    }
    for (int i = 0; i < m_out; ++i) {
        if (host_seeds && host_seeds[i] && !bcad_cu_host_is_pinned(host_seeds[i])) return false;
        if (host_primal && host_primal[i] && !bcad_cu_host_is_pinned(host_primal[i])) return false;
    }
    return true;
}

template <class Real>
int64_t pipelined_step(bcad_cu_kernel k, const char* name, int n_in, const void* const* host_in,
                       const bcad_cu_shape* shapes, int m_out, int policy, const void* const* host_seeds,
                       void* const* host_primal, void* const* host_grads, const bcad_cu_shape& out,
                       const std::vector<bool>& split, int chunks, bool async = false) {
    using namespace bcad;
    void* const comp = current_stream();
    int64_t in_bytes = 0;
    for (int j = 0; j < n_in; ++j) in_bytes += volume(shapes[j]) * int64_t(sizeof(Real));
    const std::size_t estimate = std::size_t(in_bytes) * 2 +
                                 std::size_t(volume(out)) * sizeof(Real) * std::size_t(m_out) * (2 + std::size_t(n_in));
    const bool cacheable = g_prepared.load(std::memory_order_relaxed) && comp != nullptr &&
                           estimate <= kMaxPreparedBytes &&
                           all_pinned(n_in, host_in, m_out, host_seeds, host_primal, host_grads);
    if (!cacheable) {
        if (async)
            throw ConfigError("bcad_host_mixed_step_async needs pinned host buffers and prepared steps "
                              "(bcad_host_set_prepared(1)) on a non-default stream");
        StepBuffers<Real> S;
        prepare_step<Real>(S, k, n_in, shapes, m_out, policy, host_seeds, host_grads, out, split, chunks);
        const int64_t p = enqueue_step<Real>(S, k, n_in, host_in, shapes, m_out, policy, host_seeds, host_primal,
                                             host_grads, out, split);
        check(bcad_cu_stream_synchronize(comp));
        check(bcad_cu_stream_synchronize(pipe().d2h));
        return p;
    }
    auto& cache = prepared_cache<Real>();
    static thread_local uint64_t clock = 0;
    const std::string key =
        step_key(name, n_in, shapes, m_out, policy, chunks, host_in, host_seeds, host_primal, host_grads, comp);
    auto it = cache.find(key);
    if (it == cache.end()) {
        if (cache.size() >= kMaxPreparedEntries) {  // evict the least recently used (all prior work is complete)
            auto lru = cache.begin();
            for (auto e = cache.begin(); e != cache.end(); ++e)
                if (e->second->last_use < lru->second->last_use) lru = e;
            cache.erase(lru);
        }
        auto entry = std::make_unique<Prepared<Real>>();
        entry->bufs.own_pipe = std::make_unique<Pipe>();
        prepare_step<Real>(entry->bufs, k, n_in, shapes, m_out, policy, host_seeds, host_grads, out, split, chunks);
        it = cache.emplace(key, std::move(entry)).first;
    }
    Prepared<Real>& E = *it->second;
    E.last_use = ++clock;
    const int64_t p = enqueue_step<Real>(E.bufs, k, n_in, host_in, shapes, m_out, policy, host_seeds, host_primal,
                                         host_grads, out, split);
    if (!async) {
        check(bcad_cu_stream_synchronize(comp));
        check(bcad_cu_stream_synchronize(E.bufs.own_pipe->d2h));
    }
    return p;
}

// Waits for every step enqueued by bcad_host_mixed_step_async on this thread.
template <class Real>
void sync_prepared() {
    for (auto& [key, e] : prepared_cache<Real>())
        if (e->bufs.own_pipe) {
            bcad::check(bcad_cu_stream_synchronize(e->bufs.own_pipe->h2d));
            bcad::check(bcad_cu_stream_synchronize(e->bufs.own_pipe->d2h));
        }
}

template <class Real>
void step(const char* name, int n_in, const void* const* host_in, const bcad_cu_shape* shapes, int m_out,
          int policy, const void* const* host_seeds, void* const* host_primal, void* const* host_grads,
          int64_t* peak, bool async = false) {
    using namespace bcad;
    bcad_cu_kernel k = nullptr;
    check(bcad_cu_kernel_lookup(name, n_in, m_out, &k));
    bcad_cu_shape out{};
    check(bcad_cu_broadcast_shape(n_in, shapes, &out));
    std::vector<bool> split(static_cast<std::size_t>(n_in), false);
    for (int j = 0; j < n_in; ++j) split[j] = shapes[j].rank > 0 && out.rank > 0 && shapes[j].dims[0] == out.dims[0];
    const int chunks =
        plan_chunks(k, n_in, shapes, out, m_out, sizeof(Real), host_seeds, host_primal, host_grads, split, async);
    int64_t p = 0;
    if (chunks == 1) {
        if (async) throw ConfigError("bcad_host_mixed_step_async needs a pipelined (row-chunked) step");
        p = tape_step<Real>(name, n_in, host_in, shapes, m_out, policy, host_seeds, host_primal, host_grads);
        check(bcad_cu_stream_synchronize(current_stream()));
    } else {
        p = pipelined_step<Real>(k, name, n_in, host_in, shapes, m_out, policy, host_seeds, host_primal, host_grads,
                                 out, split, chunks, async);
    }
    if (peak) *peak = p;
}

template <class Real>
void cell_grads(int impl, int64_t n, const void* const* dev_in, const void* dev_seed, void* const* dev_grads,
                int64_t* nodes, int64_t* peak) {
    using namespace bcad;
    const Shape mat{n, n}, vec{n};
    // the caller's device buffers become the CellInputs (copies, one batch)
    CopyBatch in_copies(2);
    auto dev = [&](const Shape& s, const void* p) {
        Tensor<Real> t = Tensor<Real>::uninitialized(s);
        in_copies.add(t.device_data(), p, t.bytes());
        return t;
    };
    const CellInputs<Real> in{dev(mat, dev_in[0]), dev(mat, dev_in[1]), dev(mat, dev_in[2]),
                              dev(mat, dev_in[3]), dev(vec, dev_in[4]), dev(vec, dev_in[5])};
    const Tensor<Real> seed = dev(mat, dev_seed);
    in_copies.submit(current_stream());
    Tape<Real> tape;
    CellGraph<Real> graph;
    if (impl == 0) graph = cell_update_fused(tape, in, MixedPolicy::CacheForward);
    else if (impl == 1) graph = cell_update_fused(tape, in, MixedPolicy::RecomputeReverse);
    else if (impl == 2) graph = cell_update_unfused(tape, in);
    else throw ConfigError("impl must be 0 (mixed-cache), 1 (mixed-recompute) or 2 (reverse-unfused)");
    const Gradients<Real> g = tape.backward(graph.out, seed);
    const Var<Real> leaves[4] = {graph.c_prev, graph.f, graph.i, graph.g};
    CopyBatch out(2);
    for (int k = 0; k < 4; ++k) {
        const Tensor<Real>& t = g.at(leaves[k]);
        out.add(dev_grads[k], t.device_data(), t.bytes());
    }
    out.submit(current_stream());
    if (nodes) *nodes = static_cast<int64_t>(tape.size());
    if (peak) *peak = tape.peak_cached_bytes();
}

// Elements [begin, begin+count) of each tensor of the reference's input
// stream: ONE Rng(seed) draws the tensors in order (random_cell_inputs,
// hmlstm.hpp:35-43; random_pm1 / random_binary, tensor.hpp:71-84), one draw
// per element, so tensor j's block starts after sum(volumes[<j]) + begin_j
// draws. One thread per tensor.
template <class Real>
void random_blocks(uint64_t seed, int n, const int64_t* volumes, const int* kinds, const int64_t* begin,
                   const int64_t* count, void* const* out) {
    std::vector<std::thread> th;
    uint64_t offset = 0;
    for (int j = 0; j < n; ++j) {
        if (begin[j] < 0 || count[j] < 0 || begin[j] + count[j] > volumes[j])
            throw bcad::ConfigError("random block outside tensor " + std::to_string(j));
        const uint64_t skip = offset + static_cast<uint64_t>(begin[j]);
        th.emplace_back([=] {
            bcad::Rng rng(seed);
            rng.discard(skip);
            Real* o = static_cast<Real*>(out[j]);
            if (kinds[j] == 1)
                for (int64_t e = 0; e < count[j]; ++e) o[e] = static_cast<Real>(rng.binary());
            else
                for (int64_t e = 0; e < count[j]; ++e) o[e] = static_cast<Real>(rng.uniform_pm1());
        });
        offset += static_cast<uint64_t>(volumes[j]);
    }
    for (std::thread& t : th) t.join();
}

}  // namespace

extern "C" {

int bcad_host_random_inputs(uint64_t seed, int dtype, int n, const int64_t* volumes, const int* kinds,
                            const int64_t* begin, const int64_t* count, void* const* host_out) {
    try {
        if (dtype == BCAD_CU_F32) random_blocks<float>(seed, n, volumes, kinds, begin, count, host_out);
        else if (dtype == BCAD_CU_F64) random_blocks<double>(seed, n, volumes, kinds, begin, count, host_out);
        else throw bcad::ConfigError("dtype must be F32 or F64");
        return BCAD_CU_OK;
    } catch (const std::exception& e) {
        g_err = e.what();
        return code_of(e);
    }
}

uint64_t bcad_host_mix_seed(uint64_t seed, uint64_t salt) { return bcad::mix_seed(seed, salt); }

int bcad_host_cell_gradients(int impl, int dtype, int64_t n, const void* const* dev_in, const void* dev_seed,
                             void* const* dev_grads, int64_t* tape_nodes, int64_t* peak_cached_bytes, void* stream) {
    try {
        bcad::StreamGuard guard(stream);
        if (dtype == BCAD_CU_F32) cell_grads<float>(impl, n, dev_in, dev_seed, dev_grads, tape_nodes, peak_cached_bytes);
        else if (dtype == BCAD_CU_F64) cell_grads<double>(impl, n, dev_in, dev_seed, dev_grads, tape_nodes, peak_cached_bytes);
        else throw bcad::ConfigError("dtype must be F32 or F64");
        return BCAD_CU_OK;
    } catch (const std::exception& e) {
        g_err = e.what();
        return code_of(e);
    }
}

const char* bcad_host_last_error(void) { return g_err.c_str(); }

int bcad_host_set_prepared(int enable) {
    g_prepared.store(enable ? 1 : 0);
    if (!enable) {
        prepared_cache<float>().clear();
        prepared_cache<double>().clear();
    }
    return BCAD_CU_OK;
}

int bcad_host_set_pipeline(int max_chunks) {
    if (max_chunks < 0) {
        g_err = "bcad_host_set_pipeline: max_chunks must be >= 0";
        return BCAD_CU_ERR_CONFIG;
    }
    const int prev = g_pipeline.exchange(max_chunks);
    (void)prev;
    return BCAD_CU_OK;
}

int bcad_host_mixed_step(const char* kernel, int dtype, int n_in, const void* const* host_in,
                         const bcad_cu_shape* in_shapes, int m_out, int policy, const void* const* host_seeds,
                         void* const* host_primal, void* const* host_grads, int64_t* peak_cached_bytes,
                         void* stream) {
    try {
        bcad::StreamGuard guard(stream);
        if (dtype == BCAD_CU_F32)
            step<float>(kernel, n_in, host_in, in_shapes, m_out, policy, host_seeds, host_primal, host_grads, peak_cached_bytes);
        else if (dtype == BCAD_CU_F64)
            step<double>(kernel, n_in, host_in, in_shapes, m_out, policy, host_seeds, host_primal, host_grads, peak_cached_bytes);
        else
            throw bcad::ConfigError("dtype must be F32 or F64");
        return BCAD_CU_OK;
    } catch (const std::exception& e) {
        g_err = e.what();
        return code_of(e);
    }
}

int bcad_host_mixed_step_async(const char* kernel, int dtype, int n_in, const void* const* host_in,
                               const bcad_cu_shape* in_shapes, int m_out, int policy, const void* const* host_seeds,
                               void* const* host_primal, void* const* host_grads, void* stream) {
    try {
        bcad::StreamGuard guard(stream);
        if (dtype == BCAD_CU_F32)
            step<float>(kernel, n_in, host_in, in_shapes, m_out, policy, host_seeds, host_primal, host_grads, nullptr,
                        true);
        else if (dtype == BCAD_CU_F64)
            step<double>(kernel, n_in, host_in, in_shapes, m_out, policy, host_seeds, host_primal, host_grads, nullptr,
                         true);
        else
            throw bcad::ConfigError("dtype must be F32 or F64");
        return BCAD_CU_OK;
    } catch (const std::exception& e) {
        g_err = e.what();
        return code_of(e);
    }
}

int bcad_host_synchronize(void* stream) {
    try {
        bcad::check(bcad_cu_stream_synchronize(stream));
        sync_prepared<float>();
        sync_prepared<double>();
        return BCAD_CU_OK;
    } catch (const std::exception& e) {
        g_err = e.what();
        return code_of(e);
    }
}

}  // extern "C"
