// Drop-in C++ API on the GPU: mixed-node and tape claims of the reference's
// suites (proj/tests/test_mixed.cpp, test_tape.cpp, test_forward.cpp,
// test_broadcast.cpp) against the device-backed implementation.
#include <cmath>
#include <vector>

#include "bcad/bcad.hpp"
#include "mini_test.hpp"

using namespace bcad;

namespace {

const BroadcastKernel<double>& mul_kernel() {
    static const BroadcastKernel<double> k(2, 1, "mul", [](auto in, auto out) { out[0] = in[0] * in[1]; });
    return k;
}

template <class Real>
bool identical(const Tensor<Real>& a, const Tensor<Real>& b) {
    return a.shape() == b.shape() && a.to_host() == b.to_host();
}

bool all_close(const std::vector<double>& a, const std::vector<double>& b, double rtol, double atol) {
    if (a.size() != b.size()) return false;
    for (std::size_t e = 0; e < a.size(); ++e)
        if (!mini::close(a[e], b[e], rtol, atol)) return false;
    return true;
}

// Central-difference gradient of sum_i <w_i, kernel_i(x)> on the device.
std::vector<std::vector<double>> fd_weighted(const BroadcastKernel<double>& k, std::vector<Tensor<double>> x,
                                             const std::vector<Tensor<double>>& w) {
    auto h_of = [&](const std::vector<Tensor<double>>& xs) {
        std::vector<const Tensor<double>*> p;
        for (const auto& t : xs) p.push_back(&t);
        const auto outs = broadcast_apply<double>(k, std::span<const Tensor<double>* const>(p));
        double acc = 0;
        for (std::size_t i = 0; i < outs.size(); ++i) {
            const auto o = outs[i].to_host(), wi = w[i].to_host();
            for (std::size_t e = 0; e < o.size(); ++e) acc += wi[e] * o[e];
        }
        return acc;
    };
    std::vector<std::vector<double>> grads;
    for (std::size_t j = 0; j < x.size(); ++j) {
        const Shape s = x[j].shape();
        auto base = x[j].to_host();
        std::vector<double> g(base.size());
        for (std::size_t e = 0; e < base.size(); ++e) {
            const double h = std::cbrt(2.220446049250313e-16) * std::max(1.0, std::fabs(base[e]));
            auto p = base;
            p[e] = base[e] + h;
            x[j] = Tensor<double>::from(s, p);
            const double up = h_of(x);
            p[e] = base[e] - h;
            x[j] = Tensor<double>::from(s, p);
            const double down = h_of(x);
            g[e] = (up - down) / (2 * h);
        }
        x[j] = Tensor<double>::from(s, base);
        grads.push_back(g);
    }
    return grads;
}

}  // namespace

TEST_CASE("table-style pipeline: sum(b.(x, y)) with b = mul and a scalar x") {
    Rng rng(3);
    for (MixedPolicy policy : {MixedPolicy::CacheForward, MixedPolicy::RecomputeReverse}) {
        Tape<double> tape;
        const Tensor<double> y = random_pm1<double>(Shape{7}, rng);
        const Var<double> vx = tape.input(Tensor<double>::scalar(1.3));
        const Var<double> vy = tape.input(y);
        const Var<double> vf = mixed_broadcast(tape, mul_kernel(), {vx, vy}, policy)[0];
        const Var<double> vh = tape.prim(PrimKind::SumOverDims, {vf});
        const auto grads = tape.backward(vh, Tensor<double>(tape.value(vh).shape(), 1.0));
        double sum_y = 0;
        for (double v : y.to_host()) sum_y += v;
        CHECK(mini::close(grads.at(vx)[0], sum_y, 1e-14));
        for (double v : grads.at(vy).to_host()) CHECK(v == 1.3);
    }
}

TEST_CASE("identity mixed node passes the adjoint through unchanged") {
    Rng rng(5);
    Tape<double> tape;
    const Var<double> vx = tape.input(random_pm1<double>(Shape{3, 2}, rng));
    const Var<double> vy = mixed_broadcast(tape, identity_kernel<double>(), {vx}, MixedPolicy::CacheForward)[0];
    const Tensor<double> seed = random_pm1<double>(Shape{3, 2}, rng);
    const auto grads = tape.backward(vy, seed);
    CHECK(identical(grads.at(vx), seed));
}

TEST_CASE("one tape node regardless of kernel complexity or tensor size") {
    for (std::int64_t n : {std::int64_t{1}, std::int64_t{64}, std::int64_t{512}}) {
        Rng rng(7);
        Tape<double> tape;
        const CellInputs<double> in = random_cell_inputs<double>(n, rng);
        std::vector<Var<double>> v = {tape.input(in.c_prev), tape.input(in.f), tape.input(in.i),
                                      tape.input(in.g),      tape.input(in.z1), tape.input(in.z2)};
        const std::size_t before = tape.size();
        const auto outs = mixed_broadcast<double>(tape, cell_update_kernel<double>(), std::span<const Var<double>>(v),
                                                  MixedPolicy::CacheForward);
        CHECK(tape.size() == before + 1);
        CHECK(outs.size() == 1);
        CHECK(tape.value(outs[0]).shape() == (Shape{n, n}));
    }
}

TEST_CASE("cached policy retains exactly the M*N diagonals more than recompute") {
    Rng rng(17);
    const CellInputs<double> in = random_cell_inputs<double>(8, rng);
    auto run = [&](MixedPolicy p) {
        Tape<double> tape;
        (void)cell_update_fused(tape, in, p);
        return tape.peak_cached_bytes();
    };
    const std::int64_t cached = run(MixedPolicy::CacheForward), recomputed = run(MixedPolicy::RecomputeReverse);
    CHECK(cached > recomputed);
    CHECK(cached - recomputed == 6 * 64 * static_cast<std::int64_t>(sizeof(double)));
}

TEST_CASE("multi-output mixed node accumulates over all seeded outputs (FD)") {
    const BroadcastKernel<double> two(2, 2, "two");
    Rng rng(19);
    const Tensor<double> a = random_pm1<double>(Shape{3}, rng), b = random_pm1<double>(Shape{3}, rng);
    const Tensor<double> w0 = random_pm1<double>(Shape{3}, rng), w1 = random_pm1<double>(Shape{3}, rng);
    Tape<double> tape;
    const Var<double> va = tape.input(a), vb = tape.input(b);
    const auto outs = mixed_broadcast(tape, two, {va, vb}, MixedPolicy::CacheForward);
    REQUIRE(outs.size() == 2);
    std::vector<std::pair<Var<double>, Tensor<double>>> seeds;
    seeds.emplace_back(outs[0], w0);
    seeds.emplace_back(outs[1], w1);
    const auto grads = tape.backward(std::span<const std::pair<Var<double>, Tensor<double>>>(seeds));
    const auto fd = fd_weighted(two, {a, b}, {w0, w1});
    CHECK(all_close(grads.at(va).to_host(), fd[0], 1e-5, 1e-8));
    CHECK(all_close(grads.at(vb).to_host(), fd[1], 1e-5, 1e-8));
}

TEST_CASE("broadcast (2,1) argument through a mixed node matches FD") {
    Rng rng(23);
    const Tensor<double> x = random_pm1<double>(Shape{2, 3}, rng), y = random_pm1<double>(Shape{2, 1}, rng);
    const BroadcastKernel<double> gate(2, 1, "gate");
    Tape<double> tape;
    const Var<double> vx = tape.input(x), vy = tape.input(y);
    const Var<double> vk = mixed_broadcast(tape, gate, {vx, vy}, MixedPolicy::RecomputeReverse)[0];
    const Var<double> vh = tape.prim(PrimKind::SumOverDims, {vk});
    const auto grads = tape.backward(vh, Tensor<double>(tape.value(vh).shape(), 1.0));
    const auto fd = fd_weighted(gate, {x, y}, {Tensor<double>(Shape{2, 3}, 1.0)});
    CHECK(all_close(grads.at(vx).to_host(), fd[0], 1e-5, 1e-8));
    CHECK(all_close(grads.at(vy).to_host(), fd[1], 1e-5, 1e-8));
    CHECK(grads.at(vy).shape() == (Shape{2, 1}));
}

TEST_CASE("one graph can mix policies per node") {
    Rng rng(31);
    const Tensor<double> x = random_pm1<double>(Shape{4}, rng), y = random_pm1<double>(Shape{4}, rng);
    const BroadcastKernel<double> square_gate(2, 1, "square_gate");
    auto run = [&](MixedPolicy first, MixedPolicy second) {
        Tape<double> tape;
        const Var<double> vx = tape.input(x), vy = tape.input(y);
        const Var<double> v1 = mixed_broadcast(tape, square_gate, {vx, vy}, first)[0];
        const Var<double> v2 = mixed_broadcast(tape, mul_kernel(), {v1, vy}, second)[0];
        const Var<double> vh = tape.prim(PrimKind::SumOverDims, {v2});
        const auto grads = tape.backward(vh, Tensor<double>(tape.value(vh).shape(), 1.0));
        return std::make_pair(grads.at(vx).to_host(), grads.at(vy).to_host());
    };
    const auto mixed = run(MixedPolicy::CacheForward, MixedPolicy::RecomputeReverse);
    const auto uniform = run(MixedPolicy::CacheForward, MixedPolicy::CacheForward);
    CHECK(mixed.first == uniform.first);
    CHECK(mixed.second == uniform.second);
    // h = sum sigmoid(x) y^2: dh/dx = s(1-s) y^2, dh/dy = 2 s y
    const auto xh = x.to_host(), yh = y.to_host();
    for (std::size_t e = 0; e < xh.size(); ++e) {
        const double s = xh[e] >= 0 ? 1 / (1 + std::exp(-xh[e])) : std::exp(xh[e]) / (1 + std::exp(xh[e]));
        CHECK(mini::close(mixed.first[e], s * (1 - s) * yh[e] * yh[e], 1e-12, 1e-14));
        CHECK(mini::close(mixed.second[e], 2 * s * yh[e], 1e-12, 1e-14));
    }
}

TEST_CASE("mixed nodes of different shapes in one tape reduce a shared (1,H) argument; repeatable") {
    // Two pullbacks with different reduction layouts (cross-CTA completion
    // counters at different workspace offsets) on the same tape, swept twice.
    Rng rng(43);
    const int64_t H = 256;
    const Tensor<double> x = random_pm1<double>(Shape{64, H}, rng), y = random_pm1<double>(Shape{200, H}, rng);
    const Tensor<double> b = random_pm1<double>(Shape{1, H}, rng);
    Tape<double> tape;
    const Var<double> vx = tape.input(x), vy = tape.input(y), vb = tape.input(b);
    const Var<double> p1 = mixed_broadcast(tape, mul_kernel(), {vx, vb}, MixedPolicy::CacheForward)[0];
    const Var<double> p2 = mixed_broadcast(tape, mul_kernel(), {vy, vb}, MixedPolicy::CacheForward)[0];
    const Var<double> s1 = tape.prim(PrimKind::SumOverDims, {p1});
    const Var<double> s2 = tape.prim(PrimKind::SumOverDims, {p2});
    const Var<double> h = tape.prim(PrimKind::Add, {s1, s2});
    const auto xh = x.to_host(), yh = y.to_host();
    std::vector<double> want(static_cast<std::size_t>(H), 0.0);
    for (int64_t r = 0; r < 64; ++r)
        for (int64_t c = 0; c < H; ++c) want[static_cast<std::size_t>(c)] += xh[static_cast<std::size_t>(r * H + c)];
    for (int64_t r = 0; r < 200; ++r)
        for (int64_t c = 0; c < H; ++c) want[static_cast<std::size_t>(c)] += yh[static_cast<std::size_t>(r * H + c)];
    std::vector<double> first;
    for (int sweep = 0; sweep < 3; ++sweep) {
        const auto g = tape.backward(h, Tensor<double>(tape.value(h).shape(), 1.0)).at(vb).to_host();
        CHECK(all_close(g, want, 1e-12, 1e-12));
        if (sweep == 0) first = g;
        else CHECK(g == first);
    }
}

TEST_CASE("repeated input accumulates both contributions (x * x)") {
    Rng rng(41);
    const Tensor<double> x = random_pm1<double>(Shape{5, 3}, rng);
    for (MixedPolicy p : {MixedPolicy::CacheForward, MixedPolicy::RecomputeReverse}) {
        Tape<double> tape;
        const Var<double> vx = tape.input(x);
        const Var<double> sq = mixed_broadcast(tape, mul_kernel(), {vx, vx}, p)[0];
        const auto g = tape.backward(sq, Tensor<double>(Shape{5, 3}, 1.0)).at(vx).to_host();
        const auto xh = x.to_host();
        for (std::size_t e = 0; e < xh.size(); ++e) CHECK(g[e] == xh[e] + xh[e]);
    }
}

TEST_CASE("diagonal jacobian of the elementwise product is (y, x); primals exact") {
    Rng rng(3);
    const Tensor<double> x = random_pm1<double>(Shape{4}, rng), y = random_pm1<double>(Shape{4}, rng);
    const auto fwd = broadcast_diag_jacobian(mul_kernel(), true, x, y);
    CHECK(identical(fwd.jacobian.entry(0, 0), y));
    CHECK(identical(fwd.jacobian.entry(0, 1), x));
    const auto xh = x.to_host(), yh = y.to_host(), p = fwd.primals[0].to_host();
    for (std::size_t e = 0; e < 4; ++e) CHECK(p[e] == xh[e] * yh[e]);
}

TEST_CASE("branchy kernel differentiates along the taken branch") {
    const BroadcastKernel<double> reflect(1, 1, "reflect");
    const Tensor<double> x = Tensor<double>::from(Shape{5}, {-0.8, 0.1, 0.49, 0.51, 2.0});
    const auto fwd = broadcast_diag_jacobian(reflect, false, x);
    CHECK((fwd.jacobian.entry(0, 0).to_host() == std::vector<double>{-1.0, -1.0, -1.0, 1.0, 1.0}));
}

TEST_CASE("scatter_add reduces or expands") {
    Rng rng(47);
    const Tensor<double> contrib = random_pm1<double>(Shape{3, 4}, rng);
    Tensor<double> row(Shape{3, 1});
    scatter_add(row, contrib);
    const auto c = contrib.to_host(), r = row.to_host();
    for (std::size_t i = 0; i < 3; ++i) {
        double want = 0;
        for (std::size_t j = 0; j < 4; ++j) want += c[i * 4 + j];
        CHECK(mini::close(r[i], want, 1e-15));
    }
    Tensor<double> full(Shape{3, 4}, 1.0);
    const Tensor<double> rv = random_pm1<double>(Shape{3, 1}, rng);
    scatter_add(full, rv);
    const auto f = full.to_host(), rvh = rv.to_host();
    for (std::size_t i = 0; i < 3; ++i)
        for (std::size_t j = 0; j < 4; ++j) CHECK(f[i * 4 + j] == 1.0 + rvh[i]);
}

TEST_CASE("mul backward reduces a scalar argument; accumulation is additive") {
    Rng rng(53);
    Tape<double> tape;
    const Tensor<double> a = random_pm1<double>(Shape{3, 4}, rng);
    const Var<double> va = tape.input(a), vs = tape.input(Tensor<double>::scalar(2.5));
    const Var<double> p = tape.prim(PrimKind::Mul, {va, vs});
    const Var<double> q = tape.prim(PrimKind::Add, {p, va});
    const auto grads = tape.backward(q, Tensor<double>(Shape{3, 4}, 1.0));
    double sum_a = 0;
    for (double v : a.to_host()) sum_a += v;
    CHECK(mini::close(grads.at(vs)[0], sum_a, 1e-14));
    for (double v : grads.at(va).to_host()) CHECK(v == 3.5);
}

TEST_CASE("error paths: arity, shape, seed shape, unknown kernel, device domain errors") {
    Rng rng(29);
    Tape<double> tape;
    const Var<double> va = tape.input(random_pm1<double>(Shape{2, 3}, rng));
    const Var<double> vb = tape.input(random_pm1<double>(Shape{4, 3}, rng));
    CHECK_THROWS_AS((void)mixed_broadcast(tape, mul_kernel(), {va}, MixedPolicy::CacheForward), ArityMismatch);
    CHECK_THROWS_AS((void)mixed_broadcast(tape, mul_kernel(), {va, vb}, MixedPolicy::CacheForward), ShapeMismatch);
    CHECK_THROWS_AS((void)BroadcastKernel<double>(2, 1, "no_such_kernel"), UnknownPrimitive);
    CHECK_THROWS_AS((void)BroadcastKernel<double>(0, 1, "mul"), ArityMismatch);
    const Var<double> sq = mixed_broadcast(tape, mul_kernel(), {va, va}, MixedPolicy::CacheForward)[0];
    CHECK_THROWS_AS((void)tape.backward(sq, Tensor<double>(Shape{3, 2}, 1.0)), SeedShapeMismatch);
    Tape<double> t2;
    const Var<double> neg = t2.input(Tensor<double>::from(Shape{2, 2}, {1.0, 2.0, -1.0, 3.0}));
    bool threw = false;
    try {
        (void)mixed_broadcast(t2, BroadcastKernel<double>(1, 1, "log"), {neg}, MixedPolicy::CacheForward);
    } catch (const DomainError& e) {
        threw = std::string(e.what()).find("at output index (1, 0)") != std::string::npos;
    }
    CHECK(threw);
}

MINI_MAIN
