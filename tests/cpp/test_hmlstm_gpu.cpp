// Drop-in C++ API on the GPU: the HM-LSTM cell-update claims of the
// reference's suite (proj/tests/test_hmlstm.cpp), re-expressed against the
// device-backed Tape / mixed_broadcast. Host-side expectations use libm, so
// values that pass through a transcendental compare with the reference's
// own fp64 tolerances (1e-12 / 1e-14) instead of bit equality; structural
// claims (COPY identity, zero boundary gradients, policy equivalence,
// fused == unfused primal, node counts, cached bytes) stay exact.
#include <cmath>
#include <vector>

#include "bcad/bcad.hpp"
#include "mini_test.hpp"

using namespace bcad;

namespace {

double host_sigmoid(double x) {  // two-branch form (dual.hpp:38-48)
    if (x >= 0) return 1.0 / (1.0 + std::exp(-x));
    const double e = std::exp(x);
    return e / (1.0 + e);
}

double host_cell(double c, double f, double i, double g, double z1, double z2) {
    if (z1 == 0.0 && z2 == 1.0) return host_sigmoid(f) * c + host_sigmoid(i) * std::tanh(g);
    if (z1 == 0.0 && z2 == 0.0) return c;
    return host_sigmoid(i) * std::tanh(g);
}

template <class Real>
CellInputs<Real> all_z(std::int64_t n, Rng& rng, Real z1, Real z2) {
    CellInputs<Real> in = random_cell_inputs<Real>(n, rng);
    in.z1 = Tensor<Real>(Shape{n}, z1);
    in.z2 = Tensor<Real>(Shape{n}, z2);
    return in;
}

template <class Real>
bool identical(const Tensor<Real>& a, const Tensor<Real>& b) {
    if (!(a.shape() == b.shape())) return false;
    return a.to_host() == b.to_host();
}

template <class Real>
bool all_close(const std::vector<Real>& a, const std::vector<Real>& b, double rtol, double atol) {
    if (a.size() != b.size()) return false;
    for (std::size_t e = 0; e < a.size(); ++e)
        if (!mini::close(double(a[e]), double(b[e]), rtol, atol)) return false;
    return true;
}

}  // namespace

TEST_CASE("scalar update cases through 1x1 mixed nodes: UPDATE, COPY, FLUSH") {
    const double cases[][7] = {{1.0, 0.0, 0.0, 0.0, 0.0, 1.0, 0.5},
                               {7.0, 0.3, -0.2, 0.9, 0.0, 0.0, 7.0},
                               {3.0, 0.1, 0.0, 0.0, 1.0, 1.0, 0.0},
                               {3.0, 0.1, 0.0, 0.0, 1.0, 0.0, 0.0}};  // (1,0) flushes too
    for (const auto& c : cases) {
        std::vector<Tensor<double>> t;
        for (int k = 0; k < 6; ++k) t.push_back(Tensor<double>::scalar(c[k]));
        const auto out = broadcast_apply(cell_update_kernel<double>(), t[0], t[1], t[2], t[3], t[4], t[5]);
        CHECK(out[0][0] == c[6]);
    }
}

TEST_CASE("fused cell update matches a scalar loop cell for cell") {
    Rng rng(3);
    const std::int64_t n = 6;
    const CellInputs<double> in = random_cell_inputs<double>(n, rng);
    Tape<double> tape;
    const CellGraph<double> graph = cell_update_fused(tape, in, MixedPolicy::CacheForward);
    const auto out = tape.value(graph.out).to_host();
    const auto c = in.c_prev.to_host(), f = in.f.to_host(), i = in.i.to_host(), g = in.g.to_host();
    const auto z1 = in.z1.to_host(), z2 = in.z2.to_host();
    CHECK(tape.value(graph.out).shape() == (Shape{n, n}));
    for (std::int64_t r = 0; r < n; ++r)
        for (std::int64_t k = 0; k < n; ++k) {
            const std::size_t e = std::size_t(r * n + k);
            CHECK(mini::close(out[e], host_cell(c[e], f[e], i[e], g[e], z1[std::size_t(r)], z2[std::size_t(r)]), 1e-12, 1e-14));
        }
}

TEST_CASE("all-COPY boundary input returns c_prev exactly") {
    Rng rng(5);
    const CellInputs<double> in = all_z<double>(5, rng, 0.0, 0.0);
    Tape<double> tape;
    const CellGraph<double> graph = cell_update_fused(tape, in, MixedPolicy::RecomputeReverse);
    CHECK(identical(tape.value(graph.out), in.c_prev));
}

TEST_CASE("all-UPDATE boundary input reduces to the gate formula") {
    Rng rng(7);
    const std::int64_t n = 4;
    const CellInputs<double> in = all_z<double>(n, rng, 0.0, 1.0);
    Tape<double> tape;
    const CellGraph<double> graph = cell_update_fused(tape, in, MixedPolicy::CacheForward);
    const auto out = tape.value(graph.out).to_host();
    const auto c = in.c_prev.to_host(), f = in.f.to_host(), i = in.i.to_host(), g = in.g.to_host();
    for (std::size_t e = 0; e < out.size(); ++e)
        CHECK(mini::close(out[e], host_sigmoid(f[e]) * c[e] + host_sigmoid(i[e]) * std::tanh(g[e]), 1e-12, 1e-14));
}

TEST_CASE("unfused primal is bit-identical to the fused primal (device)") {
    for (std::int64_t n : {std::int64_t{1}, std::int64_t{8}, std::int64_t{64}}) {
        Rng rng(static_cast<std::uint64_t>(n) + 100);
        const CellInputs<double> in = random_cell_inputs<double>(n, rng);
        Tape<double> a, b;
        const CellGraph<double> fused = cell_update_fused(a, in, MixedPolicy::CacheForward);
        const CellGraph<double> unfused = cell_update_unfused(b, in);
        CHECK(identical(a.value(fused.out), b.value(unfused.out)));
    }
}

TEST_CASE("unfused node count is fixed at 14; the mixed graph is 7") {
    Rng rng(9);
    for (std::int64_t n : {std::int64_t{2}, std::int64_t{32}}) {
        const CellInputs<double> in = random_cell_inputs<double>(n, rng);
        Tape<double> t1, t2;
        (void)cell_update_unfused(t1, in);
        (void)cell_update_fused(t2, in, MixedPolicy::CacheForward);
        CHECK(t1.size() == 14);
        CHECK(t2.size() == 7);
    }
}

TEST_CASE("single-cell graph reproduces the scalar gradient examples") {
    CellInputs<double> in{Tensor<double>(Shape{1, 1}, 1.0), Tensor<double>(Shape{1, 1}, 0.0),
                          Tensor<double>(Shape{1, 1}, 0.0), Tensor<double>(Shape{1, 1}, 0.0),
                          Tensor<double>(Shape{1}, 0.0),    Tensor<double>(Shape{1}, 1.0)};
    const Tensor<double> seed(Shape{1, 1}, 1.0);
    for (CellImpl impl : {CellImpl::FusedMixedCache, CellImpl::FusedMixedRecompute, CellImpl::ReverseUnfused}) {
        const CellGradients<double> g = cell_gradients(impl, in, seed);
        CHECK(g.c_prev[0] == 0.5);
        CHECK(g.f[0] == 0.25);
        CHECK(g.i[0] == 0.0);
        CHECK(g.g[0] == 0.5);
    }
}

TEST_CASE("gradient 4-tuples match the piecewise closed forms per cell") {
    for (std::uint64_t sid = 1; sid <= 6; ++sid) {
        Rng rng(sid * 13);
        const std::int64_t n = 8;
        const CellInputs<double> in = random_cell_inputs<double>(n, rng);
        const Tensor<double> seed = random_pm1<double>(Shape{n, n}, rng);
        const auto c = in.c_prev.to_host(), f = in.f.to_host(), i = in.i.to_host(), g = in.g.to_host();
        const auto z1 = in.z1.to_host(), z2 = in.z2.to_host(), w = seed.to_host();
        std::vector<double> dc(c.size(), 0.0), df(c.size(), 0.0), di(c.size(), 0.0), dg(c.size(), 0.0);
        for (std::int64_t r = 0; r < n; ++r)
            for (std::int64_t k = 0; k < n; ++k) {
                const std::size_t e = std::size_t(r * n + k);
                const double sf = host_sigmoid(f[e]), si = host_sigmoid(i[e]), tg = std::tanh(g[e]);
                const bool upd = z1[std::size_t(r)] == 0.0 && z2[std::size_t(r)] == 1.0;
                const bool cpy = z1[std::size_t(r)] == 0.0 && z2[std::size_t(r)] == 0.0;
                if (upd) {
                    dc[e] = w[e] * sf;
                    df[e] = w[e] * (sf * (1 - sf) * c[e]);
                }
                if (cpy) dc[e] = w[e];
                if (!cpy) {
                    di[e] = w[e] * (si * (1 - si) * tg);
                    dg[e] = w[e] * (si * (1 - tg * tg));
                }
            }
        for (CellImpl impl : {CellImpl::FusedMixedCache, CellImpl::FusedMixedRecompute, CellImpl::ReverseUnfused}) {
            const CellGradients<double> got = cell_gradients(impl, in, seed);
            CHECK(all_close(got.c_prev.to_host(), dc, 1e-12, 1e-14));
            CHECK(all_close(got.f.to_host(), df, 1e-12, 1e-14));
            CHECK(all_close(got.i.to_host(), di, 1e-12, 1e-14));
            CHECK(all_close(got.g.to_host(), dg, 1e-12, 1e-14));
        }
    }
}

TEST_CASE("gradients match device finite differences") {
    Rng rng(31);
    const std::int64_t n = 5;
    const CellInputs<double> in = random_cell_inputs<double>(n, rng);
    const Tensor<double> seed(Shape{n, n}, 1.0);
    const CellGradients<double> got = cell_gradients(CellImpl::FusedMixedCache, in, seed);
    const auto sum_out = [&](const std::vector<Tensor<double>>& x) {
        const auto o = broadcast_apply(cell_update_kernel<double>(), x[0], x[1], x[2], x[3], in.z1, in.z2)[0].to_host();
        double s = 0;
        for (double v : o) s += v;
        return s;
    };
    const std::vector<const Tensor<double>*> grads = {&got.c_prev, &got.f, &got.i, &got.g};
    std::vector<Tensor<double>> x = {in.c_prev, in.f, in.i, in.g};
    for (int j = 0; j < 4; ++j) {
        auto base = x[std::size_t(j)].to_host();
        const auto gj = grads[std::size_t(j)]->to_host();
        for (std::size_t e = 0; e < base.size(); e += 3) {
            const double h = std::cbrt(2.220446049250313e-16) * std::max(1.0, std::fabs(base[e]));
            auto p = base;
            p[e] = base[e] + h;
            x[std::size_t(j)] = Tensor<double>::from(Shape{n, n}, p);
            const double up = sum_out(x);
            p[e] = base[e] - h;
            x[std::size_t(j)] = Tensor<double>::from(Shape{n, n}, p);
            const double down = sum_out(x);
            x[std::size_t(j)] = Tensor<double>::from(Shape{n, n}, base);
            CHECK(mini::close(gj[e], (up - down) / (2 * h), 1e-5, 1e-7));
        }
    }
}

TEST_CASE("no gradient flows to the boundary vectors") {
    Rng rng(37);
    const std::int64_t n = 4;
    const CellInputs<double> in = random_cell_inputs<double>(n, rng);
    const Tensor<double> seed(Shape{n, n}, 1.0);
    Tape<double> t1;
    const CellGraph<double> fused = cell_update_fused(t1, in, MixedPolicy::CacheForward);
    const auto g1 = t1.backward(fused.out, seed);
    Tape<double> t2;
    const CellGraph<double> unfused = cell_update_unfused(t2, in);
    const auto g2 = t2.backward(unfused.out, seed);
    for (double v : g1.at(fused.z1).to_host()) CHECK(v == 0.0);
    for (double v : g1.at(fused.z2).to_host()) CHECK(v == 0.0);
    for (double v : g2.at(unfused.z1).to_host()) CHECK(v == 0.0);
    for (double v : g2.at(unfused.z2).to_host()) CHECK(v == 0.0);
}

TEST_CASE("both policies produce bit-identical gradients") {
    Rng rng(11);
    const CellInputs<double> cell = random_cell_inputs<double>(5, rng);
    const std::vector<Tensor<double>> args = {cell.c_prev, cell.f, cell.i, cell.g, cell.z1, cell.z2};
    CHECK(policy_equivalence_check<double>(cell_update_kernel<double>(), args));
    const std::vector<Tensor<double>> prod = {random_pm1<double>(Shape{4, 3}, rng), random_pm1<double>(Shape{4, 1}, rng)};
    CHECK(policy_equivalence_check<double>(BroadcastKernel<double>(2, 1, "mul"), prod));
}

TEST_CASE("cell input validation") {
    Rng rng(47);
    CellInputs<double> in = random_cell_inputs<double>(3, rng);
    in.validate();
    CellInputs<double> bad = random_cell_inputs<double>(3, rng);
    bad.f = random_pm1<double>(Shape{3, 4}, rng);
    CHECK_THROWS_AS(bad.validate(), ShapeMismatch);
    CellInputs<double> badz = random_cell_inputs<double>(3, rng);
    badz.z1 = Tensor<double>(Shape{3}, 0.5);
    CHECK_THROWS_AS(badz.validate(), Error);
}

TEST_CASE("32-bit path: fused and unfused agree") {
    Rng rng(53);
    const std::int64_t n = 6;
    const CellInputs<float> in = random_cell_inputs<float>(n, rng);
    const Tensor<float> seed(Shape{n, n}, 1.0f);
    const CellGradients<float> a = cell_gradients(CellImpl::FusedMixedCache, in, seed);
    const CellGradients<float> b = cell_gradients(CellImpl::ReverseUnfused, in, seed);
    CHECK(all_close(a.c_prev.to_host(), b.c_prev.to_host(), 1e-4, 1e-6));
    CHECK(all_close(a.f.to_host(), b.f.to_host(), 1e-4, 1e-6));
    CHECK(all_close(a.i.to_host(), b.i.to_host(), 1e-4, 1e-6));
    CHECK(all_close(a.g.to_host(), b.g.to_host(), 1e-4, 1e-6));
}

TEST_CASE("non-square (B,H) with per-row z and per-unit (1,H) bias through mixed_broadcast") {
    Rng rng(mix_seed(42, 64 * 1000003 + 128));
    const std::int64_t B = 64, H = 128;
    Tape<float> tape;
    std::vector<Var<float>> v;
    for (int k = 0; k < 4; ++k) v.push_back(tape.input(random_pm1<float>(Shape{B, H}, rng)));
    for (int k = 0; k < 3; ++k) v.push_back(tape.input(random_pm1<float>(Shape{1, H}, rng)));
    for (int k = 0; k < 2; ++k) v.push_back(tape.input(random_binary<float>(Shape{B}, rng)));
    const auto out = mixed_broadcast<float>(tape, cell_update_bias_kernel<float>(), std::span<const Var<float>>(v),
                                            MixedPolicy::CacheForward);
    CHECK(tape.value(out[0]).shape() == (Shape{B, H}));
    const auto grads = tape.backward(out[0], Tensor<float>(Shape{B, H}, 1.0f));
    CHECK(grads.at(v[4]).shape() == (Shape{1, H}));
    CHECK(grads.at(v[7]).shape() == (Shape{B}));
    for (float z : grads.at(v[7]).to_host()) CHECK(z == 0.0f);
}

MINI_MAIN
