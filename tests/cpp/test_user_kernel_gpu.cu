// User device bodies (include/bcad/device_kernel.cuh) and the body check of
// the reference-signature BroadcastKernel constructor (include/bcad/kernel.hpp),
// on the B200. Reference behaviour replaced: proj/include/bcad/kernel.hpp:26-43
// (any generic lambda becomes a kernel body).
#include <cmath>
#include <vector>

#include "bcad/bcad.hpp"
#include "bcad/device_kernel.cuh"
#include "mini_test.hpp"

// Two bodies registered from this translation unit at load time.
BCAD_DEVICE_KERNEL_NOTHROW(UserSoftGate, "user_soft_gate", 2, 1,
                           out[0] = sigmoid(in[0]) * tanh(in[1]) + in[0] * in[0])
BCAD_DEVICE_KERNEL(UserLogRatio, "user_log_ratio", 2, 2, out[0] = log(in[0]) / in[1]; out[1] = in[0] * in[1])
// branches on argument 1 only (a (B)-shaped gate): lane-vector evaluation when it is row-uniform
BCAD_DEVICE_KERNEL_NOTHROW_P(UserGatedSoftplus, "user_gated_softplus", 2, 1, 0x2u,
                             out[0] = in[1] > 0.5 ? log(1.0 + exp(in[0])) : in[0] * sigmoid(in[0]))

namespace {
// A body under a name the library already has, registered by hand below.
struct ShadowMul {
    static constexpr const char* kName = "mul";
    static constexpr int kIn = 2, kOut = 1;
    static constexpr bool kMayRaise = false;
    static constexpr uint32_t kPredicateArgs = ~0u;
    static constexpr bool kSelectForm = false;
    template <class S>
    BCAD_HD static void body(const S* in, S* out) { out[0] = in[0] + in[1]; }
    template <class S>
    BCAD_HD static void body_select(const S* in, S* out) { out[0] = in[0] + in[1]; }
};
}  // namespace

using namespace bcad;

namespace {
const auto soft_gate_body = [](auto in, auto out) { out[0] = sigmoid(in[0]) * tanh(in[1]) + in[0] * in[0]; };
}

TEST_CASE("a user body registered from an nvcc TU runs the mixed step; gradients match host duals") {
    for (MixedPolicy policy : {MixedPolicy::CacheForward, MixedPolicy::RecomputeReverse}) {
        const BroadcastKernel<double> k(2, 1, "user_soft_gate", soft_gate_body);
        Rng rng(5);
        const std::int64_t B = 37, H = 24;
        const Tensor<double> x = random_pm1<double>(Shape{B, H}, rng);
        const Tensor<double> b = random_pm1<double>(Shape{1, H}, rng);
        const Tensor<double> w = random_pm1<double>(Shape{B, H}, rng);
        Tape<double> tape;
        const Var<double> vx = tape.input(x), vb = tape.input(b);
        const Var<double> vy = mixed_broadcast(tape, k, {vx, vb}, policy)[0];
        const auto grads = tape.backward(vy, w);
        const auto hx = x.to_host(), hb = b.to_host(), hw = w.to_host(), hy = tape.value(vy).to_host();
        const auto gx = grads.at(vx).to_host(), gb = grads.at(vb).to_host();
        std::vector<double> want_gb(static_cast<std::size_t>(H), 0.0);
        for (std::int64_t r = 0; r < B; ++r)
            for (std::int64_t c = 0; c < H; ++c) {
                const std::size_t e = static_cast<std::size_t>(r * H + c);
                const Tag tag = fresh_tag();
                const double pt[2] = {hx[e], hb[static_cast<std::size_t>(c)]};
                Dual<double> in[2], out[1];
                seed_into<double>(std::span<const double>(pt, 2), tag, std::span<Dual<double>>(in, 2));
                k.eval(std::span<const Dual<double>>(in, 2), std::span<Dual<double>>(out, 1));
                CHECK(mini::close(hy[e], out[0].primal(), 1e-12, 1e-14));
                CHECK(mini::close(gx[e], hw[e] * out[0].partial_for(tag, 0), 1e-12, 1e-14));
                want_gb[static_cast<std::size_t>(c)] += hw[e] * out[0].partial_for(tag, 1);
            }
        for (std::int64_t c = 0; c < H; ++c)
            CHECK(mini::close(gb[static_cast<std::size_t>(c)], want_gb[static_cast<std::size_t>(c)], 1e-12, 1e-13));
    }
}

TEST_CASE("a lambda under a registered name that computes something else is refused") {
    CHECK_THROWS_AS((BroadcastKernel<double>(2, 1, "mul", [](auto in, auto out) { out[0] = in[0] + in[1]; })),
                    ConfigError);
    CHECK_THROWS_AS((BroadcastKernel<float>(2, 1, "user_soft_gate",
                                            [](auto in, auto out) { out[0] = sigmoid(in[0]) * tanh(in[1]); })),
                    ConfigError);
    // ... a body that differs only on one branch is caught by the exact 0 / 1 probe values
    CHECK_THROWS_AS((BroadcastKernel<double>(6, 1, "hmlstm_update",
                                             [](auto in, auto out) {
                                                 if (in[4] == 0.0 && in[5] == 1.0)
                                                     out[0] = sigmoid(in[1]) * in[0] + sigmoid(in[2]) * tanh(in[3]);
                                                 else if (in[4] == 0.0 && in[5] == 0.0)
                                                     out[0] = in[0];
                                                 else
                                                     out[0] = sigmoid(in[2]) * tanh(in[1]);  // FLUSH on the wrong gate
                                             })),
                    ConfigError);
    // the same math under the same names is accepted
    const BroadcastKernel<double> ok(2, 1, "mul", [](auto in, auto out) { out[0] = in[0] * in[1]; });
    CHECK(ok.has_host_body());
    const BroadcastKernel<float> okf(2, 1, "user_soft_gate", soft_gate_body);
    CHECK(okf.name() == "user_soft_gate");
}

TEST_CASE("registering a second body under a taken name is refused by the C-ABI") {
    static const bcad_cu_kernel_entry shadow = BCAD_ENTRY(ShadowMul);
    CHECK(bcad_cu_register_kernel(&shadow) == BCAD_CU_ERR_CONFIG);
    CHECK(std::string(bcad_cu_last_error()).find("already registered") != std::string::npos);
    // "mul" still multiplies
    const BroadcastKernel<double> k(2, 1, "mul");
    const double p[2] = {3.0, 4.0};
    double y = 0;
    k.eval(std::span<const double>(p, 2), std::span<double>(&y, 1));
    CHECK(y == 12.0);
}

TEST_CASE("a device-only kernel evaluates on the device, reals and duals") {
    const BroadcastKernel<double> dev(2, 1, "user_soft_gate");
    const BroadcastKernel<double> host(2, 1, "user_soft_gate", soft_gate_body);
    CHECK(!dev.has_host_body());
    const double p[2] = {0.3, -0.8};
    double yd = 0, yh = 0;
    dev.eval(std::span<const double>(p, 2), std::span<double>(&yd, 1));
    host.eval(std::span<const double>(p, 2), std::span<double>(&yh, 1));
    CHECK(mini::close(yd, yh, 1e-14, 0));
    const Tag tag = fresh_tag();
    Dual<double> in[2], od[1], oh[1];
    seed_into<double>(std::span<const double>(p, 2), tag, std::span<Dual<double>>(in, 2));
    dev.eval(std::span<const Dual<double>>(in, 2), std::span<Dual<double>>(od, 1));
    host.eval(std::span<const Dual<double>>(in, 2), std::span<Dual<double>>(oh, 1));
    for (int j = 0; j < 2; ++j) CHECK(mini::close(od[0].partial_for(tag, j), oh[0].partial_for(tag, j), 1e-13, 1e-15));
}

TEST_CASE("a user body with declared predicate arguments: lane-vector path equals the per-cell path") {
    const auto body = [](auto in, auto out) {
        out[0] = in[1] > 0.5 ? log(1.0 + exp(in[0])) : in[0] * sigmoid(in[0]);
    };
    for (int pass = 0; pass < 2; ++pass) {
        const BroadcastKernel<float> k(2, 1, "user_gated_softplus", body);
        Rng rng(21);
        const std::int64_t B = 64, H = 256;
        const Tensor<float> x = random_pm1<float>(Shape{B, H}, rng);
        // pass 0: gate of shape (B) (row-uniform -> lane vectors); pass 1: (B, H) (per cell)
        const Tensor<float> gate = pass == 0 ? random_binary<float>(Shape{B}, rng) : random_binary<float>(Shape{B, H}, rng);
        const Tensor<float> w = random_pm1<float>(Shape{B, H}, rng);
        Tape<float> tape;
        const Var<float> vx = tape.input(x), vg = tape.input(gate);
        const Var<float> vy = mixed_broadcast(tape, k, {vx, vg}, MixedPolicy::CacheForward)[0];
        const auto grads = tape.backward(vy, w);
        const auto hx = x.to_host(), hg = gate.to_host(), hw = w.to_host(), hy = tape.value(vy).to_host();
        const auto gx = grads.at(vx).to_host(), gg = grads.at(vg).to_host();
        for (std::int64_t r = 0; r < B; ++r)
            for (std::int64_t c = 0; c < H; ++c) {
                const std::size_t e = static_cast<std::size_t>(r * H + c);
                const float gv = hg[static_cast<std::size_t>(pass == 0 ? r : r * H + c)];
                const Tag tag = fresh_tag();
                const float pt[2] = {hx[e], gv};
                Dual<float> in[2], out[1];
                seed_into<float>(std::span<const float>(pt, 2), tag, std::span<Dual<float>>(in, 2));
                k.eval(std::span<const Dual<float>>(in, 2), std::span<Dual<float>>(out, 1));
                CHECK(mini::close(hy[e], out[0].primal(), 1e-5, 1e-6));
                CHECK(mini::close(gx[e], hw[e] * out[0].partial_for(tag, 0), 1e-5, 1e-6));
            }
        for (float v : gg) CHECK(v == 0.0f);  // the gate only feeds the comparison
    }
}

TEST_CASE("a may-raise user body reports the failing output index") {
    const BroadcastKernel<double> k(2, 2, "user_log_ratio");
    CHECK(k.may_raise());
    const Tensor<double> a = Tensor<double>::from(Shape{2, 2}, {1.0, 2.0, -3.0, 4.0});
    const Tensor<double> b = Tensor<double>::from(Shape{2, 2}, {1.0, 1.0, 1.0, 1.0});
    try {
        (void)broadcast_diag_jacobian(k, false, a, b);
        CHECK(false);
    } catch (const DomainError& e) {
        CHECK(std::string(e.what()).find("(1, 0)") != std::string::npos);
    }
    const Tensor<double> z = Tensor<double>::from(Shape{2, 2}, {1.0, 0.0, 1.0, 1.0});
    CHECK_THROWS_AS((void)broadcast_diag_jacobian(k, false, b, z), DivisionByZero);
}

TEST_CASE("compose_kernels applies its stages in turn; differentiating a composition is refused") {
    const BroadcastKernel<double> t(1, 1, "tanh"), s(1, 1, "sigmoid");
    const BroadcastKernel<double> c = compose_kernels(s, t);
    CHECK(c.is_composite());
    CHECK(c.name() == "sigmoid.tanh");
    Rng rng(37);
    const Tensor<double> x = random_pm1<double>(Shape{8, 8}, rng);
    const auto before = counter_totals().kernel_element_visits;
    const auto fused = broadcast_apply(c, x);
    CHECK(counter_totals().kernel_element_visits - before == 128);  // two launches over 64 cells
    const auto two_pass = broadcast_apply(s, broadcast_apply(t, x)[0]);
    const auto a = fused[0].to_host(), b = two_pass[0].to_host();
    for (std::size_t e = 0; e < a.size(); ++e) CHECK(a[e] == b[e]);
    // one scalar evaluation runs the stages too
    const double p[1] = {0.3};
    double y = 0, mid = 0, want = 0;
    c.eval(std::span<const double>(p, 1), std::span<double>(&y, 1));
    t.eval(std::span<const double>(p, 1), std::span<double>(&mid, 1));
    s.eval(std::span<const double>(&mid, 1), std::span<double>(&want, 1));
    CHECK(y == want);
    CHECK_THROWS_AS((void)broadcast_diag_jacobian(c, false, x), ConfigError);
    Tape<double> tape;
    const Var<double> v = tape.input(x);
    CHECK_THROWS_AS((void)mixed_broadcast(tape, c, {v}, MixedPolicy::CacheForward), ConfigError);
    CHECK_THROWS_AS((void)compose_kernels(BroadcastKernel<double>(2, 1, "mul"), t), ArityMismatch);
}

TEST_CASE("reduce_sum_keepdims and make_broadcast_plan (bcad/broadcast.hpp)") {
    Rng rng(41);
    const Tensor<double> a = random_pm1<double>(Shape{5, 6}, rng);
    const int ax[1] = {1};
    const Tensor<double> r = reduce_sum_keepdims(a, std::span<const int>(ax, 1));
    CHECK(r.shape() == (Shape{5, 1}));
    const auto ha = a.to_host(), hr = r.to_host();
    for (int i = 0; i < 5; ++i) {
        double want = 0;
        for (int j = 0; j < 6; ++j) want += ha[static_cast<std::size_t>(i * 6 + j)];
        CHECK(mini::close(hr[static_cast<std::size_t>(i)], want, 1e-15, 1e-15));
    }
    const Shape shapes[2] = {Shape{5, 6}, Shape{5}};
    const BroadcastPlan plan = make_broadcast_plan(std::span<const Shape>(shapes, 2));
    CHECK(plan.volume == 30);
    CHECK(plan.arg_strides[0] == (std::vector<std::int64_t>{6, 1}));
    CHECK(plan.arg_strides[1] == (std::vector<std::int64_t>{1, 0}));
    const int bad[1] = {2};
    CHECK_THROWS_AS((void)reduce_sum_keepdims(a, std::span<const int>(bad, 1)), ShapeMismatch);
}

int main() { return mini::run_all(); }
