"""GPU parity: the sm_100a path (through the C-ABI) against the CPU oracle.

Comparator: SURVEY Appendix A — elementwise |a-b| <= atol + rtol*max(|a|,|b|)
with (rtol, atol) = (1e-5, 1e-6) fp32 / (1e-12, 1e-14) fp64 (the reference's
own close(), tests/support/test_util.hpp:11-14); reduced adjoints against the
oracle's fp64-accumulated sum of the same rounded terms; branch decisions,
COPY primals and boundary-vector gradients bit-exact.
"""
import numpy as np
import pytest

import oracle as O
from helpers import GpuRunner, assert_close, assert_grads, step_terms, tol_for

pytestmark = pytest.mark.gpu

DTYPES = [np.float32, np.float64]
VARIANTS = ["canonical", "bias", "divergence"]


@pytest.fixture(scope="module")
def gpu():
    return GpuRunner()


def branch_class_from_z(z1, z2):
    # hmlstm.hpp:51-53 ordered predicate: 0 UPDATE, 1 COPY, 2 FLUSH
    z1 = np.asarray(z1)
    z2 = np.asarray(z2)
    upd = (z1 == 0) & (z2 == 1)
    cp = (z1 == 0) & (z2 == 0)
    return np.where(upd, 0, np.where(cp, 1, 2))


def branch_class_from_dc(dc):
    # Appendix A: D_c exactly 1 -> COPY, exactly 0 -> FLUSH, else UPDATE
    return np.where(dc == 1.0, 1, np.where(dc == 0.0, 2, 0))


def _z_full(z, shape):
    z = np.asarray(z)
    return np.broadcast_to(z.reshape(z.shape + (1,) * (len(shape) - z.ndim)), shape)


@pytest.mark.parametrize("dtype", DTYPES)
@pytest.mark.parametrize("variant", VARIANTS)
@pytest.mark.parametrize("policy", [O.CACHE_FORWARD, O.RECOMPUTE_REVERSE])
def test_hmlstm_config1(gpu, oracle_lib, dtype, variant, policy):
    """BASELINE config 1 (B=32, H=256) and its bias / divergence variants."""
    B, H = 32, 256
    ins = O.hmlstm_inputs(oracle_lib, B, H, dtype, variant)
    name = O.hmlstm_kernel(variant)
    rtol, atol = tol_for(dtype)
    want_p, want_d = oracle_lib.forward(name, ins)
    want_p_pol, want_g, want_a64 = oracle_lib.mixed_step(name, ins, policy)
    got_p, got_d, got_g = gpu.step(name, ins, policy=policy)

    assert_close(got_p[0], want_p_pol[0], rtol, atol, "primal")
    if policy == O.CACHE_FORWARD:
        for j, (g, w) in enumerate(zip(got_d, want_d)):
            assert_close(g, w, rtol, atol, f"partial D_0{j}")
        # branch decisions, bit-exact
        z1, z2 = ins[-2], ins[-1]
        want_cls = branch_class_from_z(_z_full(z1, (B, H)), _z_full(z2, (B, H)))
        assert np.array_equal(branch_class_from_dc(got_d[0]), want_cls)
    out_shape = (B, H)
    assert_grads(got_g, want_g, want_a64, [a.shape for a in ins], out_shape, dtype, f"{variant}",
                 terms=step_terms(oracle_lib, gpu, name, ins))
    # COPY primal == c, bit-exact; z gradients exactly zero
    cls = branch_class_from_z(_z_full(ins[-2], out_shape), _z_full(ins[-1], out_shape))
    assert np.array_equal(got_p[0][cls == 1], ins[0][cls == 1])
    assert np.all(got_g[-1] == 0) and np.all(got_g[-2] == 0)


@pytest.mark.parametrize("dtype", DTYPES)
def test_hmlstm_bias_1024_multitile(gpu, oracle_lib, dtype):
    """Config 3 at full size: (1,H) reductions over 1024 rows span many row
    tiles (cross-CTA fixed-order combination), (B) reductions many column tiles."""
    B, H = 1024, 1024
    ins = O.hmlstm_inputs(oracle_lib, B, H, dtype, "bias")
    rng = np.random.default_rng(5)
    seed = rng.uniform(-1, 1, (B, H)).astype(dtype)
    _, want_g, want_a64 = oracle_lib.mixed_step("hmlstm_update_bias", ins, seeds=[seed])
    terms = step_terms(oracle_lib, gpu, "hmlstm_update_bias", ins, [seed])
    for policy in (O.CACHE_FORWARD, O.RECOMPUTE_REVERSE):
        _, _, got_g = gpu.step("hmlstm_update_bias", ins, seeds=[seed], policy=policy)
        assert_grads(got_g, want_g, want_a64, [a.shape for a in ins], (B, H), dtype, f"bias1024 p{policy}",
                     terms=terms)


def random_shapes(rng, n_args, max_rank=3, max_len=4):
    """Broadcast-compatible random shapes (tests/support/kernel_pool.hpp:107-125)."""
    rank = 1 + int(rng.integers(0, max_rank))
    out = [1 + int(rng.integers(0, max_len)) for _ in range(rank)]
    shapes = []
    for _ in range(n_args):
        keep = int(rng.integers(0, rank + 1)) if rng.integers(0, 4) == 0 else rank
        shapes.append(tuple(1 if rng.integers(0, 3) == 0 else out[k] for k in range(keep)))
    return shapes


POOL = ["identity", "reflect", "tanh_sigmoid", "product", "gated", "prod_diff", "blend", "curl", "tanh_product_4",
        "hmlstm_update", "fanout", "fiveway", "wave", "gate", "sig_tanh", "square_gate", "two", "mul", "plus", "exp"]


@pytest.mark.parametrize("dtype", DTYPES)
def test_kernel_pool_random_shapes(gpu, oracle_lib, dtype):
    """Every pool kernel on random broadcast shapes (incl. rank-3, scalars,
    dropped trailing axes), both policies, random seeds, some outputs without
    an adjoint (tests/test_mixed.cpp:104-119 policy equivalence, 137-172)."""
    rng = np.random.default_rng(13)
    rtol, atol = tol_for(dtype)
    for name in POOL:
        n, m = oracle_lib.arity(name)
        for rep in range(4):
            shapes = random_shapes(rng, n)
            ins = [rng.uniform(-1, 1, s).astype(dtype) for s in shapes]
            if name == "hmlstm_update":
                for z in (4, 5):
                    ins[z] = (rng.uniform(0, 1, shapes[z]) < 0.5).astype(dtype)
            out_shape = O.broadcast_shape_py(shapes)
            seeds = [rng.uniform(-1, 1, out_shape).astype(dtype) for _ in range(m)]
            if m > 1 and rep % 2:
                seeds[0] = None
            _, want_g, want_a64 = oracle_lib.mixed_step(name, ins, O.CACHE_FORWARD, seeds)
            want_p, want_d = oracle_lib.forward(name, ins)
            for policy in (O.CACHE_FORWARD, O.RECOMPUTE_REVERSE):
                got_p, got_d, got_g = gpu.step(name, ins, seeds=seeds, policy=policy)
                tag = f"{name} {shapes} p{policy}"
                if policy == O.CACHE_FORWARD:
                    for i in range(m):
                        assert_close(got_p[i], want_p[i], rtol, atol, tag + f" primal{i}")
                    for k, (g, w) in enumerate(zip(got_d, want_d)):
                        assert_close(g, w, rtol, atol, tag + f" D{k}")
                assert_grads(got_g, want_g, want_a64, shapes, out_shape, dtype, tag,
                             terms=step_terms(oracle_lib, gpu, name, ins, seeds))


@pytest.mark.parametrize("dtype", DTYPES)
def test_policies_bit_identical(gpu, oracle_lib, dtype):
    """CacheForward and RecomputeReverse give bit-identical gradients
    (mixed.hpp:103-130), and the real-body primal equals the dual primal
    (test_forward.cpp 'requested primals are bit-identical')."""
    for variant in VARIANTS:
        ins = O.hmlstm_inputs(oracle_lib, 64, 512, dtype, variant)
        name = O.hmlstm_kernel(variant)
        p0, _, g0 = gpu.step(name, ins, policy=O.CACHE_FORWARD)
        p1, _, g1 = gpu.step(name, ins, policy=O.RECOMPUTE_REVERSE)
        assert np.array_equal(p0[0], p1[0])
        for a, b in zip(g0, g1):
            assert np.array_equal(a, b)


def test_deterministic_run_to_run(gpu, oracle_lib):
    ins = O.hmlstm_inputs(oracle_lib, 512, 1024, np.float32, "bias")
    r1 = gpu.step("hmlstm_update_bias", ins)
    r2 = gpu.step("hmlstm_update_bias", ins)
    for a, b in zip(r1[0] + r1[1] + r1[2], r2[0] + r2[1] + r2[2]):
        assert np.array_equal(a.view(np.uint8), b.view(np.uint8))


@pytest.mark.parametrize("dtype", DTYPES)
def test_accumulate_into_existing_slots(gpu, oracle_lib, dtype):
    """accumulate_adjoint adds into an existing slot (tape.hpp:179-183)."""
    rng = np.random.default_rng(3)
    ins = O.hmlstm_inputs(oracle_lib, 64, 256, dtype, "bias")
    existing = [rng.uniform(-1, 1, a.shape).astype(dtype) for a in ins]
    existing[7] = None  # z1 slot fresh
    _, _, got = gpu.step("hmlstm_update_bias", ins, existing=existing)
    prim, parts = oracle_lib.forward("hmlstm_update_bias", ins)
    want = [e.copy() if e is not None else np.zeros(a.shape, dtype) for e, a in zip(existing, ins)]
    acc64 = oracle_lib.pullback([a.shape for a in ins], [np.ones((64, 256), dtype)], parts, want,
                                accumulate=[e is not None for e in existing])
    assert_grads(got, want, acc64, [a.shape for a in ins], (64, 256), dtype, "accumulate",
                 terms=step_terms(oracle_lib, gpu, "hmlstm_update_bias", ins))


@pytest.mark.parametrize("dtype", DTYPES)
@pytest.mark.parametrize("shape", [(1, 1), (7, 1023), (3, 5), (1, 4096), (4096, 1), (33, 66)])
def test_edge_shapes(gpu, oracle_lib, dtype, shape):
    """Odd widths (generic path), single cells, single rows/columns."""
    B, H = shape
    rng = np.random.default_rng(B * 7 + H)
    ins = [rng.uniform(-1, 1, (B, H)).astype(dtype) for _ in range(4)]
    ins += [rng.uniform(-1, 1, (1, H)).astype(dtype) for _ in range(3)]
    ins += [(rng.uniform(0, 1, (B,)) < 0.5).astype(dtype) for _ in range(2)]
    rtol, atol = tol_for(dtype)
    want_p, want_g, want_a64 = oracle_lib.mixed_step("hmlstm_update_bias", ins)
    for policy in (0, 1):
        got_p, _, got_g = gpu.step("hmlstm_update_bias", ins, policy=policy)
        assert_close(got_p[0], want_p[0], rtol, atol, f"{shape} primal")
        assert_grads(got_g, want_g, want_a64, [a.shape for a in ins], (B, H), dtype, f"{shape}",
                     terms=step_terms(oracle_lib, gpu, "hmlstm_update_bias", ins))


def test_misaligned_views_take_scalar_tiled_path(gpu, oracle_lib):
    """4-byte-aligned views of a 2-D problem: the tiled kernels at one cell
    per thread (no 128-bit vectors) — forward and pullback, both policies."""
    import torch
    from paper_1810_08297_b200 import native
    rng = np.random.default_rng(9)
    B, H = 16, 64
    ins = [rng.uniform(-1, 1, (B, H)).astype(np.float32) for _ in range(4)]
    ins += [(rng.uniform(0, 1, (B,)) < 0.5).astype(np.float32) for _ in range(2)]
    k = native.Kernel("hmlstm_update")
    # offset every device buffer by one element -> 4-byte aligned only
    dins = []
    for a in ins:
        buf = torch.empty(a.size + 1, dtype=torch.float32, device="cuda")
        buf[1:] = torch.from_numpy(a.ravel()).cuda()
        dins.append(buf[1:].view(a.shape))
    prim_buf = torch.empty(B * H + 1, device="cuda")
    prim = [prim_buf[1:].view(B, H)]
    native.forward(k, dins, prim, None)
    want, _ = oracle_lib.forward("hmlstm_update", ins, real_body=True)
    assert_close(prim[0].cpu().numpy(), want[0], 1e-5, 1e-6, "misaligned primal")
    # the full step on misaligned buffers: partials, seeds and adjoints offset too
    def off_view(shape):
        n = int(np.prod(shape))
        return torch.empty(n + 1, dtype=torch.float32, device="cuda")[1:].view(shape)
    parts = [off_view((B, H)) for _ in range(6)]
    native.forward(k, dins, prim, parts)
    seed = off_view((B, H))
    seed.copy_(torch.from_numpy(rng.uniform(-1, 1, (B, H)).astype(np.float32)).cuda())
    shapes = [a.shape for a in ins]
    _, want_g, want_a64 = oracle_lib.mixed_step("hmlstm_update", ins, O.CACHE_FORWARD, [seed.cpu().numpy()])
    for policy_parts in (parts, None):
        adj = [off_view(s) for s in shapes]
        native.pullback(k, shapes, [seed], policy_parts, dins, adj, workspace=native.new_workspace(k, shapes, torch.float32))
        torch.cuda.synchronize()
        assert_grads([a.cpu().numpy() for a in adj], want_g, want_a64, shapes, (B, H), np.float32, "misaligned grads",
                     terms=step_terms(oracle_lib, gpu, "hmlstm_update", ins, [seed.cpu().numpy()]))


ERROR_CASES = [
    ("log", [np.array([[0.5, 2.0], [-1.0, 3.0]])], "DomainError", "(1, 0)"),
    ("div", [np.array([1.0, 2.0, 3.0]), np.array([1.0, 0.0, 0.0])], "DivisionByZero", "(1)"),
    ("sqrt", [np.array([4.0, 1.0, -2.0])], "DomainError", "(2)"),
    ("abs", [np.array([[1.0, -2.0], [0.0, 5.0]])], "NonDifferentiablePoint", "(1, 0)"),
    ("recip", [np.array([2.0, 0.0])], "DivisionByZero", "(1)"),
]


@pytest.mark.parametrize("name,ins,exc,where", ERROR_CASES)
def test_device_errors_report_output_index(gpu, oracle_lib, name, ins, exc, where):
    """Dual-rule errors surface as the reference exception, annotated with
    the first failing output index (forward.hpp:137-146)."""
    from paper_1810_08297_b200 import native
    with pytest.raises(O.OracleError) as oe:
        oracle_lib.forward(name, ins)
    assert where in oe.value.msg
    with pytest.raises(getattr(native, exc)) as ge:
        gpu.forward(name, ins)
    assert f"at output index {where}" in str(ge.value)
    # the real body never raises (broadcast_apply uses plain reals)
    gpu.forward(name, ins, want_partials=False)


def test_graph_capture_replays_the_step_bit_exact(oracle_lib):
    """bcad_cu_graph_capture_begin/_end/_launch: K1 -> K2 -> K2f of the bias
    variant (programmatic-dependent launches, a finisher, stream-ordered
    workspace) captured once and replayed equals the direct launches bit for
    bit — the kernels are graph-capturable as the bench's replay needs."""
    import ctypes as C
    import torch
    from paper_1810_08297_b200 import native
    ins = O.hmlstm_inputs(oracle_lib, 1024, 1024, np.float32, "bias")
    dins = [torch.from_numpy(a).cuda() for a in ins]
    shapes = [a.shape for a in ins]
    k = native.Kernel("hmlstm_update_bias")
    prim = [torch.empty((1024, 1024), device="cuda")]
    parts = [torch.empty((1024, 1024), device="cuda") for _ in range(9)]
    seed = [torch.rand((1024, 1024), device="cuda")]
    ws = native.new_workspace(k, shapes, torch.float32)
    adj_direct = [torch.empty(s, device="cuda") for s in shapes]
    adj_graph = [torch.empty(s, device="cuda") for s in shapes]
    stream = torch.cuda.Stream()
    sp = C.c_void_p(stream.cuda_stream)

    def step(adj):
        native.forward(k, dins, prim, parts, stream=stream)
        native.pullback(k, shapes, seed, parts, dins, adj, workspace=ws, stream=stream)

    step(adj_direct)
    torch.cuda.synchronize()
    native.check(native.LIB.bcad_cu_graph_capture_begin(sp))
    step(adj_graph)
    exe = C.c_void_p()
    native.check(native.LIB.bcad_cu_graph_capture_end(sp, C.byref(exe)))
    for _ in range(3):
        native.check(native.LIB.bcad_cu_graph_launch(exe, sp))
    torch.cuda.synchronize()
    native.check(native.LIB.bcad_cu_graph_destroy(exe))
    for a, b in zip(adj_direct, adj_graph):
        assert torch.equal(a, b)


ARITIES = [1, 2, 3, 4, 5, 8, 16, 18, 32]


@pytest.mark.parametrize("dtype", DTYPES)
@pytest.mark.parametrize("A", ARITIES)
def test_tanh_product_arity_vs_oracle(gpu, oracle_lib, dtype, A):
    """Arity study kernels (arity_workload.hpp:12-28; acceptance.cpp:334-370)
    against the oracle: every registered arity — including A = 8 (two cells
    per thread), A >= 16 (one cell per thread) — both policies, at a
    vectorised width (4096), odd widths (1023, 7: scalar tiled path), with a
    batch-broadcast (1,H) argument so one adjoint is a cross-row reduction,
    and inputs straddling reflect_below_half's 0.5 branch point."""
    rng = np.random.default_rng(1000 + A)
    rtol, atol = tol_for(dtype)
    name = f"tanh_product_{A}"
    for B, H in ((6, 4096), (37, 1023), (5, 7)):
        shapes = [(B, H)] * A
        if A > 1:
            shapes[A // 2] = (1, H)  # one batch-broadcast argument
        ins = [rng.uniform(-1, 1, s).astype(dtype) for s in shapes]
        seeds = [rng.uniform(-1, 1, (B, H)).astype(dtype)]
        want_p, want_d = oracle_lib.forward(name, ins)
        _, want_g, want_a64 = oracle_lib.mixed_step(name, ins, O.CACHE_FORWARD, seeds)
        terms = step_terms(oracle_lib, gpu, name, ins, seeds)
        for policy in (O.CACHE_FORWARD, O.RECOMPUTE_REVERSE):
            got_p, got_d, got_g = gpu.step(name, ins, seeds=seeds, policy=policy)
            tag = f"{name} {B}x{H} p{policy}"
            assert_close(got_p[0], want_p[0], rtol, atol, tag + " primal")
            if got_d is not None:
                for j in range(A):
                    assert_close(got_d[j], want_d[j], rtol, atol, tag + f" D{j}")
            assert_grads(got_g, want_g, want_a64, shapes, (B, H), dtype, tag, terms=terms)


def test_concurrent_may_raise_calls_keep_their_own_status():
    """Each may-raise call owns its device error word: two host
    threads on two streams, one failing forward (DivisionByZero at (1)) and
    one clean forward of the same kernel, repeated; every call reports its
    own status and index, never the other's."""
    import threading
    import torch
    from paper_1810_08297_b200 import native
    k = native.Kernel("div")
    n = 1 << 16
    a = torch.ones(n, dtype=torch.float64, device="cuda")
    b_bad = torch.ones(n, dtype=torch.float64, device="cuda")
    b_bad[1] = 0.0
    b_ok = torch.full((n,), 2.0, dtype=torch.float64, device="cuda")
    results = {"bad": [], "ok": []}

    def run(tag, b):
        s = torch.cuda.Stream()
        prim = [torch.empty(n, dtype=torch.float64, device="cuda")]
        parts = [torch.empty(n, dtype=torch.float64, device="cuda") for _ in range(2)]
        for _ in range(200):
            try:
                native.forward(k, [a, b], prim, parts, stream=s)
                results[tag].append("ok")
            except native.DivisionByZero as e:
                results[tag].append(str(e))

    ts = [threading.Thread(target=run, args=("bad", b_bad)), threading.Thread(target=run, args=("ok", b_ok))]
    for t in ts:
        t.start()
    for t in ts:
        t.join()
    assert results["ok"] == ["ok"] * 200
    assert len(results["bad"]) == 200 and all("at output index (1)" in r for r in results["bad"])


def test_may_raise_kernel_refuses_graph_capture():
    """A may-raise forward decodes its error word synchronously, which graph
    capture cannot do: it returns ConfigError instead of enqueuing."""
    import torch
    from paper_1810_08297_b200 import native
    k = native.Kernel("div")
    a = torch.ones(64, dtype=torch.float64, device="cuda")
    prim = [torch.empty(64, dtype=torch.float64, device="cuda")]
    parts = [torch.empty(64, dtype=torch.float64, device="cuda") for _ in range(2)]
    s = torch.cuda.Stream()
    g = torch.cuda.CUDAGraph()
    with pytest.raises(native.ConfigError, match="cannot be captured"):
        with torch.cuda.graph(g, stream=s):
            native.forward(k, [a, a], prim, parts, stream=s)


@pytest.mark.parametrize("variant,zj", [("canonical", (4, 5)), ("bias", (7, 8))])
def test_predicate_only_arguments_have_exactly_zero_partials(oracle_lib, variant, zj):
    """KHmlstm / KHmlstmBias declare z1, z2 predicate-only (kPredicateOnlyArgs):
    the RecomputeReverse pullback then skips their terms. Pins the declaration
    on the device: K1 stores exactly +0 for those partials (random inputs,
    every branch class), and both policies give exactly zero z adjoints with
    bit-identical other adjoints."""
    import torch
    from paper_1810_08297_b200 import native
    B, H = 256, 512
    ins = O.hmlstm_inputs(oracle_lib, B, H, np.float32, variant)
    name = O.hmlstm_kernel(variant)
    k = native.Kernel(name)
    dins = [torch.from_numpy(a).cuda() for a in ins]
    shapes = [a.shape for a in ins]
    prim = [torch.empty((B, H), device="cuda")]
    parts = [torch.empty((B, H), device="cuda") for _ in range(k.n_in)]
    native.forward(k, dins, prim, parts)
    for j in zj:
        d = parts[j].cpu().numpy()
        assert np.all(d == 0) and not np.any(np.signbit(d)), f"partial {j} not exactly +0"
    seed = [torch.rand((B, H), device="cuda") * 2 - 1]
    got = []
    for policy_parts in (parts, None):
        adj = [torch.full(s, 7.0, device="cuda") for s in shapes]
        native.pullback(k, shapes, seed, policy_parts, dins, adj, workspace=native.new_workspace(k, shapes, torch.float32))
        got.append([a.cpu().numpy() for a in adj])
    for j in range(k.n_in):
        assert np.array_equal(got[0][j], got[1][j]), f"adjoint {j} differs between policies"
    for j in zj:
        assert np.all(got[1][j] == 0)
