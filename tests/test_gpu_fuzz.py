"""Randomised parity of the tiled 2-D kernels against the oracle at sizes that
exercise their machinery: multi-tile ROW / COL / SCALAR reductions (the
finisher K2f), small-problem and large-problem tilings, odd widths (generic
rank-N fallback), accumulate flags, outputs without an adjoint, both
policies. Shapes follow the reference's first-axis broadcasting
(shape.hpp:13-16): each argument is full, length-1 on the batch axis (COL),
length-1 on the trailing axis / dropped (ROW) or a scalar."""
import numpy as np
import pytest

import oracle as O
from helpers import GpuRunner, assert_close, assert_grads, step_terms, tol_for

pytestmark = pytest.mark.gpu

KERNELS = ["mul", "plus", "gate", "sig_tanh", "square_gate", "blend", "fiveway", "prod_diff", "two", "fanout",
           "curl", "hmlstm_update_bias", "hmlstm_update"]


def arg_shape(rng, kind, rows, cols):
    if kind == "full":
        return (rows, cols)
    if kind == "col":
        return (1, cols)
    if kind == "row":
        return (rows,) if rng.integers(0, 2) else (rows, 1)
    return ()


@pytest.fixture(scope="module")
def gpu():
    return GpuRunner("cuda")


@pytest.mark.parametrize("dtype", [np.float32, np.float64])
def test_fuzz_tiled_kernels(gpu, oracle_lib, dtype):
    rng = np.random.default_rng(2024 if dtype == np.float32 else 2025)
    rtol, atol = tol_for(dtype)
    widths = [4, 8, 12, 64, 100, 128, 256, 1000, 1024, 2048, 4096, 6]
    for case in range(64):
        name = KERNELS[case % len(KERNELS)]
        n, m = oracle_lib.arity(name)
        cols = int(rng.choice(widths))
        rows = int(rng.integers(1, max(2, min(3000, 600_000 // cols))))
        if name.startswith("hmlstm"):
            kinds = ["full"] * 4 + (["col"] * 3 if n == 9 else []) + ["row", "row"]
        else:
            kinds = [str(rng.choice(["full", "full", "col", "row", "scalar"])) for _ in range(n)]
            kinds[int(rng.integers(0, n))] = "full"  # keep the output (rows, cols)
        shapes = [arg_shape(rng, k, rows, cols) for k in kinds]
        ins = [rng.uniform(-1, 1, s).astype(dtype) for s in shapes]
        if name.startswith("hmlstm"):
            for z in (n - 2, n - 1):
                ins[z] = (rng.uniform(0, 1, shapes[z]) < 0.5).astype(dtype)
        out_shape = O.broadcast_shape_py(shapes)
        seeds = [rng.uniform(-1, 1, out_shape).astype(dtype) for _ in range(m)]
        if m > 1 and case % 3 == 0:
            seeds[int(rng.integers(0, m))] = None
        existing = [rng.uniform(-1, 1, s).astype(dtype) if rng.integers(0, 4) == 0 else None for s in shapes]
        policy = int(rng.integers(0, 2))
        tag = f"case {case} {name} {shapes} p{policy}"
        got_p, got_d, got_g = gpu.step(name, ins, seeds=seeds, policy=policy, existing=existing)
        want_p, want_d = oracle_lib.forward(name, ins)
        _, want_g, want_a64 = oracle_lib.mixed_step(name, ins, O.CACHE_FORWARD, seeds)
        for i in range(m):
            assert_close(got_p[i], want_p[i], rtol, atol, tag + f" primal{i}")
        if got_d is not None:
            for k, (g, w) in enumerate(zip(got_d, want_d)):
                assert_close(g, w, rtol, atol, tag + f" D{k}")
        # accumulate: the device adds into the existing slot
        want_g = [w if e is None else (e.astype(np.float64) + w).astype(dtype) for w, e in zip(want_g, existing)]
        want_a64 = [w if e is None else e.astype(np.float64) + w for w, e in zip(want_a64, existing)]
        assert_grads(got_g, want_g, want_a64, shapes, out_shape, dtype, tag,
                     terms=step_terms(oracle_lib, gpu, name, ins, seeds))


@pytest.mark.parametrize("dtype", [np.float32, np.float64])
def test_fuzz_generic_rank3(gpu, oracle_lib, dtype):
    """Shapes with three irreducible axis groups run the generic rank-N
    kernels; arguments reduced over >= 32 output cells take the
    warp-per-element pullback. Both policies, accumulate flags."""
    rng = np.random.default_rng(77 if dtype == np.float32 else 78)
    rtol, atol = tol_for(dtype)
    kinds3 = [lambda B, T, C: (B, T, C), lambda B, T, C: (1, T, C), lambda B, T, C: (B, 1, C),
              lambda B, T, C: (B, T), lambda B, T, C: ()]
    for case in range(24):
        name = ["mul", "gate", "blend", "prod_diff", "two", "fiveway", "curl", "fanout"][case % 8]
        n, m = oracle_lib.arity(name)
        B, T, C = int(rng.integers(33, 200)), int(rng.integers(2, 40)), int(rng.integers(1, 9))
        picks = [0] + [int(rng.integers(0, len(kinds3))) for _ in range(n - 1)]
        rng.shuffle(picks)
        shapes = [kinds3[k](B, T, C) for k in picks]
        ins = [rng.uniform(-1, 1, s).astype(dtype) for s in shapes]
        out_shape = O.broadcast_shape_py(shapes)
        seeds = [rng.uniform(-1, 1, out_shape).astype(dtype) for _ in range(m)]
        existing = [rng.uniform(-1, 1, s).astype(dtype) if rng.integers(0, 4) == 0 else None for s in shapes]
        policy = int(rng.integers(0, 2))
        tag = f"rank3 case {case} {name} {shapes} p{policy}"
        got_p, got_d, got_g = gpu.step(name, ins, seeds=seeds, policy=policy, existing=existing)
        want_p, want_d = oracle_lib.forward(name, ins)
        _, want_g, want_a64 = oracle_lib.mixed_step(name, ins, O.CACHE_FORWARD, seeds)
        for i in range(m):
            assert_close(got_p[i], want_p[i], rtol, atol, tag + f" primal{i}")
        want_g = [w if e is None else (e.astype(np.float64) + w).astype(dtype) for w, e in zip(want_g, existing)]
        want_a64 = [w if e is None else e.astype(np.float64) + w for w, e in zip(want_a64, existing)]
        assert_grads(got_g, want_g, want_a64, shapes, out_shape, dtype, tag,
                     terms=step_terms(oracle_lib, gpu, name, ins, seeds))


@pytest.mark.parametrize("dtype", [np.float32, np.float64])
def test_fuzz_generic_segmented_reductions(gpu, oracle_lib, dtype):
    """Generic rank-N problems whose reduced arguments sum >= 4096 output
    cells per element (e.g. a (1, T, 1) argument of a (B, T, C) broadcast)
    take the segmented pullback: one CTA per (element, segment), fp64
    partials, a finisher in segment order; arguments full along the last axis
    and reduced over >= 64 cells ((1, 1, C), and (B, 1, C) when T >= 64) take
    its column form (a thread per element, the reduction cut into segments
    over the grid). Both policies, accumulate flags, against the oracle's fp64
    sums; and run to run bit-identical."""
    rng = np.random.default_rng(91 if dtype == np.float32 else 92)
    for case in range(8):
        name = ["mul", "gate", "two", "blend"][case % 4]
        n, m = oracle_lib.arity(name)
        B, T, C = int(rng.integers(64, 160)), int(rng.integers(3, 12) if case % 2 == 0 else rng.integers(64, 90)), int(rng.integers(64, 300))
        kinds = [(B, T, C), (1, T, 1), (B, 1, C), (1, 1, C)]
        shapes = [kinds[0]] + [kinds[int(rng.integers(1, len(kinds)))] for _ in range(n - 1)]
        if all(s != (1, T, 1) for s in shapes):
            shapes[-1] = (1, T, 1)
        ins = [rng.uniform(-1, 1, s).astype(dtype) for s in shapes]
        out_shape = O.broadcast_shape_py(shapes)
        seeds = [rng.uniform(-1, 1, out_shape).astype(dtype) for _ in range(m)]
        existing = [rng.uniform(-1, 1, s).astype(dtype) if rng.integers(0, 3) == 0 else None for s in shapes]
        policy = int(rng.integers(0, 2))
        tag = f"segmented case {case} {name} {shapes} p{policy}"
        got_p, _, got_g = gpu.step(name, ins, seeds=seeds, policy=policy, existing=existing)
        _, _, got_g2 = gpu.step(name, ins, seeds=seeds, policy=policy, existing=existing)
        for a, b in zip(got_g, got_g2):
            assert np.array_equal(a, b), tag + ": not run-to-run bit-identical"
        _, want_g, want_a64 = oracle_lib.mixed_step(name, ins, O.CACHE_FORWARD, seeds)
        want_g = [w if e is None else (e.astype(np.float64) + w).astype(dtype) for w, e in zip(want_g, existing)]
        want_a64 = [w if e is None else e.astype(np.float64) + w for w, e in zip(want_a64, existing)]
        assert_grads(got_g, want_g, want_a64, shapes, out_shape, dtype, tag,
                     terms=step_terms(oracle_lib, gpu, name, ins, seeds))


@pytest.mark.parametrize("dtype", [np.float32, np.float64])
def test_generic_vector_and_scalar_paths_agree(gpu, oracle_lib, dtype):
    """The generic rank-N kernels run 128-bit vectors of cells along the last
    axis when it is a multiple of the vector width and every buffer is 16-byte
    aligned (fwd_generic_vec_kernel, pull_generic_full_kernel), else one cell
    per thread. The same problem on aligned buffers and on buffers offset by
    one element (element-aligned only) must give bit-identical primals,
    partials and adjoints under both policies, equal to the oracle."""
    import torch
    from paper_1810_08297_b200 import native
    rng = np.random.default_rng(131)
    B, T, C = 24, 70, 16  # three irreducible axis groups; C a multiple of 4 and 2
    name = "gate"
    shapes = [(B, T, C), (B, 1, C)]
    ins = [rng.uniform(-1, 1, s).astype(dtype) for s in shapes]
    seed = rng.uniform(-1, 1, (B, T, C)).astype(dtype)
    k = native.Kernel(name)
    tdt = torch.float32 if dtype == np.float32 else torch.float64

    def buf(shape, offset, data=None):
        n = int(np.prod(shape))
        b = torch.empty(n + 4, dtype=tdt, device="cuda")[offset:offset + n].view(shape)
        if data is not None:
            b.copy_(torch.from_numpy(np.ascontiguousarray(data)).cuda())
        return b

    results = {}
    for offset in (0, 1):
        dins = [buf(s, offset, a) for s, a in zip(shapes, ins)]
        prim = [buf((B, T, C), offset)]
        parts = [buf((B, T, C), offset) for _ in range(k.n_in)]
        native.forward(k, dins, prim, parts)
        dseed = [buf((B, T, C), offset, seed)]
        for policy_parts in ("cache", "recompute"):
            adj = [buf(s, offset) for s in shapes]
            native.pullback(k, shapes, dseed, parts if policy_parts == "cache" else None, dins, adj,
                            workspace=native.new_workspace(k, shapes, tdt))
            torch.cuda.synchronize()
            results[(offset, policy_parts)] = [a.cpu().numpy() for a in adj]
        results[(offset, "fwd")] = [prim[0].cpu().numpy()] + [p.cpu().numpy() for p in parts]
    for key in ("fwd", "cache", "recompute"):
        for a, b in zip(results[(0, key)], results[(1, key)]):
            assert np.array_equal(a, b), f"{key}: vector and scalar paths differ"
    want_p, want_d = oracle_lib.forward(name, ins)
    rtol, atol = tol_for(dtype)
    assert_close(results[(0, "fwd")][0], want_p[0], rtol, atol, "generic primal")
    for j in range(k.n_in):
        assert_close(results[(0, "fwd")][1 + j], want_d[j], rtol, atol, f"generic D{j}")
    _, want_g, want_a64 = oracle_lib.mixed_step(name, ins, O.CACHE_FORWARD, [seed])
    for key in ("cache", "recompute"):
        assert_grads(results[(0, key)], want_g, want_a64, shapes, (B, T, C), dtype, f"generic {key}",
                     terms=step_terms(oracle_lib, gpu, name, ins, [seed]))
