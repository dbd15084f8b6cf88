"""End-to-end host call (include/bcad_host.h -> C++ Tape + mixed_broadcast ->
libbcad_cu.so): host buffers in, host gradients out, against the oracle."""
import ctypes as C
import os

import numpy as np
import pytest

import oracle as O
from helpers import GpuRunner, assert_close, assert_grads, step_terms, tol_for

pytestmark = pytest.mark.gpu

PKG = os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "paper_1810_08297_b200")


@pytest.fixture(scope="module")
def host():
    from paper_1810_08297_b200 import native  # noqa: F401 (loads libbcad_cu.so first)
    lib = C.CDLL(os.path.join(PKG, "libbcad_host.so"))
    lib.bcad_host_last_error.restype = C.c_char_p
    return lib


def host_step(lib, name, ins, seeds, policy):
    from paper_1810_08297_b200 import native
    n = len(ins)
    try:
        out_shape = O.broadcast_shape_py([a.shape for a in ins])
    except O.OracleError:  # the library must report the mismatch itself
        out_shape = ins[0].shape
    m = len(seeds)
    prim = [np.empty(out_shape, ins[0].dtype) for _ in range(m)]
    grads = [np.empty(a.shape, a.dtype) for a in ins]
    ptr = lambda arrs: (C.c_void_p * len(arrs))(*[None if a is None else a.ctypes.data for a in arrs])  # noqa: E731
    shapes = (native.Shape * n)(*[native.Shape.of(a.shape) for a in ins])
    peak = C.c_int64()
    rc = lib.bcad_host_mixed_step(name.encode(), 0 if ins[0].dtype == np.float32 else 1, n, ptr(ins), shapes, m,
                                  policy, ptr(seeds), ptr(prim), ptr(grads), C.byref(peak), None)
    if rc:
        raise native._BY_CODE.get(rc, native.Error)(lib.bcad_host_last_error().decode())
    return prim, grads, peak.value


@pytest.mark.parametrize("dtype", [np.float32, np.float64])
@pytest.mark.parametrize("variant", ["canonical", "bias"])
@pytest.mark.parametrize("policy", [0, 1])
def test_host_step_matches_oracle(host, oracle_lib, dtype, variant, policy):
    B, H = 32, 256
    ins = O.hmlstm_inputs(oracle_lib, B, H, dtype, variant)
    name = O.hmlstm_kernel(variant)
    seeds = [np.random.default_rng(1).uniform(-1, 1, (B, H)).astype(dtype)]
    want_p, want_g, want_a64 = oracle_lib.mixed_step(name, ins, policy, seeds)
    got_p, got_g, peak = host_step(host, name, ins, seeds, policy)
    rtol, atol = tol_for(dtype)
    assert_close(got_p[0], want_p[0], rtol, atol, "host primal")
    assert_grads(got_g, want_g, want_a64, [a.shape for a in ins], (B, H), dtype, "host e2e",
                 terms=step_terms(oracle_lib, GpuRunner(), name, ins, seeds))
    s = np.dtype(dtype).itemsize
    E, n = B * H, len(ins)
    inputs_bytes = sum(a.size for a in ins) * s
    assert peak == inputs_bytes + E * s + (n * E * s if policy == 0 else 0)  # tape.hpp:236-243


def test_host_step_maps_errors(host):
    from paper_1810_08297_b200 import native
    with pytest.raises(native.DomainError) as e:
        host_step(host, "log", [np.array([[1.0, -2.0]])], [np.ones((1, 2))], 0)
    assert "at output index (0, 1)" in str(e.value)
    with pytest.raises(native.ShapeMismatch):
        host_step(host, "mul", [np.ones((2, 3)), np.ones((4, 3))], [np.ones((2, 3))], 0)
    with pytest.raises(native.UnknownPrimitive):
        host_step(host, "nope", [np.ones(2)], [np.ones(2)], 0)


@pytest.mark.parametrize("dtype", [np.float32, np.float64])
def test_cell_gradients_three_impls(oracle_lib, dtype):
    """cell_gradients through the C++ tape for mixed-cache, mixed-recompute and
    reverse-unfused (hmlstm.hpp:123-142) agree with the oracle; the tape sizes
    are 7 vs 14 nodes (test_bench.cpp:73-90)."""
    import torch
    from paper_1810_08297_b200 import host
    n = 64
    ins = O.hmlstm_inputs(oracle_lib, n, n, dtype, "canonical")
    seed = np.random.default_rng(3).uniform(-1, 1, (n, n)).astype(dtype)
    _, want, want64 = oracle_lib.mixed_step("hmlstm_update", ins, seeds=[seed])
    dins = [torch.from_numpy(a).cuda() for a in ins]
    dseed = torch.from_numpy(seed).cuda()
    rtol, atol = tol_for(dtype)
    got = {}
    for impl in ("mixed-cache", "mixed-recompute", "reverse-unfused"):
        grads = [torch.empty((n, n), dtype=dins[0].dtype, device="cuda") for _ in range(4)]
        nodes, peak = host.cell_gradients(impl, dins, dseed, grads)
        torch.cuda.synchronize()
        assert nodes == (14 if impl == "reverse-unfused" else 7)
        got[impl] = [g.cpu().numpy() for g in grads]
        for k in range(4):
            assert_close(got[impl][k], want[k], rtol, atol, f"{impl} grad{k}")
    for a, b in zip(got["mixed-cache"], got["mixed-recompute"]):
        assert np.array_equal(a, b)


@pytest.mark.parametrize("dtype", [np.float32, np.float64])
@pytest.mark.parametrize("variant", ["canonical", "bias"])
@pytest.mark.parametrize("chunks", [2, 3, 7])
def test_host_step_pipelined_matches_one_shot(host, oracle_lib, dtype, variant, chunks):
    """Row-chunk pipelining (bcad_host_set_pipeline) is a schedule only: the
    batch-sharded gradients and the primal are bit-identical to the one-shot
    tape, the (1,H) bias gradients (summed over chunks) match the oracle, and
    peak_cached_bytes reports the one-shot tape's accounting."""
    from paper_1810_08297_b200 import host as H
    B, Hd = 50, 96  # 50 rows: ragged chunks
    ins = O.hmlstm_inputs(oracle_lib, B, Hd, dtype, variant)
    name = O.hmlstm_kernel(variant)
    seeds = [np.random.default_rng(2).uniform(-1, 1, (B, Hd)).astype(dtype)]
    try:
        H.set_pipeline(1)
        p1, g1, peak1 = host_step(host, name, ins, seeds, 0)
        H.set_pipeline(chunks)
        pk, gk, peakk = host_step(host, name, ins, seeds, 0)
    finally:
        H.set_pipeline(0)
    assert np.array_equal(p1[0], pk[0])
    assert peak1 == peakk
    _, want_g, want_a64 = oracle_lib.mixed_step(name, ins, 0, seeds)
    assert_grads(gk, want_g, want_a64, [a.shape for a in ins], (B, Hd), dtype, f"pipelined x{chunks}",
                 terms=step_terms(oracle_lib, GpuRunner(), name, ins, seeds), chunks=chunks)
    for j, a in enumerate(ins):
        if a.shape[0] == B:
            assert np.array_equal(g1[j], gk[j]), f"arg {j} differs between one-shot and pipelined"


def test_host_set_pipeline_rejects_negative(host):
    from paper_1810_08297_b200 import host as H
    from paper_1810_08297_b200 import native
    with pytest.raises(native.ConfigError):
        H.set_pipeline(-1)


@pytest.mark.parametrize("dtype", [np.float32, np.float64])
def test_host_step_pipelined_scalar_and_two_outputs(host, oracle_lib, dtype):
    """Pipelining with a scalar (batch-broadcast) argument, a (B, 1)-shaped
    argument and a two-output kernel (prod_diff: a*b, a-b): the scalar's
    gradient is summed over chunks, both seeds are chunked."""
    from paper_1810_08297_b200 import host as H
    rng = np.random.default_rng(7)
    B, W = 37, 48
    for shapes in ([(B, W), ()], [(B, W), (B, 1)], [(B, 1), (1, W)]):
        ins = [rng.uniform(-1, 1, s).astype(dtype) for s in shapes]
        out_shape = O.broadcast_shape_py(shapes)
        seeds = [rng.uniform(-1, 1, out_shape).astype(dtype) for _ in range(2)]
        try:
            H.set_pipeline(1)
            p1, g1, peak1 = host_step(host, "prod_diff", ins, seeds, 0)
            H.set_pipeline(5)
            pk, gk, peakk = host_step(host, "prod_diff", ins, seeds, 0)
        finally:
            H.set_pipeline(0)
        for a, b in zip(p1, pk):
            assert np.array_equal(a, b)
        assert peak1 == peakk
        _, want_g, want_a64 = oracle_lib.mixed_step("prod_diff", ins, 0, seeds)
        assert_grads(gk, want_g, want_a64, shapes, out_shape, dtype, f"pipelined prod_diff {shapes}",
                     terms=step_terms(oracle_lib, GpuRunner(), "prod_diff", ins, seeds), chunks=5)


def test_prepared_step_replay_rereads_buffers(oracle_lib):
    """Prepared pipelined steps (bcad_host_set_prepared) on pinned buffers:
    a call on kept device buffers equals the unprepared step bit for bit, and
    a call after the host inputs changed in place uses the new contents."""
    import torch
    from paper_1810_08297_b200 import host as H
    B, Hd = 512, 256
    name = O.hmlstm_kernel("bias")
    ins0 = O.hmlstm_inputs(oracle_lib, B, Hd, np.float32, "bias")
    ins1 = [np.ascontiguousarray(np.flip(a, axis=-1)) for a in ins0]  # other data, same shapes
    keep = [torch.from_numpy(np.ascontiguousarray(a)).pin_memory() for a in ins0]
    host_in = [t.numpy() for t in keep]
    seed_t = torch.from_numpy(np.random.default_rng(4).uniform(-1, 1, (B, Hd)).astype(np.float32)).pin_memory()
    grads_t = [torch.empty(a.shape, dtype=torch.float32).pin_memory() for a in ins0]
    grads = [t.numpy() for t in grads_t]
    stream = torch.cuda.Stream()
    try:
        H.set_pipeline(4)
        H.set_prepared(True)
        call = H.HostStep(name, host_in, [seed_t.numpy()], grads_out=grads, stream=int(stream.cuda_stream))
        results = []
        for data in (ins0, ins0, ins1, ins1):
            for dst, src in zip(host_in, data):
                dst[...] = src
            call()
            results.append([g.copy() for g in grads])
        H.set_prepared(False)
        for data, got in ((ins0, results[1]), (ins1, results[3])):
            for dst, src in zip(host_in, data):
                dst[...] = src
            call()
            for a, b in zip(grads, got):
                assert np.array_equal(a, b)  # prepared == unprepared pipelined step, bit for bit
        _, want_g, want_a64 = oracle_lib.mixed_step(name, ins1, 0, [seed_t.numpy()])
        assert_grads(results[3], want_g, want_a64, [a.shape for a in ins1], (B, Hd), np.float32, "prepared step",
                     terms=step_terms(oracle_lib, GpuRunner(), name, ins1, [seed_t.numpy()]), chunks=4)
        for a, b in zip(results[0], results[1]):
            assert np.array_equal(a, b)
        assert not all(np.array_equal(a, b) for a, b in zip(results[1], results[2]))
    finally:
        H.set_prepared(True)
        H.set_pipeline(0)


@pytest.mark.parametrize("variant", ["canonical", "bias"])
def test_async_host_steps_overlap_and_match(oracle_lib, variant):
    """bcad_host_mixed_step_async: a stream of steps alternating between two
    host gradient buffer sets (the overlap the e2e bench times) gives every
    step the same bits as the synchronous call — including the bias
    variant's (1,H) gradients, accumulated over chunks and downloaded after
    the last one — and steps on the same buffers stay ordered."""
    import torch
    from paper_1810_08297_b200 import host as H
    B, Hd = 2048, 1024
    ins = O.hmlstm_inputs(oracle_lib, B, Hd, np.float32, variant)
    pin = lambda a: torch.from_numpy(np.ascontiguousarray(a)).pin_memory().numpy()  # noqa: E731
    hin = [pin(a) for a in ins]
    seed = pin(np.random.default_rng(3).uniform(-1, 1, (B, Hd)).astype(np.float32))
    name = O.hmlstm_kernel(variant)
    stream = torch.cuda.Stream()
    sp = int(stream.cuda_stream)
    ref = [pin(np.zeros(a.shape, np.float32)) for a in ins]
    # the synchronous reference at the async path's chunk count (2): the
    # (1,H) gradients are summed per chunk, so their last bits follow the count
    H.set_pipeline(2)
    try:
        H.HostStep(name, hin, [seed], grads_out=ref, stream=sp)()
    finally:
        H.set_pipeline(0)
    sets = [[pin(np.full(a.shape, np.nan, np.float32)) for a in ins] for _ in range(2)]
    calls = [H.HostStep(name, hin, [seed], grads_out=g, stream=sp) for g in sets]
    for k in range(7):
        calls[k % 2].enqueue()
    H.synchronize(sp)
    for g in sets:
        for j, (x, y) in enumerate(zip(g, ref)):
            assert np.array_equal(x, y), f"grad[{j}] differs from the synchronous step"
