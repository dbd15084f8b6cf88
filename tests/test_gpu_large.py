"""Full-size parity through size-independent properties (every BASELINE
config at its full size on one GPU: 2, 3, 4, 4-divergence, 5), plus oracle
checks on sampled rows. Rows are independent
for every full-shape and per-row quantity, so a row sample of the big
problem is checked exactly like a small problem; the (1,H) reductions over
all 65536 rows are checked against an fp64 sum of the device's own rounded
terms (a checksum of the K1 output) and run-to-run bit determinism."""
import numpy as np
import pytest

import oracle as O
from helpers import assert_close, tol_for

pytestmark = pytest.mark.gpu


def device_inputs(torch, B, H, dt, variant, seed):
    g = torch.Generator(device="cuda")
    g.manual_seed(seed)
    full = (B, H)
    shapes = [full] * 4 + ([(1, H)] * 3 if variant == "bias" else [])
    zs = full if variant == "divergence" else (B,)
    ins = [torch.rand(s, generator=g, device="cuda", dtype=dt) * 2 - 1 for s in shapes]
    ins += [(torch.rand(zs, generator=g, device="cuda", dtype=dt) < 0.5).to(dt) for _ in range(2)]
    return ins


@pytest.mark.parametrize("cfg", ["cfg2", "cfg3", "cfg4", "cfg4div", "cfg5"])
def test_full_size_properties(oracle_lib, cfg):
    import torch
    from paper_1810_08297_b200 import native
    from paper_1810_08297_b200.workloads import WORKLOADS
    w = WORKLOADS[cfg]
    dt = torch.float32 if w.dtype == "f32" else torch.float64
    npdt = np.float32 if w.dtype == "f32" else np.float64
    B, H = w.B, w.H
    ins = device_inputs(torch, B, H, dt, w.variant, 5)
    k = native.Kernel(w.kernel)
    n = k.n_in
    shapes = [tuple(t.shape) for t in ins]
    prim = [torch.empty((B, H), device="cuda", dtype=dt)]
    parts = [torch.empty((B, H), device="cuda", dtype=dt) for _ in range(n)]
    native.forward(k, ins, prim, parts)
    seed = torch.rand((B, H), device="cuda", dtype=dt) * 2 - 1
    adj = [torch.empty(s, device="cuda", dtype=dt) for s in shapes]
    ws = native.new_workspace(k, shapes, dt)
    native.pullback(k, shapes, [seed], parts, ins, adj, workspace=ws)
    adj2 = [torch.empty(s, device="cuda", dtype=dt) for s in shapes]
    native.pullback(k, shapes, [seed], None, ins, adj2, workspace=ws)  # RecomputeReverse, fused
    torch.cuda.synchronize()

    z1, z2 = ins[-2], ins[-1]
    if z1.dim() == 1:
        z1, z2 = z1[:, None].expand(B, H), z2[:, None].expand(B, H)
    upd = (z1 == 0) & (z2 == 1)
    cpy = (z1 == 0) & (z2 == 0)
    dc = parts[0]
    # branch decisions, bit-exact (Appendix A)
    assert torch.equal(dc == 1.0, cpy)
    assert torch.equal(dc == 0.0, ~(upd | cpy))
    assert bool(((dc > 0) & (dc < 1) == upd).all())
    # COPY primal == c bit-exact; boundary gradients exactly zero
    assert torch.equal(prim[0][cpy], ins[0][cpy])
    assert bool((adj[-1] == 0).all()) and bool((adj[-2] == 0).all())
    # policies bit-identical
    for a, b in zip(adj, adj2):
        assert torch.equal(a, b)
    # reductions: fp64 sum of the device's own rounded terms w*D
    for j, s in enumerate(shapes):
        if s == (1, H):
            terms = (seed * parts[j]).to(torch.float64)
            want = terms.sum(dim=0, keepdim=True)
            assert torch.allclose(adj[j].to(torch.float64), want, rtol=2e-6 if dt == torch.float32 else 1e-12,
                                  atol=1e-5 if dt == torch.float32 else 1e-11)
    # sampled rows against the oracle
    rows = torch.randperm(B, device="cuda")[:48].sort().values
    host = [t.cpu().numpy() for t in ins]
    sub = [h[rows.cpu().numpy()] if s[0] == B else h for h, s in zip(host, shapes)]
    want_p, want_d = oracle_lib.forward(w.kernel, sub)
    rtol, atol = tol_for(npdt)
    assert_close(prim[0][rows].cpu().numpy(), want_p[0], rtol, atol, "sampled primal")
    for j in range(n):
        assert_close(parts[j][rows].cpu().numpy(), want_d[j], rtol, atol, f"sampled D{j}")
    wsub = np.ascontiguousarray(seed[rows].cpu().numpy())
    _, want_g, _ = oracle_lib.mixed_step(w.kernel, sub, seeds=[wsub])
    for j, s in enumerate(shapes):
        if s == (B, H):
            assert_close(adj[j][rows].cpu().numpy(), want_g[j], rtol, atol, f"sampled grad{j}")
    # determinism run to run
    adj3 = [torch.empty(s, device="cuda", dtype=dt) for s in shapes]
    native.pullback(k, shapes, [seed], parts, ins, adj3, workspace=ws)
    torch.cuda.synchronize()
    for a, b in zip(adj, adj3):
        assert torch.equal(a, b)
