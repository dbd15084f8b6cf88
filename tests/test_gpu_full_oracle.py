"""Every cell of every BASELINE config at FULL size against the CPU oracle
("full tensors for configs 1-4, and config 5 too").

The device runs the whole problem once through the C-ABI (K1 CacheForward,
K2 pullback with a U(-1,1) output seed; inputs from the reference's own Rng
stream). The oracle (oracle/liboracle.so, the pinned restatement) then
recomputes it in row blocks on the host's cores — rows are independent
under first-axis broadcasting (proj/include/bcad/shape.hpp:13-16) — and each
block is compared as it is produced, so host memory stays bounded:

* primal, all N partials, full-shape adjoints: elementwise Appendix A;
* branch decisions from D_c bit-exact against the z predicate
  (hmlstm.hpp:51-53); z adjoints exactly zero;
* (1,H) bias adjoints (config 3, 5): the oracle's fp64 sum S over ALL B rows
  of its rounded terms w*D (scatter_add, broadcast.hpp:210-217), block sums
  added in fp64, against the device's value with helpers._assert_reduced
  (1e-6 relative + the term slack sum|t_dev - t_orc|) — the device's own
  partials enter only through that slack, never as the reference sum.
"""
import concurrent.futures as cf
import os

import numpy as np
import pytest

import oracle as O
from helpers import _assert_reduced, assert_close, tol_for

pytestmark = pytest.mark.gpu

CELLS_PER_BLOCK = 1 << 22


@pytest.mark.parametrize("cfg", ["cfg2", "cfg3", "cfg4", "cfg4div", "cfg5"])
def test_full_size_every_cell_vs_oracle(oracle_lib, cfg):
    import torch
    from paper_1810_08297_b200 import native
    from paper_1810_08297_b200.workloads import WORKLOADS
    w = WORKLOADS[cfg]
    npdt = np.float32 if w.dtype == "f32" else np.float64
    dt = torch.float32 if w.dtype == "f32" else torch.float64
    B, H = w.B, w.H
    seed_val = oracle_lib.mix_seed(42, B * 1000003 + H)
    ins = oracle_lib.gen(seed_val, npdt, list(zip(w.shapes(), w.kinds())))
    seed = np.random.default_rng(17).random((B, H), dtype=np.float64 if npdt == np.float64 else np.float32)
    seed = (seed * 2 - 1).astype(npdt)

    k = native.Kernel(w.kernel)
    n = k.n_in
    shapes = [a.shape for a in ins]
    dins = [torch.from_numpy(a).to("cuda") for a in ins]
    dseed = torch.from_numpy(seed).to("cuda")
    prim = [torch.empty((B, H), device="cuda", dtype=dt)]
    parts = [torch.empty((B, H), device="cuda", dtype=dt) for _ in range(n)]
    native.forward(k, dins, prim, parts)
    adj = [torch.empty(s, device="cuda", dtype=dt) for s in shapes]
    native.pullback(k, shapes, [dseed], parts, dins, adj, workspace=native.new_workspace(k, shapes, dt))
    torch.cuda.synchronize()
    del dins, dseed

    rtol, atol = tol_for(npdt)
    batch = [s[0] == B and len(s) > 0 for s in shapes]
    reduced = [j for j, s in enumerate(shapes) if s == (1, H)]
    rows = max(1, CELLS_PER_BLOCK // H)
    blocks = [(r, min(B, r + rows)) for r in range(0, B, rows)]
    z1_idx, z2_idx = n - 2, n - 1
    div = w.variant == "divergence"

    def check_block(b0, b1):
        sub = [np.ascontiguousarray(a[b0:b1]) if bt else a for a, bt in zip(ins, batch)]
        wsub = np.ascontiguousarray(seed[b0:b1])
        want_p, want_d = oracle_lib.forward(w.kernel, sub)
        grads = [np.zeros(a.shape, npdt) for a in sub]
        acc64 = oracle_lib.pullback([a.shape for a in sub], [wsub], want_d, grads)
        got_p = prim[0][b0:b1].cpu().numpy()
        assert_close(got_p, want_p[0], rtol, atol, f"{cfg} rows {b0}:{b1} primal")
        got_d = [p[b0:b1].cpu().numpy() for p in parts]
        for j in range(n):
            assert_close(got_d[j], want_d[j], rtol, atol, f"{cfg} rows {b0}:{b1} D{j}")
        z1 = sub[z1_idx] if div else sub[z1_idx][:, None]
        z2 = sub[z2_idx] if div else sub[z2_idx][:, None]
        upd = (z1 == 0) & (z2 == 1)
        cpy = (z1 == 0) & (z2 == 0)
        dc = got_d[0]
        assert np.array_equal(dc == 1, np.broadcast_to(cpy, dc.shape)), f"{cfg} COPY class"
        assert np.array_equal(dc == 0, np.broadcast_to(~(upd | cpy), dc.shape)), f"{cfg} FLUSH class"
        assert np.array_equal(got_p[np.broadcast_to(cpy, dc.shape)], sub[0][np.broadcast_to(cpy, dc.shape)])
        for j in range(n):
            if batch[j] and shapes[j] == (B, H):
                assert_close(adj[j][b0:b1].cpu().numpy(), grads[j], rtol, atol, f"{cfg} rows {b0}:{b1} grad{j}")
            elif batch[j]:  # z: exact zeros
                assert not np.any(adj[j][b0:b1].cpu().numpy()), f"{cfg} z grad{j}"
        out = {}
        for j in reduced:  # block sums of the oracle's terms, slack, |terms|
            t_orc = (wsub * want_d[j]).astype(np.float64)
            t_dev = (wsub * got_d[j]).astype(np.float64)
            out[j] = (acc64[j].reshape(1, H), np.abs(t_dev - t_orc).sum(0, keepdims=True),
                      np.abs(t_orc).sum(0, keepdims=True))
        return out

    threads = min(16, os.cpu_count() or 4)
    with cf.ThreadPoolExecutor(threads) as ex:
        results = list(ex.map(lambda b: check_block(*b), blocks))
    for j in reduced:
        S = sum(r[j][0] for r in results)
        slack = sum(r[j][1] for r in results)
        abs_t = sum(r[j][2] for r in results)
        _assert_reduced(adj[j].cpu().numpy(), S, npdt, slack, f"{cfg} reduced grad{j} over {B} rows", (abs_t, B))
