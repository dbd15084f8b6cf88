"""Shared test helpers: run the CUDA path through the C-ABI on numpy inputs
and compare against the oracle with the SURVEY Appendix A comparator."""
from __future__ import annotations

import numpy as np

# Appendix A / reference's own close() (tests/support/test_util.hpp:11-14)
TOL = {np.float32: (1e-5, 1e-6), np.float64: (1e-12, 1e-14)}


def tol_for(dtype):
    return TOL[np.dtype(dtype).type]


def close_mask(a, b, rtol, atol):
    a = np.asarray(a, np.float64)
    b = np.asarray(b, np.float64)
    return np.abs(a - b) <= atol + rtol * np.maximum(np.abs(a), np.abs(b))


def assert_close(a, b, rtol, atol, what=""):
    m = close_mask(a, b, rtol, atol)
    if not m.all():
        idx = np.argwhere(~m)[:5]
        a64, b64 = np.asarray(a, np.float64), np.asarray(b, np.float64)
        worst = float(np.max(np.abs(a64 - b64)))
        raise AssertionError(f"{what}: {int((~m).sum())}/{m.size} cells out of tolerance "
                             f"(rtol={rtol}, atol={atol}); worst abs diff {worst}; first {idx.tolist()} "
                             f"got {a64[tuple(idx[0])]} want {b64[tuple(idx[0])]}")


def reduction_count(arg_shape, out_shape) -> int:
    return int(np.prod(out_shape, dtype=np.int64) // max(1, np.prod(arg_shape, dtype=np.int64)))


def assert_grads(got, want_serial, want_acc64, shapes, out_shape, dtype, what=""):
    """Full-shape adjoints: elementwise tolerance vs the reference arithmetic.
    Reduced adjoints: vs the fp64-accumulated sum of the same rounded terms."""
    rtol, atol = tol_for(dtype)
    for j, (g, ws, wa, s) in enumerate(zip(got, want_serial, want_acc64, shapes)):
        cnt = reduction_count(s, out_shape)
        if cnt == 1:
            assert_close(g, ws, rtol, atol, f"{what} grad[{j}] (elementwise)")
        else:
            assert_close(g, wa, rtol, atol * np.sqrt(cnt), f"{what} grad[{j}] (reduced x{cnt})")


class GpuRunner:
    """Drives libbcad_cu through native.py with torch device memory."""

    def __init__(self, device="cuda"):
        import torch
        from paper_1810_08297_b200 import native
        self.torch, self.native, self.device = torch, native, device

    def to_dev(self, a):
        return self.torch.from_numpy(np.ascontiguousarray(a)).to(self.device)

    def forward(self, name, inputs, want_primal=True, want_partials=True):
        torch, native = self.torch, self.native
        k = native.Kernel(name)
        dins = [self.to_dev(a) for a in inputs]
        out_shape = native.broadcast_shape([a.shape for a in inputs])
        dt = dins[0].dtype
        prim = [torch.empty(out_shape, dtype=dt, device=self.device) for _ in range(k.m_out)] if want_primal else None
        parts = ([torch.empty(out_shape, dtype=dt, device=self.device) for _ in range(k.m_out * k.n_in)]
                 if want_partials else None)
        native.forward(k, dins, prim, parts)
        torch.cuda.synchronize()
        return (None if prim is None else [p.cpu().numpy() for p in prim],
                None if parts is None else [p.cpu().numpy() for p in parts], (k, dins, prim, parts))

    def step(self, name, inputs, seeds=None, policy=0, existing=None):
        """One mixed step: forward then pullback. existing[j] (numpy or None)
        pre-fills adjoint slot j and sets accumulate. Returns numpy
        (primals, partials or None, grads)."""
        torch, native = self.torch, self.native
        k = native.Kernel(name)
        shapes = [a.shape for a in inputs]
        out_shape = native.broadcast_shape(shapes)
        dins = [self.to_dev(a) for a in inputs]
        dt = dins[0].dtype
        prim = [torch.empty(out_shape, dtype=dt, device=self.device) for _ in range(k.m_out)]
        parts = None
        if policy == 0:
            parts = [torch.empty(out_shape, dtype=dt, device=self.device) for _ in range(k.m_out * k.n_in)]
            native.forward(k, dins, prim, parts)
        else:
            native.forward(k, dins, prim, None)
        if seeds is None:
            seeds = [np.ones(out_shape, inputs[0].dtype) for _ in range(k.m_out)]
        dseeds = [None if s is None else self.to_dev(s) for s in seeds]
        existing = existing or [None] * k.n_in
        adj = [self.to_dev(e) if e is not None else torch.empty(s, dtype=dt, device=self.device)
               for e, s in zip(existing, shapes)]
        ws = native.new_workspace(k, shapes, dt)
        native.pullback(k, shapes, dseeds, parts, dins, adj, accumulate=[e is not None for e in existing],
                        workspace=ws)
        torch.cuda.synchronize()
        return ([p.cpu().numpy() for p in prim], None if parts is None else [p.cpu().numpy() for p in parts],
                [a.cpu().numpy() for a in adj])
