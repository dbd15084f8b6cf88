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


# Reduced adjoints (sums over broadcast axes): relative tolerance against the
# oracle's fp64-accumulated sum S of its rounded terms (Appendix A), no
# size-dependent absolute term.
RED_RTOL = {np.float32: 1e-6, np.float64: 1e-12}


def reduce_to(x, arg_shape):
    """Sum an output-shaped array down to an argument's shape under the
    reference's FIRST-axis broadcasting (shape.hpp:13-16): the argument's
    dims align with the output's leading axes; the rest, and every axis
    where the argument has extent 1, are summed (scatter_add,
    broadcast.hpp:210-217)."""
    x = np.asarray(x)
    r = len(arg_shape)
    x = x.sum(axis=tuple(range(r, x.ndim))) if x.ndim > r else x
    axes = tuple(k for k in range(r) if arg_shape[k] == 1 and x.shape[k] != 1)
    return x.sum(axis=axes, keepdims=True).reshape(arg_shape) if axes else x.reshape(arg_shape)


def term_slack(seeds, dev_partials, orc_partials, j, n_in, arg_shape, dtype):
    """sum over the reduced cells of |t_dev - t_orc|, t = fp-rounded w_i * D_ij
    (the terms backprop_diag hands to scatter_add, mixed.hpp:27-41): the
    most the device's sum can move because its partials differ from the
    oracle's by the ulps the elementwise comparator already admits (device
    libm vs glibc). Zero when the partials are bit-identical."""
    acc = 0.0
    for i, w in enumerate(seeds):
        if w is None:
            continue
        w = np.asarray(w, dtype)
        d = np.abs((w * np.asarray(dev_partials[i * n_in + j], dtype)).astype(np.float64) -
                   (w * np.asarray(orc_partials[i * n_in + j], dtype)).astype(np.float64))
        acc = acc + reduce_to(d, arg_shape)
    return acc


def abs_terms(seeds, orc_partials, j, n_in, arg_shape, dtype, out_shape):
    """(sum over the reduced cells of |t_orc|, number of terms per element)."""
    acc = 0.0
    for i, w in enumerate(seeds):
        if w is not None:
            t = (np.asarray(w, dtype) * np.asarray(orc_partials[i * n_in + j], dtype)).astype(np.float64)
            acc = acc + reduce_to(np.abs(t), arg_shape)
    n = sum(w is not None for w in seeds) * reduction_count(arg_shape, out_shape)
    return acc, n


def assert_reduced(got, want64, seed, dev_partial, orc_partial, what="", extra=0.0):
    """One reduced adjoint of a single-output node: |got - S| <= rtol*|S| +
    term_slack + extra, S = the oracle's fp64 sum."""
    dtype = np.asarray(got).dtype.type
    shape = np.asarray(want64).shape
    slack = term_slack([seed], [dev_partial], [orc_partial], 0, 1, shape, dtype)
    at = abs_terms([seed], [orc_partial], 0, 1, shape, dtype, np.shape(seed))
    _assert_reduced(got, want64, dtype, slack + extra, what, at)


def _assert_reduced(got, want64, dtype, slack, what, abs_terms=None):
    got64 = np.asarray(got, np.float64)
    want64 = np.asarray(want64, np.float64)
    bound = RED_RTOL[dtype] * np.abs(want64) + slack
    if abs_terms is not None and dtype == np.float64:
        # fp64 data: the device and the reference's serial scatter_add add
        # the same terms in different orders; recursive summation's forward
        # error bound n*eps*sum|t| (both sides) is part of the bound.
        bound = bound + abs_terms[1] * 2 * np.finfo(np.float64).eps * abs_terms[0]
    bad = np.abs(got64 - want64) > bound
    if bad.any():
        idx = np.argwhere(bad)[:5]
        rel = np.abs(got64 - want64) / np.maximum(np.abs(want64), 1e-300)
        raise AssertionError(f"{what}: {int(bad.sum())}/{bad.size} reduced elements outside rtol "
                             f"{RED_RTOL[dtype]} + term slack; worst rel {float(rel.max()):.3g}; first "
                             f"{idx.tolist()} got {got64[tuple(idx[0])]} want {want64[tuple(idx[0])]}")


def step_terms(orc, gpu, name, inputs, seeds=None):
    """(seeds, device partials, oracle partials) of one node for the
    reduced-adjoint comparator: the device's D_ij from a CacheForward K1
    through the C-ABI, the oracle's from its forward restatement."""
    _, orc_parts = orc.forward(name, inputs)
    _, dev_parts, _ = gpu.forward(name, inputs, want_primal=False)
    if seeds is None:
        out_shape = orc_parts[0].shape
        seeds = [np.ones(out_shape, inputs[0].dtype) for _ in range(len(orc_parts) // len(inputs))]
    return seeds, dev_parts, orc_parts


def assert_grads(got, want_serial, want_acc64, shapes, out_shape, dtype, what="", terms=None, chunks=1):
    """Full-shape adjoints: elementwise tolerance vs the reference arithmetic.
    Reduced adjoints: |got - S| <= rtol_red*|S| + sum|t_dev - t_orc| (+ the
    fp64 recursive-summation bound for fp64 data) with S the oracle's
    fp64-accumulated sum of its rounded terms; `terms` = step_terms(...).
    chunks > 1: the host step's row-chunk pipeline adds the chunks' rounded
    partial sums in chunk order; recursive summation of `chunks` partials
    adds at most chunks*eps*sum|t| (the bound grows with the chunk count,
    not with the batch)."""
    rtol, atol = tol_for(dtype)
    dtype = np.dtype(dtype).type
    n_in = len(shapes)
    for j, (g, ws, wa, s) in enumerate(zip(got, want_serial, want_acc64, shapes)):
        cnt = reduction_count(s, out_shape)
        if cnt == 1 and np.prod(s, dtype=np.int64) == np.prod(out_shape, dtype=np.int64):
            assert_close(g, ws, rtol, atol, f"{what} grad[{j}] (elementwise)")
            continue
        if terms is None:
            raise AssertionError(f"{what}: reduced adjoint {j} needs step_terms(...) for the comparator")
        seeds, dev_parts, orc_parts = terms
        slack = term_slack(seeds, dev_parts, orc_parts, j, n_in, tuple(s), dtype)
        at = abs_terms(seeds, orc_parts, j, n_in, tuple(s), dtype, out_shape)
        if chunks > 1:
            slack = slack + chunks * np.finfo(dtype).eps * at[0]
        _assert_reduced(np.asarray(g).reshape(s), np.asarray(wa).reshape(s), dtype, slack,
                        f"{what} grad[{j}] (reduced x{cnt})", at)


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
