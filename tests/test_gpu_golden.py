"""The CUDA path against the UNMODIFIED reference's own outputs.

Every fixture in tests/golden/ holds inputs, seeds and what the reference
computed for them (tests/golden/make_golden.py ran oracle/_ref, i.e.
/root/reference compiled from its sources): primal(s), the M*N cached
Jacobian diagonals (forward.hpp:98-150) and the leaf gradients of
Tape::backward (tape.hpp:185-211). The device step through the C-ABI must
reproduce them under SURVEY Appendix A:
  * primals, partials, full-shape gradients: |a-b| <= atol + rtol*max(|a|,|b|)
    (fp32 1e-5/1e-6, fp64 1e-12/1e-14);
  * reduced gradients: against the fp64 sum S of the reference's own rounded
    terms T(w_i * D_ij) over the broadcast axes: |got - S| <= rtol_red*|S| +
    sum|t_dev - t_ref| (rtol_red 1e-6 fp32 / 1e-12 fp64; the second term is
    what the per-cell ulp differences of the partials, already checked
    elementwise, can move the sum; zero where they are bit-identical). The
    device accumulates in fp64; the reference's serial fp32 sum is itself
    off by up to ~1e-4 relative at large B (reported, loose bound);
  * HM-LSTM branch decisions bit-exact (D_c in {0, 1, (0,1)} against the z
    predicate of hmlstm.hpp:51-53).
"""
import glob
import os

import numpy as np
import pytest

from helpers import GpuRunner, _assert_reduced, abs_terms, assert_close, reduce_to, term_slack, tol_for

pytestmark = pytest.mark.gpu

HERE = os.path.dirname(os.path.abspath(__file__))
FIXTURES = sorted(glob.glob(os.path.join(HERE, "golden", "*.npz")))


def load(path):
    d = np.load(path, allow_pickle=False)
    n, m = int(d["n_in"]), int(d["m_out"])
    ins = [d[f"in{j}"] for j in range(n)]
    seeds = [d[f"seed{i}"] if f"seed{i}" in d.files else None for i in range(m)]
    return str(d["kernel"]), ins, seeds, d, n, m


@pytest.fixture(scope="module")
def gpu():
    return GpuRunner("cuda")


def test_fixtures_present():
    assert len(FIXTURES) >= 30


@pytest.mark.parametrize("path", FIXTURES, ids=[os.path.basename(p)[:-4] for p in FIXTURES])
def test_device_matches_reference_outputs(gpu, path):
    kernel, ins, seeds, d, n, m = load(path)
    dtype = ins[0].dtype
    rtol, atol = tol_for(dtype)
    prim, parts, grads = gpu.step(kernel, ins, seeds=seeds)
    for i in range(m):
        assert_close(prim[i], d[f"primal{i}"], rtol, atol, f"{kernel} primal{i}")
    for k in range(m * n):
        assert_close(parts[k], d[f"partial{k}"], rtol, atol, f"{kernel} partial{k}")
    out_shape = d["primal0"].shape
    for j in range(n):
        want_serial = d[f"grad{j}"]
        cnt = int(np.prod(out_shape, dtype=np.int64)) // max(1, int(np.prod(ins[j].shape, dtype=np.int64)))
        if cnt == 1:
            assert_close(grads[j], want_serial, rtol, atol, f"{kernel} grad{j}")
            continue
        terms = np.zeros(out_shape, np.float64)
        for i in range(m):
            if seeds[i] is not None:  # the reference's rounded terms w_i * D_ij
                terms += (seeds[i] * d[f"partial{i * n + j}"]).astype(dtype).astype(np.float64)
        want64 = reduce_to(terms, ins[j].shape)
        ref_parts = [d[f"partial{k}"] for k in range(m * n)]
        slack = term_slack(seeds, parts, ref_parts, j, n, tuple(ins[j].shape), dtype.type)
        at = abs_terms(seeds, ref_parts, j, n, tuple(ins[j].shape), dtype.type, out_shape)
        _assert_reduced(grads[j], want64, dtype.type, slack, f"{kernel} grad{j} (reduced x{cnt})", at)
        # informational bound vs the reference's serial-fp32 sum itself
        assert_close(grads[j], want_serial, 1e-4 if dtype == np.float32 else 1e-10,
                     atol * cnt, f"{kernel} grad{j} vs serial reference")


@pytest.mark.parametrize("path", [p for p in FIXTURES if os.path.basename(p).startswith("hmlstm")],
                         ids=lambda p: os.path.basename(p)[:-4])
def test_hmlstm_branch_decisions_bit_exact(gpu, path):
    kernel, ins, seeds, d, n, m = load(path)
    _, parts, _ = gpu.step(kernel, ins, seeds=seeds)
    z1, z2 = ins[-2], ins[-1]
    out_shape = d["primal0"].shape
    z1b = np.broadcast_to(z1.reshape(z1.shape + (1,) * (len(out_shape) - z1.ndim)), out_shape)
    z2b = np.broadcast_to(z2.reshape(z2.shape + (1,) * (len(out_shape) - z2.ndim)), out_shape)
    update = (z1b == 0) & (z2b == 1)
    copy = (z1b == 0) & (z2b == 0)
    flush = ~(update | copy)
    dc = parts[0]
    assert np.array_equal(dc == 1, copy)
    assert np.array_equal(dc == 0, flush)
    assert np.array_equal((dc > 0) & (dc < 1), update)
    ref_dc = d["partial0"]  # the reference's own classes agree cell for cell
    assert np.array_equal(ref_dc == 1, copy) and np.array_equal(ref_dc == 0, flush)
