"""Batch-sharded mixed step on the DEVICE with 2 ranks.

Two processes share the test box's one B200 (NCCL refuses two ranks on one
device, so the cross-rank sum goes over gloo through host copies — the same
fp32 sum NCCL's allreduce performs over NVLink in bench.py). Each rank:
partition.plan -> its contiguous row block of c, f, i, g, z1, z2 and the
replicated (1,H) biases -> K1 + K2 through the C-ABI (native.forward /
native.pullback on cuda:0) -> allreduce of the three (1,H) bias adjoints.
The result must reproduce the oracle's single-process step on the full
batch: sharded adjoints elementwise (Appendix A), reduced adjoints against
the oracle's fp64-accumulated sum (helpers.assert_reduced) with the two
fp32 roundings of the partial sums and of their sum added to the bound.

Reference: rows are independent under first-axis broadcasting
(/root/reference/proj/include/bcad/shape.hpp:13-16); what is split is
scatter_add's sum over the batch axis (broadcast.hpp:210-217)."""
import os
import socket

import numpy as np
import pytest

import oracle as O
from helpers import assert_close, assert_reduced, tol_for

pytestmark = pytest.mark.gpu

NAME = "hmlstm_update_bias"


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _worker(rank, world, port, B, H, dtype, q):
    import torch
    import torch.distributed as dist
    from helpers import GpuRunner
    from paper_1810_08297_b200 import partition as P
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        torch.cuda.set_device(0)
        orc = O.Oracle()
        ins = O.hmlstm_inputs(orc, B, H, dtype, "bias")
        seed = np.random.default_rng(11).uniform(-1, 1, (B, H)).astype(dtype)
        p = P.plan([a.shape for a in ins], world, rank)
        local = [np.ascontiguousarray(a) for a in P.local_views(p, ins)]
        lseed = np.ascontiguousarray(seed[p.rows[0]:p.rows[1]])
        gpu = GpuRunner("cuda:0")
        prim, parts, grads = gpu.step(NAME, local, seeds=[lseed])
        partial_sums = {j: grads[j].copy() for j in p.allreduce}
        reduced = {}
        for j in p.allreduce:  # the allreduce of the batch-broadcast adjoints (fp32 sum, as NCCL)
            t = torch.from_numpy(grads[j].copy())
            dist.all_reduce(t)
            reduced[j] = t.numpy()
        q.put((rank, p.rows, prim[0], grads, partial_sums, reduced, [parts[j] for j in p.allreduce]))
    except Exception as e:  # surface the failure in the parent
        q.put((rank, repr(e)))
        raise
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("dtype,B,H", [(np.float32, 2048, 512), (np.float64, 1022, 256)])
def test_two_rank_device_step_matches_oracle(dtype, B, H):
    import torch.multiprocessing as mp
    world = 2
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, B, H, dtype, q)) for r in range(world)]
    for pr in procs:
        pr.start()
    results = [q.get(timeout=300) for _ in range(world)]
    for pr in procs:
        pr.join(timeout=120)
    for r in results:
        assert len(r) > 2, f"rank {r[0]} failed: {r[1]}"
    assert all(pr.exitcode == 0 for pr in procs)
    results.sort(key=lambda r: r[0])

    orc = O.Oracle()
    ins = O.hmlstm_inputs(orc, B, H, dtype, "bias")
    seed = np.random.default_rng(11).uniform(-1, 1, (B, H)).astype(dtype)
    want_p, want, want64 = orc.mixed_step(NAME, ins, seeds=[seed])
    _, opart = orc.forward(NAME, ins)
    rtol, atol = tol_for(dtype)
    assert results[0][1] == (0, B // 2) and results[1][1] == (B // 2, B)
    assert_close(np.concatenate([r[2] for r in results]), want_p[0], rtol, atol, "sharded primal")
    for j in (0, 1, 2, 3, 7, 8):  # batch-sharded adjoints: rows independent, elementwise
        got = np.concatenate([r[3][j] for r in results], axis=0)
        assert_close(got, want[j], rtol, atol, f"sharded grad[{j}]")
    for j in (7, 8):
        assert not np.any(np.concatenate([r[3][j] for r in results])), "z adjoints must be exactly 0"
    eps = np.finfo(dtype).eps / 2
    for k, j in enumerate((4, 5, 6)):
        got = results[0][5][j]
        assert np.array_equal(got, results[1][5][j]), "every rank holds the same allreduced sum"
        # device terms of both ranks (its own partials) against the oracle's terms
        dev_terms = np.concatenate([r[6][k] for r in results], axis=0)
        # the fp32/fp64 rounding of each rank's partial sum and of the cross-rank sum
        rounding = eps * (sum(np.abs(r[4][j].astype(np.float64)) for r in results) +
                          np.abs(got.astype(np.float64)))
        assert_reduced(got, want64[j], seed, dev_terms, opart[j], f"2-rank grad[{j}]", extra=rounding)
