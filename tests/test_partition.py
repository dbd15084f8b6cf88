"""Batch partitioner and the multi-rank reduction, on CPU with gloo.

World size 2 (and 3, for ragged splits) processes each take their row block
of the bias-variant HM-LSTM step, compute their local mixed
step with the CPU oracle standing in for the device kernels, all-reduce the
batch-broadcast (1, H) adjoints (gloo here; NCCL via bcad_cu_allreduce_adjoints
on the GPUs), and must reproduce the single-process result: sharded adjoints
exactly, reduced ones within the fp64-accumulation comparator.
"""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

import oracle as O
from paper_1810_08297_b200 import partition as P


def test_shard_rows_cover_and_balance():
    for B in (1, 7, 64, 65536, 65537):
        for world in (1, 2, 3, 8):
            spans = [P.shard_rows(B, world, r) for r in range(world)]
            assert spans[0][0] == 0 and spans[-1][1] == B
            assert all(a[1] == b[0] for a, b in zip(spans, spans[1:]))
            sizes = [e - b for b, e in spans]
            assert max(sizes) - min(sizes) <= 1


def test_plan_classifies_batch_broadcast_args():
    shapes = [(64, 32)] * 4 + [(1, 32)] * 3 + [(64,)] * 2
    p = P.plan(shapes, 4, 1)
    assert p.rows == (16, 32)
    assert p.sharded == (True,) * 4 + (False,) * 3 + (True,) * 2
    assert p.allreduce == (4, 5, 6)
    assert p.local_shape((64, 32), 0) == (16, 32) and p.local_shape((1, 32), 4) == (1, 32)
    canonical = P.plan([(64, 32)] * 4 + [(64,)] * 2, 8, 0)
    assert canonical.allreduce == ()  # canonical kernel: independent shards, no collective
    with pytest.raises(ValueError):
        P.plan([(64, 32), (5, 32)], 2, 0)


def test_unsplittable_node_is_owned_by_rank0():
    """Output batch extent 1: nothing to split. Rank 0 computes the node, the
    other ranks are inactive and contribute zeros to the allreduce, so the
    summed adjoints equal the single-process ones (not world times them)."""
    shapes = [(1, 32), (1, 32), ()]
    plans = [P.plan(shapes, 3, r) for r in range(3)]
    assert [p.active for p in plans] == [True, False, False]
    assert plans[0].rows == (0, 1) and plans[1].rows == (0, 0)
    assert plans[0].allreduce == (0, 1, 2)
    assert all(p.active for p in (P.plan([(4, 2)], 3, r) for r in range(3)))


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _worker(rank, world, port, B, H, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        orc = O.Oracle()
        ins = O.hmlstm_inputs(orc, B, H, np.float32, "bias")
        rng = np.random.default_rng(7)
        seed = rng.uniform(-1, 1, (B, H)).astype(np.float32)
        p = P.plan([a.shape for a in ins], world, rank)
        local = [np.ascontiguousarray(a) for a in P.local_views(p, ins)]
        lseed = np.ascontiguousarray(seed[p.rows[0]:p.rows[1]])
        _, grads, acc64 = orc.mixed_step("hmlstm_update_bias", local, seeds=[lseed])
        # batch-broadcast adjoints: partial sums over local rows -> allreduce
        reduced = {}
        for j in p.allreduce:
            t = torch.from_numpy(acc64[j].astype(np.float64).copy())
            dist.all_reduce(t)
            reduced[j] = t.numpy()
        q.put((rank, p.rows, grads, reduced))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world,B", [(2, 64), (3, 61)])
def test_gloo_sharded_step_matches_single_process(world, B):
    H = 32
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, B, H, q)) for r in range(world)]
    for pr in procs:
        pr.start()
    results = [q.get(timeout=120) for _ in range(world)]
    for pr in procs:
        pr.join(timeout=60)
        assert pr.exitcode == 0
    results.sort(key=lambda r: r[0])

    orc = O.Oracle()
    ins = O.hmlstm_inputs(orc, B, H, np.float32, "bias")
    seed = np.random.default_rng(7).uniform(-1, 1, (B, H)).astype(np.float32)
    _, want, want64 = orc.mixed_step("hmlstm_update_bias", ins, seeds=[seed])
    p0 = P.plan([a.shape for a in ins], world, 0)
    for j in range(len(ins)):
        if p0.sharded[j]:
            got = np.concatenate([r[2][j] for r in results], axis=0)
            assert np.array_equal(got, want[j]), j  # rows are independent: exact
        else:
            for r in results:  # every rank holds the same all-reduced sum
                assert np.allclose(r[3][j].ravel(), want64[j].ravel(), rtol=1e-12, atol=1e-12)
