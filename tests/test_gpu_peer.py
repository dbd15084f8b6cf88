"""Fused pullback allreduce over a peer-memory group (bcad_cu_peer_group_*,
bcad_cu_pullback_allreduce; kernels.cuh pull_finish_ar_kernel) — the
compute+collective form of SURVEY §8(e)'s batch-sharded step.

The test box has one B200, so the ranks share it: two ranks in ONE process
on two streams (their kernels run concurrently and exchange flags through
device memory), and two PROCESSES whose buffers are mapped by CUDA IPC (the
mechanism the multi-GPU run uses over NVLink). In both cases every rank must
end with bit-identical (1,H) bias adjoints equal to the oracle's fp64 sum
over the whole batch (1e-6 relative plus the term slack of
helpers.assert_reduced), its own batch rows' adjoints elementwise, and the
same bits on every repeated step (the flag / slot double buffering).

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


def _rank_state(torch, native, P, ins, seed, world, rank, stream):
    p = P.plan([a.shape for a in ins], world, rank)
    local = [np.ascontiguousarray(a) for a in P.local_views(p, ins)]
    lseed = np.ascontiguousarray(seed[p.rows[0]:p.rows[1]])
    k = native.Kernel(NAME)
    dins = [torch.from_numpy(a).cuda() for a in local]
    shapes = [a.shape for a in local]
    rows = shapes[0][0]
    H = shapes[0][1]
    prim = [torch.empty((rows, H), device="cuda", dtype=dins[0].dtype)]
    parts = [torch.empty((rows, H), device="cuda", dtype=dins[0].dtype) for _ in range(k.n_in)]
    with torch.cuda.stream(stream):
        native.forward(k, dins, prim, parts, stream=stream)
    adj = [torch.empty(s, device="cuda", dtype=dins[0].dtype) for s in shapes]
    ws = native.new_workspace(k, shapes, dins[0].dtype)
    return dict(p=p, k=k, dins=dins, shapes=shapes, parts=parts, adj=adj, ws=ws,
                seed=torch.from_numpy(lseed).cuda())


def _check(results, ins, seed, dtype, B, H, tag):
    orc = O.Oracle()
    want_p, want, want64 = orc.mixed_step(NAME, ins, seeds=[seed])
    _, opart = orc.forward(NAME, ins)
    rtol, atol = tol_for(dtype)
    for j in (0, 1, 2, 3, 7, 8):  # batch-sharded adjoints: elementwise
        got = np.concatenate([r["adj"][j] for r in results], axis=0)
        assert_close(got, want[j], rtol, atol, f"{tag} sharded grad[{j}]")
    eps = np.finfo(dtype).eps / 2
    for k, j in enumerate((4, 5, 6)):
        got = results[0]["adj"][j]
        for r in results[1:]:
            assert np.array_equal(got, r["adj"][j]), f"{tag}: ranks disagree on grad[{j}]"
        dev_terms = np.concatenate([r["terms"][k] for r in results], axis=0)
        # one fp32 rounding of the fp64 world sum
        assert_reduced(got, want64[j], seed, dev_terms, opart[j], f"{tag} grad[{j}]",
                       extra=eps * np.abs(got.astype(np.float64)))


@pytest.mark.parametrize("dtype,B,H,world", [(np.float32, 2048, 512, 2), (np.float64, 1022, 256, 2),
                                             (np.float32, 2050, 384, 4), (np.float32, 4096, 256, 8)])
def test_ranks_in_one_process_fused_allreduce(oracle_lib, dtype, B, H, world):
    """world ranks on world streams of one process (ragged row shards when B
    is not a multiple of world); 8 = the peer group's maximum."""
    import torch
    from paper_1810_08297_b200 import native
    from paper_1810_08297_b200 import partition as P
    ins = O.hmlstm_inputs(oracle_lib, B, H, dtype, "bias")
    seed = np.random.default_rng(11).uniform(-1, 1, (B, H)).astype(dtype)
    streams = [torch.cuda.Stream() for _ in range(world)]
    st = [_rank_state(torch, native, P, ins, seed, world, r, streams[r]) for r in range(world)]
    torch.cuda.synchronize()
    groups = [native.PeerGroup(r, world, 3 * H) for r in range(world)]
    for g in groups:
        g.connect([x.blob for x in groups])
    try:
        prev = None
        for step in range(3):  # both step parities and a wrap
            for r in range(world):  # both ranks' launches in flight at once
                s = st[r]
                native.pullback_allreduce(s["k"], s["shapes"], [s["seed"]], s["parts"], s["dins"], s["adj"], groups[r],
                                          workspace=s["ws"], stream=streams[r])
            torch.cuda.synchronize()
            res = [dict(adj=[a.cpu().numpy() for a in s["adj"]],
                        terms=[s["parts"][j].cpu().numpy() for j in (4, 5, 6)]) for s in st]
            _check(res, ins, seed, dtype, B, H, f"in-process step {step}")
            if prev is not None:
                for a, b in zip(prev, res):
                    for x, y in zip(a["adj"], b["adj"]):
                        assert np.array_equal(x, y), "repeated steps must be bit-identical"
            prev = res
    finally:
        for g in groups:
            g.close()


def _free_port():
    with socket.socket() as sk:
        sk.bind(("127.0.0.1", 0))
        return sk.getsockname()[1]


def _worker(rank, world, port, B, H, dtype, q):
    import torch
    import torch.distributed as dist
    from paper_1810_08297_b200 import native
    from paper_1810_08297_b200 import partition as P
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        torch.cuda.set_device(0)
        orc = O.Oracle()
        ins = O.hmlstm_inputs(orc, B, H, dtype, "bias")
        seed = np.random.default_rng(11).uniform(-1, 1, (B, H)).astype(dtype)
        stream = torch.cuda.Stream()
        s = _rank_state(torch, native, P, ins, seed, world, rank, stream)
        g = native.PeerGroup(rank, world, 3 * H)
        blobs = [None] * world
        dist.all_gather_object(blobs, g.blob)
        g.connect(blobs)  # the other process's buffer through CUDA IPC
        dist.barrier()
        outs = []
        for _ in range(2):
            native.pullback_allreduce(s["k"], s["shapes"], [s["seed"]], s["parts"], s["dins"], s["adj"], g,
                                      workspace=s["ws"], stream=stream)
            torch.cuda.synchronize()
            outs.append([a.cpu().numpy() for a in s["adj"]])
            dist.barrier()
        terms = [s["parts"][j].cpu().numpy() for j in (4, 5, 6)]
        dist.barrier()
        g.close()
        q.put((rank, outs, terms))
    except Exception as e:
        q.put((rank, repr(e), None))
        raise
    finally:
        dist.destroy_process_group()


def test_two_processes_ipc_fused_allreduce():
    import torch.multiprocessing as mp
    dtype, B, H, world = np.float32, 1024, 256, 2
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, B, H, dtype, q)) for r in range(world)]
    for pr in procs:
        pr.start()
    results = [q.get(timeout=600) for _ in range(world)]
    for pr in procs:
        pr.join(timeout=120)
    for r in results:
        assert r[2] is not None, f"rank {r[0]} failed: {r[1]}"
    assert all(pr.exitcode == 0 for pr in procs)
    results.sort(key=lambda r: r[0])
    orc = O.Oracle()
    ins = O.hmlstm_inputs(orc, B, H, dtype, "bias")
    seed = np.random.default_rng(11).uniform(-1, 1, (B, H)).astype(dtype)
    res = [dict(adj=r[1][-1], terms=r[2]) for r in results]
    _check(res, ins, seed, dtype, B, H, "2-process IPC")
    for r in results:
        for x, y in zip(r[1][0], r[1][1]):
            assert np.array_equal(x, y)


def test_bench_two_ranks_fused_allreduce_on_one_gpu():
    """The driver's N-rank bench path end to end with the fused allreduce:
    `bench.py --gpus 2 --allreduce fused` re-launches itself with two ranks,
    exchanges the peer handles over torch.distributed, captures the step
    (K1 -> K2 -> K2f-AR) as a CUDA graph and replays it. --share-device puts
    both ranks on the test box's one GPU (timings meaningless there); the
    line must be a valid contract line reporting 2 GPUs and the fused path."""
    import json
    import subprocess
    import sys
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    env = {k: v for k, v in os.environ.items() if k not in ("WORLD_SIZE", "RANK", "LOCAL_RANK")}
    r = subprocess.run([sys.executable, os.path.join(root, "bench.py"), "--gpus", "2", "--share-device",
                        "--allreduce", "fused", "--config", "cfg3", "--steps", "3", "--warmup", "3", "--extra", "none",
                        "--no-cpu-baseline", "--e2e-steps", "1"], capture_output=True, text=True, timeout=900,
                       cwd=root, env=env)
    assert r.returncode == 0, r.stdout[-3000:] + r.stderr[-3000:]
    lines = [l for l in r.stdout.splitlines() if l.strip().startswith("{")]
    assert len(lines) == 1, r.stdout
    d = json.loads(lines[0])
    assert d["n_gpus"] == 2 and d["value"] > 0 and d["gpu_launches"] > 0
    assert d["multi_gpu"]["world_size"] == 2 and d["multi_gpu"]["allreduce"].startswith("fused")
