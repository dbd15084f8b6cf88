#!/usr/bin/env python3
"""Benchmark of the north-star path: HM-LSTM cell-update mixed-mode gradient
(fused dual-number forward K1 + adjoint-reduction pullback K2, plus the NCCL
allreduce of batch-broadcast adjoints when sharded), BASELINE.json metric
"HM-LSTM cell-update grad elements/s & ms/step at 1/2/4/8 B200; % HBM roofline".

  python bench.py [--gpus N] [--steps K] [--warmup W] [--config cfgX] [--impl native|reference]
  python -m torch.distributed.run --nproc-per-node N --master-addr 127.0.0.1 bench.py --gpus N

--gpus N > 1 without a torchrun environment re-launches itself under
torch.distributed.run with N ranks (one per GPU); under torchrun WORLD_SIZE
must equal --gpus. Default workload: config 2 (1024x1024 fp32, BASELINE's
"on 1 B200" config) at N = 1; config 5 (65536x4096 fp32 bias variant,
batch-sharded, strong scaling) at N > 1, the 3 (1,H) adjoints allreduced
inside the pullback's finisher over NVLink peer memory (--allreduce fused,
default; --allreduce nccl for ncclAllReduce after the pullback). --dry-run runs the N-rank plumbing on CPU over gloo (no GPU work).

One step = one pass of the hot path over one batch: bcad_cu_forward (primal +
M*N partials) then bcad_cu_pullback (all input adjoints) — what the
reference's run_cell_once("mixed-cache") times (proj/src/bench.cpp:112-128).
`value` = grad elements (output cells) per second over all ranks, inputs
resident in HBM, L2 flushed between steps (a 1 GiB write then a 1 GiB read,
so the flush's own dirty lines are written back before the step; outside the timed
events). `e2e` = the same step through the C-ABI with HOST buffers: pinned
H2D of the step's inputs and seed, forward, pullback, D2H of the gradients.

--impl reference times the reference's own CPU implementation (the
unmodified /root/reference code compiled into oracle/_ref) on the host cores.
"""
from __future__ import annotations

import argparse
import json
import math
import os
import statistics
import subprocess
import sys
import tempfile
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

from paper_1810_08297_b200.partition import plan as shard_plan  # noqa: E402
from paper_1810_08297_b200.workloads import WORKLOADS, Workload  # noqa: E402

PEAKS_PATH = os.path.join(ROOT, "MEASURED_PEAKS.json")
FALLBACK_HBM_GBS = 6650.0  # /opt/skills/guides/B200_PROFILING.md fallback
NCU_SUMMARY = os.path.join(ROOT, "profiles", "ncu_traffic.json")


def hbm_peak():
    try:
        with open(PEAKS_PATH) as f:
            return float(json.load(f)["hbm_gbs"]), "measured (MEASURED_PEAKS.json hbm_gbs)"
    except Exception:
        return FALLBACK_HBM_GBS, "fallback (B200_PROFILING.md)"


# ----------------------------------------------------------------- clocks
class ClockSampler:
    """nvidia-smi clocks + throttle reasons sampled during the timed region
    (B200_PROFILING.md 'clocks' line)."""

    Q = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
         "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
         "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, gpu_index: int):
        self.idx = gpu_index
        self.proc = None
        self.path = None

    def start(self):
        try:
            fd, self.path = tempfile.mkstemp(suffix=".csv")
            os.close(fd)
            self.proc = subprocess.Popen(["nvidia-smi", "-i", str(self.idx), f"--query-gpu={self.Q}",
                                          "--format=csv,noheader,nounits", "-lms", "100"],
                                         stdout=open(self.path, "w"), stderr=subprocess.DEVNULL)
        except Exception:
            self.proc = None
        time.sleep(0.25)

    def stop(self):
        if not self.proc:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        time.sleep(0.25)
        self.proc.terminate()
        try:
            self.proc.wait(timeout=5)
        except Exception:
            self.proc.kill()
        sm, mx, reasons = [], None, set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        with open(self.path) as f:
            for line in f:
                parts = [p.strip() for p in line.split(",")]
                if len(parts) < 9:
                    continue
                try:
                    sm.append(float(parts[1]))
                    mx = float(parts[2])
                except ValueError:
                    continue
                for nm, v in zip(names, parts[5:9]):
                    if v.lower() == "active":
                        reasons.add(nm)
        os.unlink(self.path)
        busy = [s for s in sm if mx and s > 0.5 * mx] or sm
        return {"sm_mhz": statistics.median(busy) if busy else None, "sm_max_mhz": mx,
                "reasons": sorted(reasons), "samples": len(sm)}


# ------------------------------------------------- shared by both arms
DATA = ("synthetic: bcad Rng (mt19937_64) inputs in the reference's order, mix_seed(42, B*1000003+H) "
        "(proj/src/bench.cpp:31-37; U(-1,1) gates, exact-binary z with p=1/2), output seed of ones")


def input_seed(w: Workload) -> int:
    from paper_1810_08297_b200 import host
    return host.mix_seed(42, w.B * 1000003 + w.H)


def bench_config(w: Workload, world: int, policy: int) -> dict:
    """`config` of the JSON line, identical for the GPU arm and the
    reference arm so the driver can compare them."""
    return {"workload": w.describe, "B": w.B, "H": w.H, "variant": w.variant, "dtype": w.dtype,
            "policy": "CacheForward" if policy == 0 else "RecomputeReverse",
            "parallelism": (f"batch rows sharded over {world} ranks, allreduce of batch-broadcast adjoints"
                            if world > 1 else "single GPU"),
            "l2": l2_description(w, world, policy)}


# B200 L2 (126 MB); steps whose bytes are below 4 x this rotate buffer sets.
L2_BYTES = 126 * 2**20


def rotation_sets(step_bytes: int) -> int:
    """Independent batch buffer sets the timed steps cycle through so that
    no step starts with its operands in L2: each set is revisited only after
    >= 2 x L2 of other steps' traffic (R = 1 when one step moves > 4 x L2)."""
    if step_bytes >= 4 * L2_BYTES:
        return 1
    return max(3, math.ceil(2 * L2_BYTES / step_bytes) + 1)


def l2_description(w: Workload, world: int, policy: int) -> str:
    B_local = w.B if scaling_of(w) == "weak" or world == 1 else -(-w.B // world)
    R = rotation_sets(w.step_bytes(B_local, policy))
    if R == 1:
        return ("inputs larger than L2: one step moves > 4 x the 126 MB L2; the K steps run back to back as one "
                "CUDA graph, no flush")
    return (f"inputs larger than L2: {R} independent batch buffer sets, step k on set k % {R} (each set revisited "
            f"after >= 2 x the 126 MB L2 of other steps' traffic); the K steps run back to back as one CUDA graph, "
            f"no flush")


def scaling_of(w: Workload) -> str:
    return "strong" if w.key == "cfg5" else "weak"


# -------------------------------------------------------------- reference
def cpu_model() -> str:
    try:
        for line in open("/proc/cpuinfo"):
            if line.startswith("model name"):
                return line.split(":", 1)[1].strip()
    except OSError:
        pass
    return "unknown"


def reference_split(ref, w: Workload, ins, rows: int, reps: int, threads: int = 0) -> dict:
    """the reference step's forward (tape inputs + mixed_broadcast)
    and backward (Tape::backward + gradient copies) medians, scaled to the
    full batch like ms_per_step."""
    f, b = ref.time_mixed_split(w.kernel, ins, threads=threads, reps=reps)
    scale = w.B / rows
    return {"forward_ms": statistics.median(f) / 1e6 * scale, "backward_ms": statistics.median(b) / 1e6 * scale}


def cpu_reference_rate(w: Workload, budget_s: float, min_reps: int = 1, threads: int = 0):
    """Time the unmodified reference (oracle/_ref) on host cores: Tape +
    mixed_broadcast(CacheForward) + backward(ones), bench.cpp:112-128.
    Bounded sample: full rows up to a row cap sized to the budget."""
    import numpy as np
    import oracle as O
    ref = O.Reference() if O.reference_available() else None
    kind = "reference" if ref else "port"
    lib = ref or O.Oracle()
    # cells the reference processes per second is ~5e6 on 8 cores; cap rows
    # so one rep stays well inside the budget.
    rows = w.B
    while rows > 1 and rows * w.H > 4e6 * max(1.0, budget_s / 4):
        rows //= 2
    sample = Workload(w.key, rows, w.H, w.dtype, w.variant, w.describe)
    dtype = np.float32 if w.dtype == "f32" else np.float64
    s = O.Oracle().mix_seed(42, w.B * 1000003 + w.H)
    ins = lib.gen(s, dtype, list(zip(sample.shapes(), sample.kinds())))
    ns = []
    t_end = time.time() + budget_s
    if ref:
        ref.time_mixed(w.kernel, ins, threads=threads, warmup=1, reps=1)
        while len(ns) < min_reps or time.time() < t_end:
            ns += ref.time_mixed(w.kernel, ins, threads=threads, warmup=0, reps=1)
        cores = ref.max_threads() if threads == 0 else threads
    else:
        while len(ns) < min_reps or time.time() < t_end:
            t0 = time.perf_counter_ns()
            lib.mixed_step(w.kernel, ins)
            ns.append(time.perf_counter_ns() - t0)
        cores = 1
    med = statistics.median(ns)
    cells = rows * w.H
    out = {"value": cells / (med * 1e-9), "unit": "grad elements/s", "cores": cores, "kind": kind,
           "sample": f"{rows}x{w.H} rows of {w.B}x{w.H} {w.dtype} {w.variant}, {len(ns)} reps, median "
                     f"{med / 1e6:.2f} ms/rep",
           "ms_per_rep": med / 1e6, "reps": len(ns), "cpu_model": cpu_model(), "omp_threads": cores}
    if ref:
        out["split"] = reference_split(ref, w, ins, rows, 3, threads)
    return out


def run_reference_arm(args, w: Workload, rank: int, world: int):
    if rank != 0:
        return
    import numpy as np  # noqa: F401
    import oracle as O
    ref = O.Reference() if O.reference_available() else None
    kind = "reference" if ref else "port"
    lib = ref or O.Oracle()
    rows = w.B
    while rows > 1 and rows * w.H > 2.1e6:  # a bounded sample per step (~0.2-0.5 s on 8 cores)
        rows //= 2
    sample = Workload(w.key, rows, w.H, w.dtype, w.variant, w.describe)
    dtype = np.float32 if w.dtype == "f32" else np.float64
    s = O.Oracle().mix_seed(42, w.B * 1000003 + w.H)
    ins = lib.gen(s, dtype, list(zip(sample.shapes(), sample.kinds())))
    if ref:
        ref.time_mixed(w.kernel, ins, warmup=args.warmup, reps=1)
        ns = ref.time_mixed(w.kernel, ins, warmup=0, reps=args.steps)
        cores = ref.max_threads()
    else:
        for _ in range(args.warmup):
            lib.mixed_step(w.kernel, ins)
        ns = []
        for _ in range(args.steps):
            t0 = time.perf_counter_ns()
            lib.mixed_step(w.kernel, ins)
            ns.append(time.perf_counter_ns() - t0)
        cores = 1
    total_s = sum(ns) * 1e-9
    cells = rows * w.H * len(ns)
    val = cells / total_s
    line = {"impl": "reference", "metric": "HM-LSTM cell-update grad elements/s", "value": val,
            "unit": "grad elements/s", "n_gpus": world, "steps": args.steps, "warmup": args.warmup,
            "ms_per_step": total_s * 1e3 / len(ns) * (w.B / rows), "higher_is_better": True,
            "scaling": scaling_of(w), "vs_baseline": None, "dtype": w.dtype, "data": DATA,
            "config": bench_config(w, world, 0),
            "cpu_baseline": {"value": val, "unit": "grad elements/s", "cores": cores, "kind": kind,
                             "sample": f"{rows}x{w.H} of {w.B}x{w.H} per step (rows are independent)",
                             "cpu_model": cpu_model(), "omp_threads": cores,
                             "nproc": os.cpu_count()},
            "e2e": {"value": val, "unit": "grad elements/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    if ref:
        line["breakdown_ms"] = reference_split(ref, w, ins, rows, max(1, args.steps))
    print(json.dumps(line), flush=True)


# ------------------------------------------------------------------ native
class L2Flush:
    """Between timed steps: write 1 GiB (> the 126 MB L2), then read another
    1 GiB so the written lines are cleaned out of L2 before the next step —
    the step starts with a cold, clean L2 and does not pay the write-back of
    the flush's own dirty lines."""

    DESCRIPTION = ("flushed between steps outside the timed events: 1 GiB write (> 126 MB L2) then a 1 GiB read "
                   "so no flush-dirty lines remain")

    def __init__(self, device):
        import torch
        self.w = torch.empty(256 * 1024 * 1024, dtype=torch.float32, device=device)
        self.r = torch.zeros(256 * 1024 * 1024, dtype=torch.float32, device=device)
        self.acc = torch.zeros((), dtype=torch.float32, device=device)

    def __call__(self):
        import torch
        self.w.fill_(1.0)
        torch.sum(self.r, dim=0, out=self.acc)


class Case:
    """Device buffers of one mixed step on this rank's batch shard [b0, b1).

    inputs="rng": the reference's own input stream (bcad Rng, mix_seed(42,
    B*1000003+H), bcad_host_random_inputs) for this rank's rows of the FULL
    batch — the union of the shards of any world size is the single-GPU
    batch, and the replicated (1,H) bias arguments are identical on every
    rank; generated into pinned host buffers that the e2e leg reuses.
    inputs="philox": device Philox draws (secondary measurements only)."""

    def __init__(self, w: Workload, device, rows=None, policy: int = 0, inputs: str = "rng", seed: int = 99):
        import numpy as np
        import torch
        from paper_1810_08297_b200 import native
        b0, b1 = rows if rows is not None else (0, w.B)
        B_local = b1 - b0
        self.w, self.B, self.policy, self.rows = w, B_local, policy, (b0, b1)
        dt = torch.float32 if w.dtype == "f32" else torch.float64
        self.dt = dt
        shapes = w.shapes(B_local)
        self.shapes = shapes
        self.host_ins = None
        if inputs == "rng":
            from paper_1810_08297_b200 import host
            p = shard_plan(w.shapes(), 1, 0)  # which arguments carry the batch axis
            blocks = []
            for j, full in enumerate(w.shapes()):
                vol = int(math.prod(full))
                if p.sharded[j]:
                    row = vol // full[0]
                    blocks.append((b0 * row, B_local * row))
                else:
                    blocks.append((0, vol))
            self.host_ins = [torch.empty(s_, dtype=dt, pin_memory=True) for s_ in shapes]
            host.random_inputs(input_seed(w), np.float32 if dt == torch.float32 else np.float64,
                               list(zip(w.shapes(), w.kinds())), blocks,
                               out=[t.numpy().reshape(-1) for t in self.host_ins])
            ins = [t.to(device, non_blocking=False) for t in self.host_ins]
        else:
            g = torch.Generator(device=device)
            g.manual_seed(seed)
            ins = []
            for s_, kind in zip(shapes, w.kinds()):
                if kind == "pm1":
                    ins.append(torch.rand(s_, generator=g, device=device, dtype=dt) * 2 - 1)
                else:
                    ins.append((torch.rand(s_, generator=g, device=device, dtype=dt) < 0.5).to(dt))
        self.ins = ins
        self.k = native.Kernel(w.kernel)
        out = (B_local, w.H)
        self.primal = [torch.empty(out, device=device, dtype=dt)]
        self.partials = ([torch.empty(out, device=device, dtype=dt) for _ in range(self.k.n_in)]
                         if policy == 0 else [])
        self.seed = torch.ones(out, device=device, dtype=dt)
        # Input adjoints; the (1,H) bias adjoints share one contiguous
        # buffer so a single allreduce combines them.
        self.adj = []
        self.bias_adj = None
        if w.variant == "bias":
            self.bias_adj = torch.empty((3, w.H), device=device, dtype=dt)
        for j, s_ in enumerate(shapes):
            if w.variant == "bias" and 4 <= j <= 6:
                self.adj.append(self.bias_adj[j - 4:j - 3])
            else:
                self.adj.append(torch.empty(s_, device=device, dtype=dt))
        self.ws = native.new_workspace(self.k, shapes, dt, device)
        # K1 + K2, plus the finisher K2f when a reduction spans CTAs
        code = native.F32 if dt == torch.float32 else native.F64
        self.launches = 1 + native.pullback_launches(self.k, shapes, code)
        self.step = native.PreparedStep(self.k, ins, self.primal, self.partials, [self.seed], self.adj, self.ws,
                                        policy=policy)


def run_native(args, w: Workload, rank: int, world: int):
    import torch
    import torch.distributed as dist
    from paper_1810_08297_b200 import native

    local = 0 if args.share_device else int(os.environ.get("LOCAL_RANK", "0"))
    if torch.cuda.device_count() <= local:
        raise SystemExit(f"bench.py: rank {rank} needs cuda:{local} but {torch.cuda.device_count()} GPU(s) are "
                         f"visible; run --gpus N with at most the visible GPU count")
    torch.cuda.set_device(local)
    device = torch.device("cuda", local)
    native.check(native.LIB.bcad_cu_set_device(local))

    strong = scaling_of(w) == "strong"
    if strong:  # partition.plan: contiguous batch-row block of this rank
        p = shard_plan(w.shapes(), world, rank)
        b0, b1 = p.rows
    else:
        b0, b1 = 0, w.B  # weak scaling: one B-row batch per GPU
    B_local = b1 - b0
    case = Case(w, device, rows=(b0, b1), policy=args.policy, inputs="rng")
    stream = torch.cuda.Stream(device)
    sp = int(stream.cuda_stream)

    comm = None
    peer = None
    nccl_nranks = None
    fused_error = None
    if world > 1 and w.variant == "bias" and args.allreduce == "fused":
        # K2f fused with the allreduce: fp64 column sums stored into every
        # rank's buffer over NVLink (CUDA IPC), summed in rank order. If any
        # rank cannot set the group up (no peer access / IPC), every rank
        # falls back to the NCCL allreduce.
        ok = 1
        try:
            peer = native.PeerGroup(rank, world, 3 * w.H)
            blobs = [None] * world
            dist.all_gather_object(blobs, peer.blob)
            peer.connect(blobs)
        except Exception as e:  # noqa: BLE001 - reported in the line, NCCL used instead
            ok, fused_error, peer = 0, repr(e)[:200], None
        flags = [None] * world
        dist.all_gather_object(flags, ok)
        if min(flags) == 1:
            case.step = native.PreparedStep(case.k, case.ins, case.primal, case.partials, [case.seed], case.adj,
                                            case.ws, policy=args.policy, peer=peer)
        else:
            peer = None
            fused_error = fused_error or "a peer rank could not join the peer group"
        dist.barrier()
    if world > 1 and w.variant == "bias" and peer is None:
        uid = [native.nccl_unique_id() if rank == 0 else None]
        dist.broadcast_object_list(uid, src=0)
        comm = native.Comm(world, uid[0], rank)
        nccl_nranks = comm.nranks
        assert nccl_nranks == world, (nccl_nranks, world)

    K, W = args.steps, args.warmup
    # Inputs larger than L2 (the contract's alternative to flushing): R
    # independent batch buffer sets, step k runs on set k % R, so every set is
    # revisited only after at least 2 x L2 of other steps' traffic and starts
    # each step out of L2; R = 1 when one step alone moves > 4 x L2.
    R = rotation_sets(w.step_bytes(B_local, args.policy))
    cases = [case] + [Case(w, device, rows=(b0, b1), policy=args.policy, inputs="rng") for _ in range(R - 1)]
    if peer is not None:
        for c in cases[1:]:
            c.step = native.PreparedStep(c.k, c.ins, c.primal, c.partials, [c.seed], c.adj, c.ws,
                                         policy=args.policy, peer=peer)

    def one_step(c, evs=None):
        # K1 -> K2 [-> allreduce] of buffer set c; evs: external events
        # around K1, K2 and the collective (breakdown graphs only)
        if evs:
            evs[0].record(stream)
        c.step.forward(sp)
        if evs:
            evs[1].record(stream)
        c.step.pullback(sp)
        if evs:
            evs[2].record(stream)
        if comm is not None:
            comm.allreduce([c.bias_adj], stream=stream)
        if evs:
            evs[3].record(stream)

    with torch.cuda.stream(stream):
        for k in range(max(W, 2 * R)):
            one_step(cases[k % R])
    torch.cuda.synchronize(device)
    if world > 1:
        dist.barrier()

    # The K timed steps, back to back, captured as ONE CUDA graph (K1 -> K2
    # edges programmatic, PDL) and replayed once untimed, then once between
    # a start and an end event with a barrier + synchronize on both sides.
    graph = torch.cuda.CUDAGraph()
    with torch.cuda.stream(stream):
        with torch.cuda.graph(graph, stream=stream):
            for k in range(K):
                one_step(cases[k % R])
    ev_start, ev_end = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    # the clock sampler starts first (its start-up sleep would otherwise leave
    # the GPU idle right before the timed replay); warm replays then bring the
    # GPU to its loaded clocks, and the timed replay follows at once
    clocks = ClockSampler(local)
    clocks.start()
    with torch.cuda.stream(stream):
        for _ in range(3):
            graph.replay()
    torch.cuda.synchronize(device)
    if world > 1:
        dist.barrier()
    with torch.cuda.stream(stream):
        ev_start.record(stream)
        graph.replay()
        ev_end.record(stream)
    torch.cuda.synchronize(device)
    if world > 1:
        dist.barrier()
    clock_info = clocks.stop()
    total_ms = ev_start.elapsed_time(ev_end)
    # informational (SURVEY §8(d) min / median over >= 20 repetitions): 20
    # more replays of the same K-step graph, each between its own events
    reps = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(20)]
    with torch.cuda.stream(stream):
        for a, b in reps:
            a.record(stream)
            graph.replay()
            b.record(stream)
    torch.cuda.synchronize(device)
    rep_ms = sorted(a.elapsed_time(b) / K for a, b in reps)
    del graph

    # Breakdown (not the reported number): each piece of the step alone, K
    # launches back to back over the same rotating sets as one graph between
    # events (steady state, operands out of L2; K2 alone then reads the
    # partials from HBM, where inside the step they are still in L2).
    def alone(piece):
        g = torch.cuda.CUDAGraph()
        with torch.cuda.stream(stream):
            with torch.cuda.graph(g, stream=stream):
                for k in range(K):
                    piece(cases[k % R])
            for _ in range(3):
                g.replay()
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a.record(stream)
            g.replay()
            b.record(stream)
        torch.cuda.synchronize(device)
        del g
        return a.elapsed_time(b) / K

    k1_alone = alone(lambda c: c.step.forward(sp))
    k2_alone = alone(lambda c: c.step.pullback(sp))
    ar_alone = alone(lambda c: comm.allreduce([c.bias_adj], stream=stream)) if comm is not None else None
    k1_ms, k2_ms = [k1_alone], [k2_alone]
    ar_ms = [ar_alone] if ar_alone is not None else []
    # For comparison only: the round-1 method — L2 flushed, every step timed
    # alone (events around one replay of a 1-step graph), which adds the
    # launch latency of a step that starts from an idle stream.
    l2 = L2Flush(device)
    g1 = torch.cuda.CUDAGraph()
    with torch.cuda.stream(stream):
        with torch.cuda.graph(g1, stream=stream):
            one_step(case)
        iso = [[torch.cuda.Event(enable_timing=True) for _ in range(2)] for _ in range(K)]
        for k in range(3 + K):
            l2()
            if k >= 3:
                iso[k - 3][0].record(stream)
            g1.replay()
            if k >= 3:
                iso[k - 3][1].record(stream)
    torch.cuda.synchronize(device)
    iso_ms = statistics.mean(a.elapsed_time(b) for a, b in iso)
    del g1, l2
    if world > 1:
        t = torch.tensor([total_ms], device=device if dist.get_backend() == "nccl" else "cpu", dtype=torch.float64)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        total_ms = float(t.item())
    ms_per_step = total_ms / K
    cells_per_step = (w.B if strong else w.B * world) * w.H
    value = cells_per_step / (ms_per_step * 1e-3)

    # ---- end to end through the C-ABI with host buffers
    e2e = run_e2e(case, stream, args.e2e_steps, device)
    if world > 1:
        t = torch.tensor([e2e["ms_per_step"]], device=device if dist.get_backend() == "nccl" else "cpu",
                         dtype=torch.float64)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        e2e["ms_per_step"] = float(t.item())
    e2e_value = cells_per_step / (e2e["ms_per_step"] * 1e-3)

    # ---- roofline of the dominant kernel
    peak, peak_src = hbm_peak()
    k1_avg, k2_avg = statistics.mean(k1_ms), statistics.mean(k2_ms)
    dom = "K1_forward" if k1_avg >= k2_avg else "K2_pullback"
    dom_bytes = w.k1_bytes(B_local, args.policy) if dom == "K1_forward" else w.k2_bytes(B_local, args.policy)
    dom_ms = max(k1_avg, k2_avg)
    achieved = dom_bytes / (dom_ms * 1e-3) / 1e9
    traffic = None
    try:
        with open(NCU_SUMMARY) as f:
            traffic = json.load(f).get(w.key, {}).get(dom)
    except Exception:
        pass
    step_bytes = w.step_bytes(B_local, args.policy)

    if rank != 0:
        return
    extra = {}
    if world == 1 and args.extra:
        for key in ("" if args.extra == "none" else args.extra).split(","):
            if not key or key == w.key:
                continue
            if key == "tape":
                extra[key] = measure_tape(device, stream, max(20, K))
            elif key == "shards":
                extra[key] = measure_shards(device, stream, max(20, K))
            elif key == "arity":
                extra[key] = measure_arity(device, stream, max(20, K))
            elif key.endswith(":r"):  # RecomputeReverse: K1p primal + fused K2r
                extra[key] = measure_secondary(WORKLOADS[key[:-2]], device, stream, max(20, K), 1, bool(args.graph))
            else:
                extra[key] = measure_secondary(WORKLOADS[key], device, stream, max(20, K), args.policy, bool(args.graph))

    cpu = None
    if world == 1 and not args.no_cpu_baseline:
        cpu = cpu_reference_rate(w, budget_s=args.cpu_budget)

    line = {
        "metric": "HM-LSTM cell-update grad elements/s", "value": value, "unit": "grad elements/s",
        "n_gpus": world, "steps": K, "warmup": W, "ms_per_step": ms_per_step, "higher_is_better": True,
        "scaling": scaling_of(w), "vs_baseline": None, "dtype": w.dtype, "data": DATA,
        "config": bench_config(w, world, args.policy),
        "run": {"B_per_gpu": B_local, "rows_rank0": [b0, b1], "buffer_sets": R,
                "launch": "the K steps as one CUDA graph replay (K1 -> K2 edges programmatic, PDL)"},
        "breakdown_ms": {"K1_forward": k1_avg, "K2_pullback": k2_avg,
                         "timing": "each kernel alone: K launches over the rotating sets as one CUDA graph between "
                                   "events, divided by K (K2 alone reads its partials from HBM)",
                         "allreduce": statistics.mean(ar_ms) if ar_ms else None},
        "replays_ms_per_step": {"min": rep_ms[0], "median": rep_ms[len(rep_ms) // 2], "max": rep_ms[-1],
                                "n": len(rep_ms), "note": "20 further replays of the timed K-step graph (informational; "
                                                          "the reported value is the single bracketed replay)"},
        "isolated_step": {"ms_per_step": iso_ms, "value": cells_per_step / (iso_ms * 1e-3),
                          "method": "round-1 method, for comparison: L2 flushed before every step, each step timed "
                                    "alone (one 1-step graph replay between events) — adds the launch latency of "
                                    "a step issued to an idle stream"},
        "step_roofline": {"bytes": step_bytes, "achieved_GBps": step_bytes / (ms_per_step * 1e-3) / 1e9,
                          "frac": step_bytes / (ms_per_step * 1e-3) / 1e9 / peak},
        "roofline": {"bound": "hbm", "kernel": dom, "achieved": achieved, "peak": peak, "unit": "GB/s",
                     "frac": achieved / peak, "traffic": traffic, "algorithmic_bytes_per_launch": dom_bytes,
                     "kernel_timing": "K launches of the kernel alone over the rotating buffer sets as one CUDA "
                                      "graph between CUDA events on its stream, divided by K (steady state, operands "
                                      "out of L2)",
                     "peak_source": peak_src},
        "e2e": {"value": e2e_value, "unit": "grad elements/s", "h2d_bytes_per_step": e2e["h2d"],
                "d2h_bytes_per_step": e2e["d2h"], "ms_per_step": e2e["ms_per_step"],
                "path": (("a stream of steps through bcad_host_mixed_step_async (include/bcad_host.h, 2 row chunks "
                          "per step): consecutive steps overlap (step k+1's uploads during step k's downloads), each "
                          "step uploading its inputs and seed and downloading its gradients; wall clock to "
                          "bcad_host_synchronize / steps. " if e2e["overlapped"] else "") +
                         "Default schedule: row-chunk pipelined over copy/compute streams, prepared (device buffers "
                         "kept across calls on the same pinned buffers); each chunk is bcad_cu_forward + "
                         "bcad_cu_pullback through the C-ABI, not through the C++ Tape"),
                "per_call_ms_per_step": e2e["per_call_ms_per_step"],
                "tape_path": {"ms_per_step": e2e["one_shot_ms_per_step"],
                              "value": cells_per_step / (e2e["one_shot_ms_per_step"] * 1e-3),
                              "path": "bcad_host_mixed_step one-shot (bcad_host_set_pipeline(1)): C++ Tape + "
                                      "mixed_broadcast + Tape::backward over device tensors, reference run_cell_once "
                                      "order (bench.cpp:112-128)"},
                "pipelined_unprepared_ms_per_step": e2e["pipelined_unprepared_ms_per_step"], "pcie": e2e["pcie"]},
        "gpu_launches": case.launches * K,
        "clocks": clock_info,
    }
    if world > 1:
        line["multi_gpu"] = {"nccl_nranks": nccl_nranks, "world_size": world,
                             "allreduce": ("fused: K2f-AR stores fp64 column sums into every rank's buffer over "
                                           "NVLink peer memory (CUDA IPC), flag exchange, rank-order sum "
                                           "(bcad_cu_pullback_allreduce)" if peer is not None
                                           else "NCCL ncclAllReduce of the 3 x H fp32 bias adjoints after K2f"
                                           if comm is not None else None),
                             "fused_fallback_reason": fused_error,
                             "allreduce_us_per_step": (statistics.mean(ar_ms) * 1e3 if ar_ms else None),
                             "allreduce_bytes": (case.bias_adj.numel() * case.bias_adj.element_size()
                                                 if comm is not None else 0),
                             "timing": "max over ranks of the K-step device time (CUDA events, barrier + sync "
                                       "on both sides)"}
    if cpu:
        line["cpu_baseline"] = cpu
    if extra:
        line["extra"] = extra
    print(json.dumps(line), flush=True)


def run_e2e(case: Case, stream, steps: int, device):
    """The user-facing call with HOST buffers (include/bcad_host.h ->
    C++ Tape + mixed_broadcast + backward over libbcad_cu.so), every step:
    pinned H2D of the inputs and the seed, K1, K2, D2H of every input
    gradient, stream-synchronised return. Wall-clock per call. Reported with
    the library's default row-chunk pipelining (bcad_host_set_pipeline(0));
    the one-shot schedule (one tape over the whole batch) and the bare PCIe
    copy rates of the same bytes are measured beside it."""
    import torch
    from paper_1810_08297_b200 import host
    host_in = case.host_ins if case.host_ins is not None else [t.cpu().pin_memory() for t in case.ins]
    host_seed = case.seed.cpu().pin_memory()
    host_grad = [torch.empty(t.shape, dtype=t.dtype).pin_memory() for t in case.adj]
    np_in = [t.numpy() for t in host_in]
    np_grad = [t.numpy() for t in host_grad]
    call = host.HostStep(case.w.kernel, np_in, [host_seed.numpy()], grads_out=np_grad, policy=case.policy,
                         stream=int(stream.cuda_stream))
    h2d = sum(a.nbytes for a in np_in) + host_seed.numpy().nbytes
    d2h = sum(a.nbytes for a in np_grad)

    def wall(n):
        for _ in range(2):
            call()
        torch.cuda.synchronize(device)
        t0 = time.perf_counter()
        for _ in range(n):
            call()
        return (time.perf_counter() - t0) * 1e3 / n

    try:
        host.set_pipeline(1)
        one_shot = wall(steps)
        host.set_pipeline(0)
        host.set_prepared(False)
        unprepared = wall(steps)
    finally:
        host.set_pipeline(0)
        host.set_prepared(True)
    per_call = wall(steps)

    # A stream of steps through the asynchronous call (bcad_host_mixed_step_async):
    # step k+1's uploads run while step k's downloads drain (each step still
    # uploads its inputs and seed and downloads its gradients; steps on the
    # same buffers are ordered by the library). Wall clock from the first
    # enqueue to bcad_host_synchronize, divided by the steps.
    sp = int(stream.cuda_stream)
    try:
        for k in range(4):
            call.enqueue()
        host.synchronize(sp)
        n = max(steps, 10)
        t0 = time.perf_counter()
        for k in range(n):
            call.enqueue()
        host.synchronize(sp)
        ms = (time.perf_counter() - t0) * 1e3 / n
        overlapped = True
    except Exception:  # noqa: BLE001 - a problem too small to chunk: per-call timing stands
        ms, overlapped = per_call, False
    # bare copy rates of the same byte volumes (pinned, one stream)
    dev_in = torch.empty(h2d // 4, dtype=torch.float32, device=device)
    hin = torch.empty(h2d // 4, dtype=torch.float32).pin_memory()
    dev_out = torch.empty(d2h // 4, dtype=torch.float32, device=device)
    hout = torch.empty(d2h // 4, dtype=torch.float32).pin_memory()
    with torch.cuda.stream(stream):
        def copy_ms(fn, n=10):
            fn()
            torch.cuda.synchronize(device)
            t0 = time.perf_counter()
            for _ in range(n):
                fn()
            torch.cuda.synchronize(device)
            return (time.perf_counter() - t0) * 1e3 / n
        h2d_ms = copy_ms(lambda: dev_in.copy_(hin, non_blocking=True))
        d2h_ms = copy_ms(lambda: hout.copy_(dev_out, non_blocking=True))
    return {"ms_per_step": ms, "h2d": h2d, "d2h": d2h, "one_shot_ms_per_step": one_shot,
            "pipelined_unprepared_ms_per_step": unprepared, "per_call_ms_per_step": per_call,
            "overlapped": overlapped,
            "pcie": {"h2d_GBps": h2d / (h2d_ms * 1e-3) / 1e9, "d2h_GBps": d2h / (d2h_ms * 1e-3) / 1e9,
                     "serial_copy_ms": h2d_ms + d2h_ms}}


def measure_secondary(w: Workload, device, stream, steps: int, policy: int, graph_step: bool = True):
    """A secondary config measured like the headline: `steps` steps back to
    back as one CUDA graph over rotating buffer sets (inputs larger than L2);
    K1 and K2 each alone the same way for the per-kernel split."""
    import torch
    R = rotation_sets(w.step_bytes(policy=policy))
    cases = [Case(w, device, policy=policy, inputs="philox", seed=99 + r) for r in range(R)]
    sp = int(stream.cuda_stream)
    K = steps
    with torch.cuda.stream(stream):
        for k in range(2 * R):
            cases[k % R].step.forward(sp)
            cases[k % R].step.pullback(sp)

    def timed(piece):
        g = torch.cuda.CUDAGraph()
        with torch.cuda.stream(stream):
            with torch.cuda.graph(g, stream=stream):
                for k in range(K):
                    piece(cases[k % R])
            for _ in range(3):
                g.replay()
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a.record(stream)
            g.replay()
            b.record(stream)
        torch.cuda.synchronize(device)
        del g
        return a.elapsed_time(b) / K

    def both(c):
        c.step.forward(sp)
        c.step.pullback(sp)

    step = timed(both)
    k1 = timed(lambda c: c.step.forward(sp))
    k2 = timed(lambda c: c.step.pullback(sp))
    peak, _ = hbm_peak()
    b1, b2 = w.k1_bytes(policy=policy), w.k2_bytes(policy=policy)
    out = {"workload": w.describe, "ms_per_step": step, "value": w.E / (step * 1e-3), "unit": "grad elements/s",
           "launch": f"{K} steps back to back as one CUDA graph over {R} rotating buffer set(s); K1 / K2 each alone "
                     f"the same way",
           "K1_ms": k1, "K2_ms": k2, "K1_frac_hbm": b1 / (k1 * 1e-3) / 1e9 / peak,
           "K2_frac_hbm": b2 / (k2 * 1e-3) / 1e9 / peak,
           "step_frac_hbm": (b1 + b2) / (step * 1e-3) / 1e9 / peak}
    del cases
    torch.cuda.empty_cache()
    return out


def timed_steps(fn, stream, device, steps):
    """Median device time of fn() over `steps` runs, L2 flushed before each."""
    import torch
    l2 = L2Flush(device)
    ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(steps)]
    with torch.cuda.stream(stream):
        for _ in range(3):
            l2()
            fn()
        for a, b in ev:
            l2()
            a.record(stream)
            fn()
            b.record(stream)
    torch.cuda.synchronize(device)
    return statistics.median(a.elapsed_time(b) for a, b in ev)


def measure_tape(device, stream, steps: int):
    """Paper Fig. 1 on B200: the four gradients of the n x n cell update
    through the C++ tape (cell_gradients, hmlstm.hpp:123-142) — mixed-mode
    (one fused node) vs the reverse-mode vectorised-select baseline (8 tensor
    primitives), device-resident, tape input copies included as in the
    reference's run_cell_once (bench.cpp:112-128)."""
    import torch
    from paper_1810_08297_b200 import host
    n = 1024
    g = torch.Generator(device=device)
    g.manual_seed(5)
    ins = [torch.rand((n, n), generator=g, device=device) * 2 - 1 for _ in range(4)]
    ins += [(torch.rand(n, generator=g, device=device) < 0.5).float() for _ in range(2)]
    seed = torch.ones((n, n), device=device)
    grads = [torch.empty((n, n), device=device) for _ in range(4)]
    out = {"n": n, "dtype": "f32"}
    for impl in ("mixed-cache", "mixed-recompute", "reverse-unfused"):
        nodes, peak = host.cell_gradients(impl, ins, seed, grads, stream)
        ms = timed_steps(lambda: host.cell_gradients(impl, ins, seed, grads, stream), stream, device, steps)
        out[impl] = {"ms": ms, "tape_nodes": nodes, "peak_cached_bytes": peak}
    out["speedup_mixed_cache_vs_reverse_unfused"] = out["reverse-unfused"]["ms"] / out["mixed-cache"]["ms"]
    return out


def measure_shards(device, stream, steps: int):
    """Config 5 strong scaling, the compute side, on one GPU: the step of the
    batch shard one of G GPUs owns (B = 65536 / G rows of the bias variant,
    partition.plan) timed here for G = 1, 2, 4, 8. The projected G-GPU step
    is the shard step plus the allreduce of the 3 x H reduced (1,H)
    adjoints (48 KB; fused into the pullback's finisher in the multi-GPU run),
    which this single-GPU run cannot time; efficiency is reported without it.
    A projection, not a multi-GPU measurement."""
    base = WORKLOADS["cfg5"]
    out = {"workload": base.describe, "note": "per-shard step on one B200; allreduce of 3*H fp32 not included"}
    t1 = None
    for G in (1, 2, 4, 8):
        w = Workload(base.key, base.B // G, base.H, base.dtype, base.variant, base.describe)
        r = measure_secondary(w, device, stream, steps, 0)
        t1 = r["ms_per_step"] if G == 1 else t1
        out[f"G{G}"] = {"B_per_gpu": w.B, "shard_ms_per_step": r["ms_per_step"], "step_frac_hbm": r["step_frac_hbm"],
                        "projected_value": base.B * base.H / (r["ms_per_step"] * 1e-3),
                        "projected_efficiency": t1 / (G * r["ms_per_step"])}
    return out


def measure_arity(device, stream, steps: int):
    """Paper §3.4.1 / Fig. 3 on B200: forward-mode diagonal Jacobian of
    tanh_product_A (arity_workload.hpp:19-28) at 4096 x 4096 fp32 (large
    enough that launch costs vanish), one fused K1 per call; bytes = (A
    inputs + primal + A partials) * 4 per cell. Cells per thread drop from 4
    to 2 (A = 8) and 1 (A >= 16) to keep the A-wide duals in registers."""
    import torch
    from paper_1810_08297_b200 import native
    n = 4096
    peak, _ = hbm_peak()
    out = {"n": n, "cells_per_thread": {"1": 4, "2": 4, "4": 4, "8": 2, "16": 1, "18": 1, "32": 1}}
    g = torch.Generator(device=device)
    g.manual_seed(9)
    for A in (1, 2, 4, 8, 16, 18, 32):
        k = native.Kernel(f"tanh_product_{A}")
        ins = [torch.rand((n, n), generator=g, device=device) * 2 - 1 for _ in range(A)]
        prim = [torch.empty((n, n), device=device)]
        parts = [torch.empty((n, n), device=device) for _ in range(A)]
        ms = timed_steps(lambda: native.forward(k, ins, prim, parts, stream=stream), stream, device, steps)
        b = (2 * A + 1) * n * n * 4
        out[f"A{A}"] = {"ms": ms, "GBps": b / (ms * 1e-3) / 1e9, "frac_hbm": b / (ms * 1e-3) / 1e9 / peak}
        del ins, parts
    return out


def spawn_ranks(n: int) -> int:
    """Re-launch this command under torch.distributed.run with n ranks on
    this node (rendezvous on 127.0.0.1); returns the launcher's exit code."""
    import socket
    with socket.socket() as sk:
        sk.bind(("127.0.0.1", 0))
        port = sk.getsockname()[1]
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={n}",
           "--master-addr=127.0.0.1", f"--master-port={port}", os.path.abspath(__file__), *sys.argv[1:]]
    env = dict(os.environ, OMP_NUM_THREADS=os.environ.get("OMP_NUM_THREADS", "1"))
    return subprocess.call(cmd, env=env)


def run_dry(args, w: Workload, rank: int, world: int):
    """--dry-run: the N-rank plumbing on CPU (gloo): every rank plans its
    batch shard, the ranks are counted by an allreduce, and rank 0 prints
    the plan. No GPU work, no timing."""
    import torch
    import torch.distributed as dist
    p = shard_plan(w.shapes(), world, rank) if scaling_of(w) == "strong" else shard_plan(w.shapes(), 1, 0)
    one = torch.ones(1, dtype=torch.int64)
    if world > 1:
        dist.all_reduce(one)
    rows = [None] * world
    if world > 1:
        dist.all_gather_object(rows, list(p.rows))
    else:
        rows = [list(p.rows)]
    if rank == 0:
        print(json.dumps({"dry_run": True, "n_gpus": world, "ranks_seen": int(one.item()),
                          "backend": dist.get_backend() if world > 1 else None, "scaling": scaling_of(w),
                          "config": bench_config(w, world, args.policy), "rows_per_rank": rows,
                          "allreduce_args": list(p.allreduce)}), flush=True)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=None, help="ranks (one per GPU); default: WORLD_SIZE or 1")
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--config", default=None, choices=sorted(WORKLOADS),
                    help="default cfg2 at one GPU, cfg5 (strong scaling, NCCL allreduce) at N > 1")
    ap.add_argument("--impl", default="native", choices=["native", "reference"])
    ap.add_argument("--policy", type=int, default=0, help="0 CacheForward, 1 RecomputeReverse")
    ap.add_argument("--share-device", action="store_true",
                    help="test aid: every rank on cuda:0 (exercises the N-rank path and the fused peer allreduce on "
                         "a one-GPU box; NCCL refuses it; timings are meaningless)")
    ap.add_argument("--allreduce", choices=("nccl", "fused"), default="fused",
                    help="N > 1, bias variant: the pullback's finisher fused with the allreduce over NVLink peer "
                         "memory (bcad_cu_pullback_allreduce; default, falls back to NCCL if a rank cannot join), "
                         "or the NCCL allreduce after the pullback")
    ap.add_argument("--e2e-steps", type=int, default=10)
    ap.add_argument("--graph", type=int, default=1,
                    help="kept for compatibility: the timed steps always run as one captured CUDA graph")
    ap.add_argument("--extra", default="cfg3,cfg4,cfg4div,cfg5,cfg2:r,cfg5:r,tape,arity,shards",
                    help="secondary measurements at N=1 ('none' for none): configs, <cfg>:r = RecomputeReverse, "
                         "tape = cell_gradients mixed vs reverse-unfused, arity = tanh_product study, "
                         "shards = config 5's per-GPU batch shards at G = 2, 4, 8 timed on this GPU")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--cpu-budget", type=float, default=12.0)
    ap.add_argument("--dry-run", action="store_true", help="N-rank plumbing only, gloo on CPU")
    args = ap.parse_args()
    if args.warmup < 3:
        ap.error("--warmup must be >= 3")

    if "WORLD_SIZE" not in os.environ and (args.gpus or 1) > 1:
        sys.exit(spawn_ranks(args.gpus))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    if args.gpus is not None and args.gpus != world:
        ap.error(f"--gpus {args.gpus} but the launcher started {world} rank(s)")
    w = WORKLOADS[args.config or ("cfg2" if world == 1 else "cfg5")]
    if args.dry_run:
        import torch.distributed as dist
        if world > 1:
            dist.init_process_group("gloo")
        try:
            run_dry(args, w, rank, world)
        finally:
            if world > 1:
                dist.destroy_process_group()
        return
    if args.impl == "reference":
        run_reference_arm(args, w, rank, world)
        return
    if world > 1:
        import torch
        import torch.distributed as dist
        if args.share_device:  # NCCL refuses two ranks on one GPU; plumbing over gloo
            torch.cuda.set_device(0)
            dist.init_process_group("gloo")
        else:
            torch.cuda.set_device(int(os.environ.get("LOCAL_RANK", "0")))
            dist.init_process_group("nccl", device_id=torch.device("cuda", int(os.environ.get("LOCAL_RANK", "0"))))
    try:
        run_native(args, w, rank, world)
    finally:
        if world > 1:
            import torch.distributed as dist
            dist.destroy_process_group()


if __name__ == "__main__":
    main()
