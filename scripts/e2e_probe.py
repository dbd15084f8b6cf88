"""Dev probe (run under gpurun): wall time of the host C-ABI step
(bcad_host_mixed_step) vs the pipeline chunk count, for cfg2 and cfg3."""
import json
import os
import sys
import time

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from bench import Case  # noqa: E402
from paper_1810_08297_b200 import host  # noqa: E402
from paper_1810_08297_b200.workloads import WORKLOADS  # noqa: E402

dev = torch.device("cuda", 0)
stream = torch.cuda.Stream(dev)
out = {}
for key in ("cfg2", "cfg3"):
    w = WORKLOADS[key]
    case = Case(w, w.B, dev, seed=1)
    host_in = [t.cpu().pin_memory() for t in case.ins]
    host_seed = case.seed.cpu().pin_memory()
    host_grad = [torch.empty(t.shape, dtype=t.dtype).pin_memory() for t in case.adj]
    call = host.HostStep(w.kernel, [t.numpy() for t in host_in], [host_seed.numpy()],
                         grads_out=[t.numpy() for t in host_grad], stream=int(stream.cuda_stream))
    for chunks in (1, 2, 3, 4, 6, 8, 12, 16, 0):
        host.set_pipeline(chunks)
        for _ in range(3):
            call()
        ts = []
        for _ in range(15):
            t0 = time.perf_counter()
            call()
            ts.append((time.perf_counter() - t0) * 1e3)
        ts.sort()
        out[f"{key}_chunks{chunks}_ms"] = ts[len(ts) // 2]
    host.set_pipeline(0)
    del case
# PCIe: H2D alone, D2H alone, both at once on two streams (20 MiB each)
n = 5 << 20
hin = torch.empty(n).pin_memory()
hout = torch.empty(n).pin_memory()
din = torch.empty(n, device=dev)
dout = torch.empty(n, device=dev)
s1, s2 = torch.cuda.Stream(dev), torch.cuda.Stream(dev)


def wall(fn, reps=20):
    fn()
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    for _ in range(reps):
        fn()
    torch.cuda.synchronize()
    return (time.perf_counter() - t0) * 1e3 / reps


def both():
    with torch.cuda.stream(s1):
        din.copy_(hin, non_blocking=True)
    with torch.cuda.stream(s2):
        hout.copy_(dout, non_blocking=True)


with torch.cuda.stream(s1):
    out["h2d_20MiB_ms"] = wall(lambda: din.copy_(hin, non_blocking=True))
    out["d2h_20MiB_ms"] = wall(lambda: hout.copy_(dout, non_blocking=True))
out["both_20MiB_ms"] = wall(both)
# host-side cost of one call: a tiny problem (GPU time negligible)
from paper_1810_08297_b200.workloads import Workload  # noqa: E402
w = Workload("tiny", 64, 1024, "f32", "canonical", "tiny")
case = Case(w, 64, dev, seed=2)
hi = [t.cpu().pin_memory() for t in case.ins]
hs = case.seed.cpu().pin_memory()
hg = [torch.empty(t.shape, dtype=t.dtype).pin_memory() for t in case.adj]
call = host.HostStep(w.kernel, [t.numpy() for t in hi], [hs.numpy()], grads_out=[t.numpy() for t in hg],
                     stream=int(stream.cuda_stream))
for chunks in (1, 2, 4, 8):
    host.set_pipeline(chunks)
    out[f"tiny64x1024_chunks{chunks}_ms"] = wall(call, 50)
host.set_pipeline(0)
print(json.dumps(out, indent=1))
