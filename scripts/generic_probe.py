"""Dev probe: throughput of the generic rank-N kernels (problems whose
broadcast pattern does not reduce to 2-D) against a 2-D problem of the same
volume, forward (CacheForward) and pullback, fp32."""
import json
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1810_08297_b200 import native  # noqa: E402


def run(shapes, name="gate", reps=20):
    k = native.Kernel(name)
    ins = [torch.rand(s, device="cuda") for s in shapes]
    out = torch.broadcast_shapes(*[s + (1,) * (max(len(x) for x in shapes) - len(s)) for s in shapes])
    prim = [torch.empty(out, device="cuda")]
    parts = [torch.empty(out, device="cuda") for _ in range(k.n_in)]
    seed = [torch.ones(out, device="cuda")]
    adj = [torch.empty(s, device="cuda") for s in shapes]
    ws = native.new_workspace(k, shapes, torch.float32)
    for _ in range(3):
        native.forward(k, ins, prim, parts)
        native.pullback(k, shapes, seed, parts, ins, adj, workspace=ws)
    torch.cuda.synchronize()
    a, b, c = [torch.cuda.Event(enable_timing=True) for _ in range(3)]
    a.record()
    for _ in range(reps):
        native.forward(k, ins, prim, parts)
    b.record()
    for _ in range(reps):
        native.pullback(k, shapes, seed, parts, ins, adj, workspace=ws)
    c.record()
    torch.cuda.synchronize()
    E = prim[0].numel()
    fb = (sum(t.numel() for t in ins) + (1 + k.n_in) * E) * 4
    pb = ((1 + k.n_in) * E + sum(t.numel() for t in ins)) * 4
    return {"shapes": [list(s) for s in shapes], "fwd_us": a.elapsed_time(b) / reps * 1e3,
            "pull_us": b.elapsed_time(c) / reps * 1e3,
            "fwd_GBps": fb / (a.elapsed_time(b) / reps * 1e-3) / 1e9,
            "pull_GBps": pb / (b.elapsed_time(c) / reps * 1e-3) / 1e9,
            "pull_launches": native.pullback_launches(k, shapes, native.F32)}


out = [run([(64, 256, 1024), (64, 1, 1024)]),   # 3 axis groups: generic
       run([(64, 256, 1024), (1, 256, 1)]),     # generic
       run([(64, 256, 1024), (1, 1, 1024)]),    # 2-D (COL) after axis merging
       run([(64, 256, 1024), (1, 256, 1024)]),  # 2-D (COL)
       run([(64, 256, 1024), (64, 256, 1)]),    # 2-D (ROW)
       run([(4, 256, 1024), (4, 1, 1024)]),     # generic, small argument (column segments)
       run([(64 * 256, 1024), (1, 1024)]),      # 2-D of the same volume
       run([(64 * 256, 1024), (64 * 256, 1)])]
print(json.dumps(out, indent=1))
