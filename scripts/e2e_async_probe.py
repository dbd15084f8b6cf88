"""Dev probe: wall time per step of a stream of asynchronous host steps
(bcad_host_mixed_step_async, two alternating gradient buffer sets) against
the chunk count, config 2."""
import json
import os
import sys
import time

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from bench import Case  # noqa: E402
from paper_1810_08297_b200 import host  # noqa: E402
from paper_1810_08297_b200.workloads import WORKLOADS  # noqa: E402

dev = torch.device("cuda", 0)
stream = torch.cuda.Stream(dev)
sp = int(stream.cuda_stream)
out = {}
w = WORKLOADS["cfg2"]
case = Case(w, dev, rows=(0, w.B), policy=0, inputs="philox", seed=1)
hin = [t.cpu().pin_memory().numpy() for t in case.ins]
seed = case.seed.cpu().pin_memory().numpy()
grads = [[torch.empty(t.shape).pin_memory().numpy() for t in case.adj] for _ in range(3)]
for chunks in (2, 3, 4, 6, 8, 0):
    host.set_pipeline(chunks)
    for nsets in (1, 2, 3):
        calls = [host.HostStep(w.kernel, hin, [seed], grads_out=grads[s], stream=sp) for s in range(nsets)]
        for k in range(6):
            calls[k % nsets].enqueue()
        host.synchronize(sp)
        ts = []
        for rep in range(5):
            t0 = time.perf_counter()
            for k in range(30):
                calls[k % nsets].enqueue()
            host.synchronize(sp)
            ts.append((time.perf_counter() - t0) * 1e3 / 30)
        ts.sort()
        out[f"chunks{chunks}_sets{nsets}_ms"] = ts[2]
        # host enqueue cost alone
    t0 = time.perf_counter()
    for k in range(30):
        calls[k % nsets].enqueue()
    t1 = time.perf_counter()
    host.synchronize(sp)
    out[f"chunks{chunks}_enqueue_ms_per_step"] = (t1 - t0) * 1e3 / 30
host.set_pipeline(0)
print(json.dumps(out))
