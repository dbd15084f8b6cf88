"""Dev probe: steady-state step time with R rotating batch buffer sets (inputs
larger than L2 in aggregate) vs the flushed, individually timed step."""
import json
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from bench import Case, L2Flush  # noqa: E402
from paper_1810_08297_b200.workloads import WORKLOADS  # noqa: E402

dev = torch.device("cuda", 0)
stream = torch.cuda.Stream(dev)
sp = int(stream.cuda_stream)
out = {}
for key in ("cfg2", "cfg3"):
    w = WORKLOADS[key]
    step_bytes = w.step_bytes() if hasattr(w, "step_bytes") else None
    for R in (1, 3, 5, 8):
        cases = [Case(w, dev, rows=(0, w.B), policy=0, inputs="philox", seed=17 + r) for r in range(R)]
        K = 40
        g = torch.cuda.CUDAGraph()
        with torch.cuda.stream(stream):
            for k in range(2 * R):  # warm
                c = cases[k % R]
                c.step.forward(sp)
                c.step.pullback(sp)
            with torch.cuda.graph(g, stream=stream):
                for k in range(K):
                    c = cases[k % R]
                    c.step.forward(sp)
                    c.step.pullback(sp)
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            ts = []
            for rep in range(7):
                L2Flush(dev)() if rep == 0 else None
                e0.record(stream)
                g.replay()
                e1.record(stream)
                stream.synchronize()
                ts.append(e0.elapsed_time(e1) / K)
        ts.sort()
        out[f"{key}_R{R}_ms_per_step"] = ts[len(ts) // 2]
        del g, cases
        torch.cuda.empty_cache()
print(json.dumps(out))
