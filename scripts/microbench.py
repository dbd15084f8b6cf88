"""Dev micro-benchmarks (run under gpurun): fixed per-launch cost of K1/K2 at
tiny sizes, a plain device copy of cfg2's byte volume, and K1/K2 vs size —
to separate launch/drain overhead from bandwidth at the cfg2 scale."""
import json
import os
import statistics
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from bench import Case, L2Flush  # noqa: E402
from paper_1810_08297_b200.workloads import Workload  # noqa: E402

dev = torch.device("cuda", 0)
stream = torch.cuda.Stream(dev)
sp = int(stream.cuda_stream)
flush_w = torch.empty(256 * 1024 * 1024, dtype=torch.float32, device=dev)
l2 = L2Flush(dev)
MODE = {"mode": "write+read"}


def timeit(fn, reps=30, do_flush=True):
    ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(reps)]
    with torch.cuda.stream(stream):
        for _ in range(3):
            fn()
        for a, b in ev:
            if do_flush:
                if MODE["mode"] == "write":
                    flush_w.fill_(1.0)
                else:
                    l2()
            a.record(stream)
            fn()
            b.record(stream)
    torch.cuda.synchronize()
    return statistics.median(a.elapsed_time(b) * 1e3 for a, b in ev)


out = {}
MODE["mode"] = "write"
MODE["mode"] = "write+read"
out["empty_event_pair_us"] = timeit(lambda: None)
x = torch.empty(92_291_072 // 4, device=dev)
y = torch.empty_like(x)
out["copy_46MB_read_46MB_write_us"] = timeit(lambda: y.copy_(x))
x2 = torch.empty(16 * 1024 * 1024 // 4, device=dev)
out["fill_16MB_us"] = timeit(lambda: x2.fill_(2.0))
for mode in ("write", "write+read"):
    MODE["mode"] = mode
    out[f"{mode}_copy_46MB_us"] = timeit(lambda: y.copy_(x))
    w = Workload("t", 1024, 1024, "f32", "canonical", "t")
    c = Case(w, 1024, dev, seed=1)
    out[f"{mode}_cfg2_K1K2_us"] = timeit(lambda: (c.step.forward(sp), c.step.pullback(sp)))
    del c
MODE["mode"] = "write+read"
for B in (8, 64, 256, 1024, 4096):
    w = Workload("t", B, 1024, "f32", "canonical", "t")
    c = Case(w, B, dev, seed=1)
    k1 = timeit(lambda: c.step.forward(sp))
    both = timeit(lambda: (c.step.forward(sp), c.step.pullback(sp)))
    out[f"B{B}_K1_us"] = k1
    out[f"B{B}_K1K2_us"] = both
    out[f"B{B}_step_GBps"] = w.step_bytes(B) / (both * 1e-6) / 1e9
    del c
print(json.dumps(out, indent=1))
