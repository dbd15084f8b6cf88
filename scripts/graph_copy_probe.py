import json, time, torch
dev = torch.device("cuda", 0)
n = 5 << 20
hin = torch.empty(n).pin_memory(); din = torch.empty(n, device=dev)
hout = torch.empty(n).pin_memory(); dout = torch.empty(n, device=dev)
s0 = torch.cuda.Stream(); s1 = torch.cuda.Stream(); s2 = torch.cuda.Stream()
def issue():
    ev = torch.cuda.Event()
    ev.record(s0)
    s1.wait_event(ev); s2.wait_event(ev)
    with torch.cuda.stream(s1):
        din.copy_(hin, non_blocking=True)
    with torch.cuda.stream(s2):
        hout.copy_(dout, non_blocking=True)
    e1 = torch.cuda.Event(); e2 = torch.cuda.Event()
    e1.record(s1); e2.record(s2)
    s0.wait_event(e1); s0.wait_event(e2)
def wall(fn, reps=20):
    fn(); torch.cuda.synchronize()
    t0 = time.perf_counter()
    for _ in range(reps): fn()
    torch.cuda.synchronize()
    return (time.perf_counter() - t0) * 1e3 / reps
out = {"direct_ms": wall(issue)}
g = torch.cuda.CUDAGraph()
with torch.cuda.stream(s0):
    torch.cuda.synchronize()
    with torch.cuda.graph(g, stream=s0):
        issue()
out["graph_ms"] = wall(lambda: g.replay())
with torch.cuda.stream(s1):
    out["h2d_only_ms"] = wall(lambda: din.copy_(hin, non_blocking=True))
print(json.dumps(out))
