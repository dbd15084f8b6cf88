import json, time, torch
dev = torch.device("cuda", 0)
out = {}
n = 5 << 20  # 20 MiB of floats
hin = torch.empty(n).pin_memory(); din = torch.empty(n, device=dev)
hout = torch.empty(n).pin_memory(); dout = torch.empty(n, device=dev)
ss = [torch.cuda.Stream(dev) for _ in range(4)]
def wall(fn, reps=30):
    fn(); torch.cuda.synchronize()
    t0 = time.perf_counter()
    for _ in range(reps): fn()
    torch.cuda.synchronize()
    return (time.perf_counter() - t0) * 1e3 / reps
for k in (1, 2, 4):
    def h2d():
        for q in range(k):
            with torch.cuda.stream(ss[q]):
                din[q * n // k:(q + 1) * n // k].copy_(hin[q * n // k:(q + 1) * n // k], non_blocking=True)
    def d2h():
        for q in range(k):
            with torch.cuda.stream(ss[q]):
                hout[q * n // k:(q + 1) * n // k].copy_(dout[q * n // k:(q + 1) * n // k], non_blocking=True)
    out[f"h2d_{k}streams_GBps"] = n * 4 / (wall(h2d) * 1e-3) / 1e9
    out[f"d2h_{k}streams_GBps"] = n * 4 / (wall(d2h) * 1e-3) / 1e9
print(json.dumps(out, indent=1))
