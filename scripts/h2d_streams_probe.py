"""Dev probe: pinned H2D bandwidth of config 2's step inputs (21 MB) as one
copy on one stream vs split across 2 / 4 streams (copy engines) issued
concurrently, and the same for D2H (17 MB)."""
import json
import sys

import torch


def timed(fn, reps=20):
    for _ in range(3):
        fn()
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(reps):
        fn()
    b.record()
    torch.cuda.synchronize()
    return a.elapsed_time(b) / reps


def main():
    out = {}
    for kind, nbytes in (("h2d", 21 * 2**20), ("d2h", 17 * 2**20)):
        h = torch.empty(nbytes, dtype=torch.uint8, pin_memory=True)
        h.fill_(1)
        d = torch.empty(nbytes, dtype=torch.uint8, device="cuda")
        for ns in (1, 2, 4):
            streams = [torch.cuda.Stream() for _ in range(ns)]
            chunk = nbytes // ns
            main_s = torch.cuda.current_stream()

            def fn():
                ev = torch.cuda.Event()
                ev.record(main_s)
                for k, s in enumerate(streams):
                    s.wait_event(ev)
                    with torch.cuda.stream(s):
                        sl = slice(k * chunk, (k + 1) * chunk)
                        if kind == "h2d":
                            d[sl].copy_(h[sl], non_blocking=True)
                        else:
                            h[sl].copy_(d[sl], non_blocking=True)
                for s in streams:
                    main_s.wait_stream(s)
            ms = timed(fn)
            out[f"{kind}_{ns}streams_GBps"] = nbytes / (ms * 1e-3) / 1e9
    json.dump(out, sys.stdout)
    print()


if __name__ == "__main__":
    main()
