"""Dev probe: does the host NUMA node of the pinned buffers change PCIe
bandwidth? Prints the GPU's PCI NUMA node / local CPUs, then pinned H2D and
D2H GB/s of a 21 MB transfer (config 2's step inputs) with the process bound
to each NUMA node's CPUs (buffers allocated after binding: first touch)."""
import glob
import json
import os
import sys

import torch


def gpu_sysfs():
    import pynvml
    pynvml.nvmlInit()
    h = pynvml.nvmlDeviceGetHandleByIndex(0)
    bus = pynvml.nvmlDeviceGetPciInfo(h).busId
    bus = bus.decode() if isinstance(bus, bytes) else bus
    bus = bus.lower()
    # nvml gives 8 hex digits of domain; sysfs uses 4
    dom, rest = bus.split(":", 1)
    path = f"/sys/bus/pci/devices/{dom[-4:]}:{rest}"
    def rd(name):
        try:
            return open(os.path.join(path, name)).read().strip()
        except OSError:
            return None
    return {"bus": bus, "numa_node": rd("numa_node"), "local_cpulist": rd("local_cpulist")}


def parse_cpulist(s):
    out = []
    for part in s.split(","):
        if "-" in part:
            a, b = part.split("-")
            out += list(range(int(a), int(b) + 1))
        elif part:
            out.append(int(part))
    return out


def bw(nbytes=21 * 2**20, reps=20):
    h = torch.empty(nbytes, dtype=torch.uint8, pin_memory=True)
    h.fill_(1)
    d = torch.empty(nbytes, dtype=torch.uint8, device="cuda")
    s = torch.cuda.Stream()
    out = {}
    for name, fn in (("h2d", lambda: d.copy_(h, non_blocking=True)), ("d2h", lambda: h.copy_(d, non_blocking=True))):
        with torch.cuda.stream(s):
            for _ in range(3):
                fn()
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a.record(s)
            for _ in range(reps):
                fn()
            b.record(s)
        s.synchronize()
        out[name] = nbytes * reps / (a.elapsed_time(b) * 1e-3) / 1e9
    return out


def main():
    info = gpu_sysfs()
    nodes = {}
    for p in sorted(glob.glob("/sys/devices/system/node/node*/cpulist")):
        nodes[os.path.basename(os.path.dirname(p))] = open(p).read().strip()
    res = {"gpu": info, "nodes": nodes, "all_cpus": bw()}
    for node, cl in nodes.items():
        cpus = parse_cpulist(cl)
        if not cpus:
            continue
        os.sched_setaffinity(0, cpus)
        res[node] = bw()
    json.dump(res, sys.stdout)
    print()


if __name__ == "__main__":
    main()
