"""Summarise ncu evidence into profiles/ (run here, on the reports gpurun
brought back). Writes profiles/<round>/ncu_summary.md, the launch-list
shares, and profiles/ncu_traffic.json (per-launch DRAM traffic of K1/K2 that
bench.py reports as roofline.traffic).

  python scripts/ncu_summary.py gpurun_out/prof r01
"""
import csv
import io
import json
import os
import subprocess
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1810_08297_b200.workloads import WORKLOADS  # noqa: E402

METRICS = {
    "gpu__time_duration.sum": "duration_us",
    "dram__bytes_read.sum": "dram_read",
    "dram__bytes_write.sum": "dram_write",
    "launch__registers_per_thread": "regs",
    "launch__grid_size": "grid",
    "sm__warps_active.avg.pct_of_peak_sustained_active": "occupancy_pct",
    "smsp__inst_executed.sum": "warp_inst",
    "sm__inst_executed.avg.per_cycle_active": "ipc",
    "dram__throughput.avg.pct_of_peak_sustained_elapsed": "dram_pct_peak",
    "sm__cycles_active.avg": "sm_active_cycles",
    "sm__cycles_elapsed.avg": "sm_elapsed_cycles",
    "lts__t_sectors_srcunit_tex_op_read_lookup_hit.sum": "l2_read_hit_sectors",
    "lts__t_sectors_srcunit_tex_op_read.sum": "l2_read_sectors",
}

UNIT_SCALE = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "nsecond": 1e-3, "usecond": 1, "msecond": 1e3,
              "ns": 1e-3, "us": 1, "ms": 1e3}


def raw(report):
    if report.endswith(".csv.gz"):  # raw page exported on the GPU box (scripts/gpu_profile.sh)
        import gzip
        out = gzip.open(report, "rt").read()
    else:
        out = subprocess.run(["ncu", "-i", report, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    head, units = rows[0], rows[1]
    res = []
    for r in rows[2:]:
        d = {}
        for k, u, v in zip(head, units, r):
            if k in METRICS:
                try:
                    x = float(v.replace(",", ""))
                except ValueError:
                    continue
                d[METRICS[k]] = x * UNIT_SCALE.get(u, 1)
        name = r[head.index("Kernel Name")]
        d["kernel"] = ("K1_forward" if "fwd2d" in name else "K2_pullback" if "pull2d" in name
                       else "K2f_finish" if "pull_finish" in name else name[:40])
        d["name"] = name.split("(")[0][:110]
        res.append(d)
    return res


def launch_shares(path):
    rows = [r for r in csv.reader(open(path)) if r and not r[0].startswith("==")]
    head = rows[0]
    ki, mi, vi, ui = head.index("Kernel Name"), head.index("Metric Name"), head.index("Metric Value"), head.index("Metric Unit")
    per = {}
    for r in rows[1:]:
        if r[mi] != "gpu__time_duration.sum":
            continue
        name = r[ki]
        key = ("K1 fwd2d" if "fwd2d" in name else "K2 pull2d" if "pull2d" in name else "K2f pull_finish"
               if "pull_finish" in name else ("nccl" if "nccl" in name.lower() else "other (torch flush/fill/copy)"))
        t = float(r[vi].replace(",", "")) * UNIT_SCALE.get(r[ui], 1)
        per.setdefault(key, []).append(t)
    return per


def main():
    src, rnd = sys.argv[1], sys.argv[2]
    dst = os.path.join("profiles", rnd)
    os.makedirs(dst, exist_ok=True)
    lines = [f"# ncu summary ({rnd})", "",
             "Captured with `scripts/gpu_profile.sh` under gpurun on one B200: `ncu --set full --clock-control none "
             "--import-source on -k regex:\"fwd2d|pull2d\"` on `bench.py --config <cfg>` (cold caches: ncu flushes "
             "between replays, so K2 reads its cached partials from DRAM here while in the timed bench they are still "
             "L2-resident after K1 at config 2). Algorithmic bytes per launch are SURVEY §8(d)'s reference-faithful "
             "counts (paper_1810_08297_b200/workloads.py); peak = MEASURED_PEAKS.json hbm_gbs of this container.", ""]
    traffic = {}
    peak = 6538.0
    try:
        peak = float(json.load(open("MEASURED_PEAKS.json"))["hbm_gbs"])
    except Exception:
        pass
    for cfg in ("cfg2", "cfg3", "cfg5", "cfg4div"):
        rep = os.path.join(src, f"full_{cfg}.ncu-rep")
        if not os.path.exists(rep):
            rep = os.path.join(src, f"full_{cfg}.raw.csv.gz")
        if not os.path.exists(rep):
            continue
        w = WORKLOADS[cfg]
        lines += [f"## {cfg}: {w.describe}", "",
                  "| kernel | regs | grid | occ % | warp inst | IPC | SM active/elapsed | dur µs | DRAM read MB | DRAM write MB | algorithmic MB | alg GB/s | frac of peak |",
                  "|---|---|---|---|---|---|---|---|---|---|---|---|---|"]
        seen = set()
        for d in raw(rep):
            if d["kernel"] in seen:
                continue
            seen.add(d["kernel"])
            if d["kernel"] == "K2f_finish":  # reads the fp64 tile partials, writes the reduced adjoints
                alg = d.get("dram_read", 0) + d.get("dram_write", 0)
            else:
                alg = w.k1_bytes() if d["kernel"] == "K1_forward" else w.k2_bytes()
            dur = d.get("duration_us", float("nan"))
            gbs = alg / (dur * 1e-6) / 1e9
            act = d.get("sm_active_cycles", 0) / max(1, d.get("sm_elapsed_cycles", 1))
            lines.append(f"| {d['kernel']} | {d.get('regs', 0):.0f} | {d.get('grid', 0):.0f} | {d.get('occupancy_pct', 0):.1f} | "
                         f"{d.get('warp_inst', 0):.3g} | {d.get('ipc', 0):.2f} | {act:.2f} | {dur:.1f} | "
                         f"{d.get('dram_read', 0) / 1e6:.1f} | {d.get('dram_write', 0) / 1e6:.1f} | {alg / 1e6:.1f} | "
                         f"{gbs:.0f} | {gbs / peak:.2f} |")
            traffic.setdefault(cfg, {})[d["kernel"]] = d.get("dram_read", 0) + d.get("dram_write", 0)
        lines.append("")
    for cfg in ("cfg2", "cfg5"):
        p = os.path.join(src, f"launches_{cfg}.csv")
        if not os.path.exists(p):
            continue
        per = launch_shares(p)
        tot = sum(sum(v) for v in per.values())
        lines += [f"### launch list, `bench.py --config {cfg}` (ncu --metrics gpu__time_duration.sum, serialised)", "",
                  "| kernel group | launches | mean µs | share of listed time |", "|---|---|---|---|"]
        for k, v in sorted(per.items()):
            lines.append(f"| {k} | {len(v)} | {sum(v) / len(v):.1f} | {sum(v) / tot:.1%} |")
        lines.append("")
    open(os.path.join(dst, "ncu_summary.md"), "w").write("\n".join(lines) + "\n")
    json.dump(traffic, open(os.path.join("profiles", "ncu_traffic.json"), "w"), indent=1)
    print("\n".join(lines))


if __name__ == "__main__":
    main()
