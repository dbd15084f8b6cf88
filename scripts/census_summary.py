"""Summarise gpurun_out/census (scripts/gpu_census.sh) into a markdown table:
executed MUFU (XU-pipe transcendental) thread instructions per output cell of
K1, by SASS opcode, per boundary case and body form."""
import csv
import gzip
import io
import os
import re
import sys
from collections import Counter

D = sys.argv[1] if len(sys.argv) > 1 else "gpurun_out/census"
CELLS = 1024 * 1024
rows = []
for form in ("canonical", "select"):
    for case in ("copy", "update", "flush", "random"):
        p = os.path.join(D, f"k1_{form}_{case}.sass.csv.gz")
        if not os.path.exists(p):
            continue
        lines = gzip.open(p, "rt").read().splitlines()
        r = list(csv.reader(io.StringIO("\n".join(lines[1:]))))
        h = r[0]
        src, thr = h.index("Source"), h.index("Predicated-On Thread Instructions Executed")
        mufu, total = Counter(), 0
        for row in r[1:]:
            try:
                n = int(row[thr])
            except ValueError:
                continue
            total += n
            m = re.match(r"\s*(@!?U?P\w+\s+)?MUFU\.(\w+)", row[src])
            if m:
                mufu[m.group(2)] += n
        rows.append((form, case, {k: v / CELLS for k, v in sorted(mufu.items())}, sum(mufu.values()) / CELLS,
                     total / CELLS))
print("| body form | boundary case | MUFU per cell (by op) | MUFU per cell | thread instructions per cell |")
print("|---|---|---|---|---|")
for form, case, by, m, t in rows:
    ops = ", ".join(f"{k} {v:.2f}" for k, v in by.items()) or "—"
    print(f"| {form} | {case} | {ops} | {m:.2f} | {t:.1f} |")
