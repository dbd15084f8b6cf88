#!/usr/bin/env python3
"""Dev tool: attribute ncu warp-stall samples of one kernel to CUDA source
lines. ncu's CSV source page has per-SASS-instruction samples; nvdisasm -g
on the binary's cubin maps instruction offsets to file:line.

  python scripts/ncu_lines.py <report.ncu-rep> <binary-or-.so> [kernel-substring] [top]
"""
import collections
import csv
import glob
import io
import os
import re
import subprocess
import sys
import tempfile


def sass_samples(rep, kernel_sub):
    out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"],
                         capture_output=True, text=True).stdout
    blocks, cur = [], None
    for row in csv.reader(io.StringIO(out)):
        if row and row[0] == "Kernel Name":
            cur = {"name": row[1], "rows": []}
            blocks.append(cur)
        elif row and row[0] == "Address":
            cur["hdr"] = row
        elif cur is not None and row:
            cur["rows"].append(row)
    blocks = [b for b in blocks if kernel_sub in b["name"]]
    if not blocks:
        sys.exit(f"no kernel matching {kernel_sub!r}")
    b = blocks[0]
    h = b["hdr"]
    ia, isrc, iss = h.index("Address"), h.index("Source"), h.index("Warp Stall Sampling (All Samples)")
    base = int(b["rows"][0][ia], 16)
    return b["name"], [(int(r[ia], 16) - base, r[isrc].strip(), float(r[iss] or 0)) for r in b["rows"]]


def line_maps(binary):
    d = tempfile.mkdtemp()
    subprocess.run(["cuobjdump", "-xelf", "all", os.path.abspath(binary)], cwd=d, capture_output=True)
    funcs = {}
    for cub in glob.glob(os.path.join(d, "*.cubin")):
        txt = subprocess.run(["nvdisasm", "-g", "-c", cub], capture_output=True, text=True).stdout
        fn, loc = None, None
        for line in txt.splitlines():
            m = re.match(r"\s*\.text\.(\S+):", line)
            if m:
                fn, loc = m.group(1), None
                funcs[fn] = {}
                continue
            m = re.search(r'//## File "([^"]+)", line (\d+)', line)
            if m:
                loc = (os.path.basename(m.group(1)), int(m.group(2)))
                continue
            m = re.match(r"\s*/\*([0-9a-f]{4,})\*/\s+(.*?)\s*;", line)
            if m and fn:
                funcs[fn][int(m.group(1), 16)] = (loc, m.group(2))
    return funcs


def main():
    rep, binary = sys.argv[1], sys.argv[2]
    sub = sys.argv[3] if len(sys.argv) > 3 else ""
    top = int(sys.argv[4]) if len(sys.argv) > 4 else 40
    name, samples = sass_samples(rep, sub)
    funcs = line_maps(binary)
    n = len(samples)
    # the function with the same (normalised) demangled name, else the same
    # instruction count
    def norm(x):
        x = re.sub(r"\((int|bool|unsigned int)\)", "", x).replace("false", "0").replace("true", "1")
        return re.sub(r"\s+", "", x.split("(bcad_dev::")[0].split("(const")[0])
    names = list(funcs)
    dem = subprocess.run(["cu++filt"], input="\n".join(names), capture_output=True, text=True).stdout.splitlines()
    want = norm(name)
    cands = [f for f, dm in zip(names, dem) if norm(dm) == want and len(funcs[f]) == n]
    if not cands:
        cands = [f for f, m in funcs.items() if len(m) == n]
    if not cands:
        sys.exit(f"no function with {n} instructions in {binary}")
    fmap = funcs[cands[0]]
    offs = sorted(fmap)
    total = sum(s for _, _, s in samples) or 1.0
    by_line = collections.Counter()
    for k, (_, _, s) in enumerate(samples):
        loc = fmap[offs[k]][0] if k < len(offs) else None
        by_line[loc] += s
    print(f"{name[:120]}\n{int(total)} samples, {n} instructions ({len(cands)} candidate function(s))")
    for loc, s in by_line.most_common(top):
        print(f"{s / total * 100:6.1f}%  {loc}")


if __name__ == "__main__":
    main()
