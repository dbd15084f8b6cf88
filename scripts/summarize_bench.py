"""Print the key numbers of a bench JSON line (dev helper)."""
import json
import sys

d = json.load(open(sys.argv[1]))
print("value %.4g cells/s  ms/step %.4f  step frac %.3f" % (d["value"], d["ms_per_step"], d["step_roofline"]["frac"]))
print("breakdown", {k: round(v, 4) for k, v in d["breakdown_ms"].items()})
print("roofline", {k: d["roofline"][k] for k in ("kernel", "achieved", "frac", "traffic")})
print("e2e", {k: (round(v, 4) if isinstance(v, float) else v) for k, v in d["e2e"].items()})
print("clocks", d["clocks"], "cpu", {k: d.get("cpu_baseline", {}).get(k) for k in ("value", "cores", "kind")})
for k, v in d.get("extra", {}).items():
    print(k, {a: (round(b, 4) if isinstance(b, float) else b) for a, b in v.items() if a not in ("workload", "unit")})
