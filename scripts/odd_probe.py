import json, sys, os, torch
sys.path.insert(0, os.getcwd())
from bench import Case, measure_secondary
from paper_1810_08297_b200.workloads import Workload
dev = torch.device("cuda", 0); st = torch.cuda.Stream(dev)
out = {}
for H in (1024, 1023, 1026):
    for variant in ("canonical", "bias"):
        w = Workload("odd", 8192, H, "f32", variant, f"{variant} 8192x{H}")
        r = measure_secondary(w, dev, st, 5, 0)
        out[f"{variant}_H{H}"] = {"K1_ms": r["K1_ms"], "K2_ms": r["K2_ms"], "step_frac": r["step_frac_hbm"]}
print(json.dumps(out, indent=1))
