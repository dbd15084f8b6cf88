"""Step throughput vs batch size (run under gpurun): the canonical fp32 HM-LSTM
step (K1 + K2, CacheForward) at H = 1024 for B = 64 ... 65536, L2 flushed
between steps, timed with CUDA events. Shows where per-launch fixed costs
stop mattering: the HBM fraction of the step against the measured copy peak."""
import json
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from bench import hbm_peak, measure_secondary  # noqa: E402
from paper_1810_08297_b200.workloads import Workload  # noqa: E402

dev = torch.device("cuda", 0)
stream = torch.cuda.Stream(dev)
peak, _ = hbm_peak()
rows = []
for variant, kern in (("canonical", "hmlstm_update"), ("bias", "hmlstm_update_bias")):
    for B in (64, 256, 1024, 4096, 16384, 65536):
        w = Workload("sweep", B, 1024, "f32", variant, f"{variant} fp32 B={B} H=1024")
        r = measure_secondary(w, dev, stream, 15, 0)
        rows.append({"variant": variant, "B": B, "H": 1024, "step_us": r["ms_per_step"] * 1e3,
                     "step_bytes_MB": w.step_bytes() / 1e6, "step_frac_hbm": r["step_frac_hbm"],
                     "K1_frac": r["K1_frac_hbm"], "K2_frac": r["K2_frac_hbm"], "grad_elems_per_s": r["value"]})
        print(json.dumps(rows[-1]), flush=True)
