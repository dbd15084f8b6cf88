"""Probe (GPU): how far the device's reduced (1,H) adjoints sit from the
oracle's fp64-accumulated sums, and why. Per bias argument: bitwise
differing partials device vs oracle, worst relative error of the reduced
adjoint vs the oracle's fp64 sum (S_orc) and vs the fp64 sum of the
device's own rounded terms (S_dev), and the term-discrepancy bound
sum_k |t_dev - t_orc|."""
import json
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path[:0] = [ROOT, os.path.join(ROOT, "tests")]
import oracle as O  # noqa: E402
from helpers import GpuRunner  # noqa: E402

orc = O.Oracle()
gpu = GpuRunner("cuda:0")
out = []
for dtype, B, H, seedkind in [(np.float32, 1024, 1024, "ones"), (np.float32, 1024, 1024, "pm1"),
                              (np.float32, 16384, 1024, "pm1"), (np.float64, 1024, 512, "pm1")]:
    ins = O.hmlstm_inputs(orc, B, H, dtype, "bias")
    seed = np.ones((B, H), dtype) if seedkind == "ones" else \
        np.random.default_rng(3).uniform(-1, 1, (B, H)).astype(dtype)
    _, pd = orc.forward("hmlstm_update_bias", ins)
    _, want, want64 = orc.mixed_step("hmlstm_update_bias", ins, seeds=[seed])
    _, gparts, got = gpu.step("hmlstm_update_bias", ins, seeds=[seed])
    rec = {"dtype": np.dtype(dtype).name, "B": B, "H": H, "seed": seedkind}
    for j in (4, 5, 6):
        t_orc = (seed * pd[j]).astype(dtype)
        t_dev = (seed * gparts[j]).astype(dtype)
        s_orc = t_orc.astype(np.float64).sum(0)
        s_dev = t_dev.astype(np.float64).sum(0)
        g = got[j].ravel().astype(np.float64)
        slack = np.abs(t_dev.astype(np.float64) - t_orc.astype(np.float64)).sum(0)
        rel = lambda a, b: float(np.max(np.abs(a - b) / np.maximum(np.abs(b), 1e-300)))  # noqa: E731
        rec[f"arg{j}"] = {"partials_bitdiff_frac": float(np.mean(pd[j] != gparts[j])),
                          "max_partial_ulps": float(np.max(np.abs(pd[j].astype(np.float64) - gparts[j]) /
                                                           np.maximum(np.spacing(np.abs(pd[j])), 1e-300))),
                          "rel_vs_orc64": rel(g, s_orc), "rel_vs_dev64": rel(g, s_dev),
                          "acc64_matches_S_orc": float(np.max(np.abs(want64[j].ravel() - s_orc))),
                          "n_fail_rel1e-6_vs_orc": int(np.sum(np.abs(g - s_orc) > 1e-6 * np.abs(s_orc))),
                          "n_fail_rel1e-6_plus_slack": int(np.sum(np.abs(g - s_orc) > 1e-6 * np.abs(s_orc) + slack)),
                          "old_comparator_abs": 1e-6 * np.sqrt(B)}
    out.append(rec)
    print(json.dumps(rec), flush=True)
