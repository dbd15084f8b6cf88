"""One config-5 RecomputeReverse step (K1p then K2r, bias variant 65536 x
4096 fp32) through the C-ABI, repeated, for ncu captures of K2r:
  ncu -k regex:pull2d -s 1 -c 1 python scripts/k2r_probe.py [B] [H]"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_1810_08297_b200 import native  # noqa: E402

B = int(sys.argv[1]) if len(sys.argv) > 1 else 65536
H = int(sys.argv[2]) if len(sys.argv) > 2 else 4096
k = native.Kernel("hmlstm_update_bias")
shapes = [(B, H)] * 4 + [(1, H)] * 3 + [(B,)] * 2
g = torch.Generator(device="cuda")
g.manual_seed(3)
ins = [torch.rand(s, generator=g, device="cuda") * 2 - 1 for s in shapes[:7]]
ins += [(torch.rand((B,), generator=g, device="cuda") < 0.5).float() for _ in range(2)]
prim = [torch.empty((B, H), device="cuda")]
seed = [torch.ones((B, H), device="cuda")]
adj = [torch.empty(s, device="cuda") for s in shapes]
ws = native.new_workspace(k, shapes, torch.float32)
for _ in range(3):
    native.forward(k, ins, prim, None)
    native.pullback(k, shapes, seed, None, ins, adj, workspace=ws)
torch.cuda.synchronize()
print("ok")
