"""Device transcendental census (the device analogue of the reference's
untaken-branch accounting, proj/tests/test_hmlstm.cpp:185-220): one K1
forward of the HM-LSTM cell update at B x H = 1024 x 1024 fp32 with all
boundary bits set to one case, for ncu to count the executed MUFU (XU pipe)
instructions.

  python scripts/census.py <form> <case>
    form: canonical  (z1, z2 of shape (B): row-uniform, the branchy body on
                      lane vectors — one branch taken per row)
          select     (z1, z2 of shape (B, H): per-cell bits, the branch-free
                      select form that evaluates every gate and keeps one)
    case: copy | update | flush | random
"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_1810_08297_b200 import native  # noqa: E402

form, case = sys.argv[1], sys.argv[2]
B = H = 1024
zshape = (B,) if form == "canonical" else (B, H)
g = torch.Generator(device="cuda")
g.manual_seed(5)
c, f, i, gg = [torch.rand((B, H), generator=g, device="cuda") * 2 - 1 for _ in range(4)]
if case == "random":
    z1 = (torch.rand(zshape, generator=g, device="cuda") < 0.5).float()
    z2 = (torch.rand(zshape, generator=g, device="cuda") < 0.5).float()
else:
    bits = {"copy": (0.0, 0.0), "update": (0.0, 1.0), "flush": (1.0, 1.0)}[case]
    z1 = torch.full(zshape, bits[0], device="cuda")
    z2 = torch.full(zshape, bits[1], device="cuda")
k = native.Kernel("hmlstm_update")
prim = [torch.empty((B, H), device="cuda")]
parts = [torch.empty((B, H), device="cuda") for _ in range(6)]
native.forward(k, [c, f, i, gg, z1, z2], prim, parts)
torch.cuda.synchronize()
print("ok", form, case)
