"""tanh_product_A forward at 4096 x 4096 fp32 (bench.py extra.arity), a few
launches per arity, for ncu captures: python scripts/arity_probe.py 16 32"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_1810_08297_b200 import native  # noqa: E402

n = 4096
for A in [int(a) for a in sys.argv[1:]] or [16, 32]:
    k = native.Kernel(f"tanh_product_{A}")
    ins = [torch.rand((n, n), device="cuda") * 2 - 1 for _ in range(A)]
    prim = [torch.empty((n, n), device="cuda")]
    parts = [torch.empty((n, n), device="cuda") for _ in range(A)]
    for _ in range(3):
        native.forward(k, ins, prim, parts)
    torch.cuda.synchronize()
    del ins, parts
print("ok")
