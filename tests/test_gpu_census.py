"""Device transcendental census (bcad_cu_eval_counters; kernels.cuh census_kernel):
the kernels count exp / log / sin / cos / tanh / sigmoid evaluations like the
reference's counting wrappers (dual.hpp:55-60, 280-320) — per cell and per
branch taken: UPDATE 3, FLUSH 2, COPY 0 for cell_update_scalar
(hmlstm.hpp:49-54), on the canonical lane-vector path ((B) boundary bits) and
per cell on the branch-free select form ((B,H) bits: every cell evaluates all
three), for the dual forward (K1), the primal-only forward (K1p) and the
RecomputeReverse pullback (K2r), and the cached pullback evaluates nothing."""
import numpy as np
import pytest

pytestmark = pytest.mark.gpu

B, H = 64, 256  # 16384 cells


def _delta(native, fn):
    before = native.transcendental_evals()
    fn()
    return native.transcendental_evals() - before


@pytest.mark.parametrize("case,per_cell", [("copy", 0), ("update", 3), ("flush", 2)])
def test_counts_per_boundary_case(case, per_cell):
    import torch
    from paper_1810_08297_b200 import native
    k = native.Kernel("hmlstm_update")
    z1v, z2v = {"copy": (0.0, 0.0), "update": (0.0, 1.0), "flush": (1.0, 0.0)}[case]
    ins = [torch.rand((B, H), device="cuda") * 2 - 1 for _ in range(4)]
    ins += [torch.full((B,), z1v, device="cuda"), torch.full((B,), z2v, device="cuda")]
    prim = [torch.empty((B, H), device="cuda")]
    parts = [torch.empty((B, H), device="cuda") for _ in range(6)]
    native.transcendental_evals()  # arm
    assert _delta(native, lambda: native.forward(k, ins, prim, parts)) == per_cell * B * H  # K1
    assert _delta(native, lambda: native.forward(k, ins, prim, None)) == per_cell * B * H  # K1p
    shapes = [tuple(t.shape) for t in ins]
    seed = [torch.ones((B, H), device="cuda")]
    adj = [torch.empty(s, device="cuda") for s in shapes]
    ws = native.new_workspace(k, shapes, torch.float32)
    assert _delta(native, lambda: native.pullback(k, shapes, seed, parts, ins, adj, workspace=ws)) == 0  # K2
    assert _delta(native, lambda: native.pullback(k, shapes, seed, None, ins, adj, workspace=ws)) == \
        per_cell * B * H  # K2r re-derives the partials


def test_per_cell_bits_take_the_select_form_and_count_three():
    import torch
    from paper_1810_08297_b200 import native
    k = native.Kernel("hmlstm_update")
    g = torch.Generator(device="cuda")
    g.manual_seed(5)
    ins = [torch.rand((B, H), device="cuda", generator=g) * 2 - 1 for _ in range(4)]
    ins += [(torch.rand((B, H), device="cuda", generator=g) < 0.5).float() for _ in range(2)]
    prim = [torch.empty((B, H), device="cuda")]
    parts = [torch.empty((B, H), device="cuda") for _ in range(6)]
    native.transcendental_evals()
    assert _delta(native, lambda: native.forward(k, ins, prim, parts)) == 3 * B * H


def test_arity_and_generic_paths():
    import torch
    from paper_1810_08297_b200 import native
    native.transcendental_evals()
    for A in (1, 5, 16):
        k = native.Kernel(f"tanh_product_{A}")
        ins = [torch.rand((B, H), device="cuda") for _ in range(A)]
        prim = [torch.empty((B, H), device="cuda")]
        parts = [torch.empty((B, H), device="cuda") for _ in range(A)]
        assert _delta(native, lambda: native.forward(k, ins, prim, parts)) == A * B * H  # one tanh per input
    # rank-3 shapes: the generic kernels count too
    k = native.Kernel("gate")  # sigmoid(x) * tanh(y) + x
    ins = [torch.rand((8, 16, 32), device="cuda"), torch.rand((8, 1, 32), device="cuda")]
    prim = [torch.empty((8, 16, 32), device="cuda")]
    parts = [torch.empty((8, 16, 32), device="cuda") for _ in range(2)]
    assert _delta(native, lambda: native.forward(k, ins, prim, parts)) == 2 * 8 * 16 * 32
    assert np.isfinite(prim[0].cpu().numpy()).all()
