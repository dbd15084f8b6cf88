"""The drop-in boundary on CPU: the C-ABI libraries load, export every symbol
their headers declare, and their host-side logic (registry, arity rules,
first-axis broadcast, error mapping, workspace sizing) behaves like the
reference without touching a GPU."""
import ctypes as C
import os
import re
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
PKG = os.path.join(ROOT, "paper_1810_08297_b200")


def declared(header):
    text = open(os.path.join(ROOT, "include", header)).read()
    text = re.sub(r"/\*.*?\*/", "", text, flags=re.S)
    return sorted(set(re.findall(r"\b(bcad_(?:cu|host)_\w+)\s*\(", text)))


def exported(so):
    out = subprocess.run(["nm", "-D", "--defined-only", so], capture_output=True, text=True, check=True).stdout
    return {line.split()[-1] for line in out.splitlines() if line.strip()}


@pytest.mark.parametrize("header,so", [("bcad_cu.h", "libbcad_cu.so"), ("bcad_host.h", "libbcad_host.so")])
def test_library_exports_every_declared_symbol(header, so):
    path = os.path.join(PKG, so)
    assert os.path.exists(path), f"{so} not built"
    C.CDLL(path)  # loads without a GPU
    names = declared(header)
    assert len(names) >= (25 if header == "bcad_cu.h" else 2)
    missing = [n for n in names if n not in exported(path)]
    assert not missing, missing


def test_python_binding_covers_the_header():
    from paper_1810_08297_b200 import native
    assert set(declared("bcad_cu.h")) == set(native.PROTOS)


def test_registry_and_arity_rules():
    from paper_1810_08297_b200 import native
    names = native.kernel_names()
    assert len(names) == len(set(names)), "every registered name binds exactly one body"
    for required in ("hmlstm_update", "hmlstm_update_bias", "identity", "mul", "tanh_product_32", "sigmoid_bwd",
                     "tanh_product_3", "tanh_product_5"):
        assert required in names
    k = native.Kernel("hmlstm_update")
    assert (k.n_in, k.m_out, k.may_raise) == (6, 1, False)
    assert native.Kernel("log").may_raise
    with pytest.raises(native.UnknownPrimitive):
        native.Kernel("does_not_exist", 1, 1)
    with pytest.raises(native.ArityMismatch):
        native.Kernel("hmlstm_update", 5, 1)
    with pytest.raises(native.ArityMismatch):  # kernel.hpp:30-35 range
        native.Kernel("identity", 33, 1)
    with pytest.raises(native.ArityMismatch):
        native.Kernel("identity", 1, 9)


def test_first_axis_broadcast_shape():
    from paper_1810_08297_b200 import native
    import oracle as O
    cases = [[(4, 3), (4,)], [(4, 3), (1, 3)], [(), (2, 5)], [(2, 1, 3), (2, 4)], [(1,), (1, 1)], [(7,), (7, 1, 2)]]
    for shapes in cases:
        assert native.broadcast_shape(shapes) == O.broadcast_shape_py(shapes)
    with pytest.raises(native.ShapeMismatch):
        native.broadcast_shape([(2, 3), (4, 3)])
    with pytest.raises(native.ShapeMismatch):
        native.broadcast_shape([(0, 3)])


def test_workspace_sizing_is_host_only():
    from paper_1810_08297_b200 import native
    kb = native.Kernel("hmlstm_update_bias")
    small = native.pullback_workspace(kb, [(32, 256)] * 4 + [(1, 256)] * 3 + [(32,)] * 2, native.F32)
    big = native.pullback_workspace(kb, [(65536, 4096)] * 4 + [(1, 4096)] * 3 + [(65536,)] * 2, native.F32)
    step_bytes = (28 * 65536 * 4096 + 6 * 4096 + 4 * 65536) * 4
    assert 0 < small < big < 0.003 * step_bytes  # fp64 tile partials stay < 0.3% of the step's bytes
    # odd widths run the one-cell-per-thread tiled kernel: its (small) tile workspace
    odd = native.pullback_workspace(kb, [(7, 1023)] * 4 + [(1, 1023)] * 3 + [(7,)] * 2, native.F32)
    assert 256 <= odd < 1 << 20
    # three irreducible axis groups: the generic kernel, no tile workspace
    assert native.pullback_workspace(kb, [(4, 3, 8)] * 4 + [(1, 3, 8)] * 3 + [(4, 1, 8)] * 2, native.F32) == 256


def test_status_codes_match_reference_errors():
    """One status per proj/include/bcad/errors.hpp type, shared with the oracle."""
    from paper_1810_08297_b200 import native
    hdr = open(os.path.join(ROOT, "include", "bcad_cu.h")).read()
    codes = dict((m.group(1), int(m.group(2))) for m in re.finditer(r"BCAD_CU_(ERR_\w+|OK)\s*=\s*(\d+)", hdr))
    assert codes["ERR_TAG_MISMATCH"] == native.TagMismatch.code
    assert codes["ERR_DOMAIN"] == native.DomainError.code
    assert codes["ERR_SEED_SHAPE_MISMATCH"] == native.SeedShapeMismatch.code
    assert codes["ERR_UNKNOWN_PRIMITIVE"] == native.UnknownPrimitive.code
    assert len(codes) == 17  # OK + 13 reference error types + Error + CUDA + NCCL


def test_no_cpu_fallback_without_device():
    """Compute calls fail loudly (CUDA error) instead of silently running on CPU."""
    import numpy as np
    import torch
    if torch.cuda.is_available():
        pytest.skip("device present")
    from paper_1810_08297_b200 import native
    k = native.Kernel("mul")
    a = (C.c_double * 4)()
    ptrs = (C.c_void_p * 2)(C.addressof(a), C.addressof(a))
    shapes = (native.Shape * 2)(native.Shape.of((4,)), native.Shape.of((4,)))
    outs = (C.c_void_p * 1)(C.addressof(a))
    rc = native.LIB.bcad_cu_forward(k.handle, native.F64, 2, ptrs, shapes, 1, outs, None, None)
    assert rc == native.CudaError.code
    del np


def test_pullback_launch_count():
    from paper_1810_08297_b200 import native
    k = native.Kernel("hmlstm_update")
    kb = native.Kernel("hmlstm_update_bias")
    # config 2: (B)-reductions finish inside a CTA (one K2 launch)
    assert native.pullback_launches(k, [(1024, 1024)] * 4 + [(1024,)] * 2, native.F32) == 1
    # (1,H) reductions over 1024 rows span CTAs: K2 + the finisher K2f
    assert native.pullback_launches(kb, [(1024, 1024)] * 4 + [(1, 1024)] * 3 + [(1024,)] * 2, native.F32) == 2
    # generic rank-N (three irreducible axis groups): the full-shape argument's
    # elementwise kernel + a segmented reduction (segments + finisher)
    g = native.Kernel("mul")
    assert native.pullback_launches(g, [(64, 256, 1024), (64, 1, 1024)], native.F32) == 3
    assert native.pullback_launches(g, [(64, 256, 1024), (1, 256, 1)], native.F32) == 3
    # ... a small reduction (< 64 cells per element): thread per element
    assert native.pullback_launches(g, [(64, 8, 1024), (64, 1, 1024)], native.F32) == 2
