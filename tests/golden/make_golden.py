"""Generate the golden vectors in tests/golden/ from the UNMODIFIED reference.

Runs in the build container only (needs oracle/_ref/libbcad_ref.so, which
oracle/Makefile compiles from /root/reference). Each fixture holds the inputs
and the reference's own outputs of one mixed step — primal(s), the M*N
cached Jacobian diagonals (broadcast_diag_jacobian, proj/include/bcad/
forward.hpp:98-150) and the leaf gradients of Tape::backward with the given
seeds (proj/include/bcad/tape.hpp:185-211, serial scatter_add order).

    python tests/golden/make_golden.py
"""
import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(os.path.dirname(HERE))
sys.path.insert(0, ROOT)

import oracle as O  # noqa: E402


def random_shapes(rng, n_args, max_rank=3, max_len=4):
    rank = 1 + int(rng.integers(0, max_rank))
    out = [1 + int(rng.integers(0, max_len)) for _ in range(rank)]
    shapes = []
    for _ in range(n_args):
        keep = int(rng.integers(0, rank + 1)) if rng.integers(0, 4) == 0 else rank
        shapes.append(tuple(1 if rng.integers(0, 3) == 0 else out[k] for k in range(keep)))
    return shapes


def save(name, kernel, ins, seeds, ref, policy=O.CACHE_FORWARD):
    prim, parts = ref.forward(kernel, ins)
    p2, grads, peak = ref.mixed_step(kernel, ins, policy, seeds)
    assert all(np.array_equal(a, b) for a, b in zip(prim, p2))
    d = {"kernel": np.array(kernel), "n_in": np.array(len(ins)), "m_out": np.array(len(prim)),
         "peak_cached_bytes": np.array(peak)}
    for j, a in enumerate(ins):
        d[f"in{j}"] = a
    for i, s in enumerate(seeds):
        if s is not None:
            d[f"seed{i}"] = s
    for i, p in enumerate(prim):
        d[f"primal{i}"] = p
    for k, p in enumerate(parts):
        d[f"partial{k}"] = p
    for j, g in enumerate(grads):
        d[f"grad{j}"] = g
    np.savez_compressed(os.path.join(HERE, name + ".npz"), **d)


def main():
    ref = O.Reference()
    # HM-LSTM: config 1 (B=32, H=256) canonical fp32 + bias / divergence
    # variants, fp64 at a smaller size. Inputs drawn exactly as SURVEY §8(d):
    # Rng(mix_seed(42, B*1000003 + H)), order c, f, i, g, [bf, bi, bg], z1, z2.
    for (B, H, dt, variant) in [(32, 256, np.float32, "canonical"), (16, 64, np.float64, "canonical"),
                                (16, 128, np.float32, "bias"), (16, 64, np.float64, "bias"),
                                (8, 64, np.float32, "divergence")]:
        ins = O.hmlstm_inputs(ref, B, H, dt, variant)
        seeds = [np.ones((B, H), dt)]
        save(f"hmlstm_{variant}_{np.dtype(dt).name}_{B}x{H}", O.hmlstm_kernel(variant), ins, seeds, ref)
    # random adjoint seed through the bias variant (reductions of signed terms)
    rng = np.random.default_rng(2)
    ins = O.hmlstm_inputs(ref, 24, 64, np.float32, "bias")
    save("hmlstm_bias_float32_24x64_randseed", "hmlstm_update_bias", ins,
         [rng.uniform(-1, 1, (24, 64)).astype(np.float32)], ref)
    # Kernel pool on random broadcast shapes (tests/support/kernel_pool.hpp)
    rng = np.random.default_rng(11)
    pool = ["identity", "reflect", "tanh_sigmoid", "product", "gated", "prod_diff", "blend", "curl",
            "tanh_product_4", "hmlstm_update", "fanout", "fiveway", "wave", "two", "gate", "square_gate"]
    for name in pool:
        n, m = O.Oracle().arity(name)
        for rep in range(2):
            shapes = random_shapes(rng, n)
            dt = np.float64 if rep == 0 else np.float32
            ins = [rng.uniform(-1, 1, s).astype(dt) for s in shapes]
            if name == "hmlstm_update":
                for z in (4, 5):
                    ins[z] = (rng.uniform(0, 1, shapes[z]) < 0.5).astype(dt)
            out = O.broadcast_shape_py(shapes)
            seeds = [rng.uniform(-1, 1, out).astype(dt) for _ in range(m)]
            save(f"pool_{name}_{rep}", name, ins, seeds, ref)
    print("golden fixtures written to", HERE)


if __name__ == "__main__":
    main()
