"""ORACLE — TEST INFRASTRUCTURE ONLY.

ctypes front-end to the two CPU checkers built by ``oracle/Makefile``:

* ``liboracle.so``        — this repo's restatement of the reference algorithm
  (``oracle/oracle.cpp``; every function cites the reference file:line).
* ``_ref/libbcad_ref.so`` — the unmodified reference (``/root/reference/proj``)
  compiled from its own sources, driven through its public API
  (``oracle/ref_driver.cpp``).

Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s cpu_baseline /
``--impl reference`` legs may import this package, and only as the checker or
the timed CPU baseline — never as the product path.
"""
from __future__ import annotations

import ctypes as C
import os
from typing import Sequence

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ORACLE_SO = os.path.join(HERE, "liboracle.so")
REF_SO = os.path.join(HERE, "_ref", "libbcad_ref.so")

MAX_RANK = 8
CACHE_FORWARD, RECOMPUTE_REVERSE = 0, 1


class Shape(C.Structure):
    """Layout-compatible with ``bcad_cu_shape`` (include/bcad_cu.h)."""

    _fields_ = [("rank", C.c_int32), ("pad", C.c_int32), ("dims", C.c_int64 * MAX_RANK)]

    @classmethod
    def of(cls, dims: Sequence[int]) -> "Shape":
        s = cls()
        s.rank = len(dims)
        for k, d in enumerate(dims):
            s.dims[k] = int(d)
        return s

    def tuple(self) -> tuple:
        return tuple(int(self.dims[k]) for k in range(self.rank))


class OracleError(RuntimeError):
    def __init__(self, code: int, msg: str):
        super().__init__(f"[{code}] {msg}")
        self.code = code
        self.msg = msg


def _dt(dtype) -> int:
    return 0 if np.dtype(dtype) == np.float32 else 1


def _np_dtype(code: int):
    return np.float32 if code == 0 else np.float64


def _ptrs(arrays):
    arr = (C.c_void_p * max(1, len(arrays)))()
    for k, a in enumerate(arrays):
        arr[k] = None if a is None else a.ctypes.data
    return arr


def _shapes(shapes):
    arr = (Shape * max(1, len(shapes)))()
    for k, s in enumerate(shapes):
        arr[k] = Shape.of(s)
    return arr


def broadcast_shape_py(shapes: Sequence[Sequence[int]]) -> tuple:
    """First-axis aligned broadcast (proj/include/bcad/shape.hpp:70-90)."""
    rank = max((len(s) for s in shapes), default=0)
    out = []
    for k in range(rank):
        ln = 1
        for s in shapes:
            d = s[k] if k < len(s) else 1
            if d == 1:
                continue
            if ln == 1:
                ln = d
            elif d != ln:
                raise OracleError(5, f"broadcast shape mismatch at dim {k}")
        out.append(ln)
    return tuple(out)


class _Base:
    prefix = ""

    def __init__(self, path: str):
        if not os.path.exists(path):
            raise FileNotFoundError(f"{path} not built (run `make -C oracle`)")
        self.path = path
        self.lib = C.CDLL(path)
        self.lib.__getattr__(self.prefix + "last_error").restype = C.c_char_p

    def _fn(self, name):
        return getattr(self.lib, self.prefix + name)

    def _check(self, rc: int):
        if rc != 0:
            raise OracleError(rc, self._fn("last_error")().decode())

    def gen(self, seed: int, dtype, specs: Sequence[tuple]) -> list[np.ndarray]:
        """Draw tensors in order from one Rng(seed). specs: (shape, kind) with
        kind 'pm1' (random_pm1) or 'binary' (random_binary)."""
        outs = [np.empty(int(np.prod(s, dtype=np.int64)), dtype=dtype) for s, _ in specs]
        vols = (C.c_int64 * len(specs))(*[o.size for o in outs])
        kinds = (C.c_int * len(specs))(*[1 if k == "binary" else 0 for _, k in specs])
        f = self._fn("gen")
        f.argtypes = [C.c_uint64, C.c_int, C.c_int, C.c_void_p, C.c_void_p, C.c_void_p]
        self._check(f(C.c_uint64(seed), _dt(dtype), len(specs), vols, kinds, _ptrs(outs)))
        return [o.reshape(s) for o, (s, _) in zip(outs, specs)]

    def forward(self, name: str, inputs: Sequence[np.ndarray], want_primal=True, want_partials=True,
                real_body=False, m_out: int | None = None):
        """broadcast_diag_jacobian / broadcast_apply. Returns (primals, partials)
        with partials laid out [i*N + j] at the output shape."""
        dtype = inputs[0].dtype
        shapes = [a.shape for a in inputs]
        out_shape = broadcast_shape_py(shapes)
        n = len(inputs)
        m = m_out if m_out is not None else self.arity(name)[1]
        primals = [np.empty(out_shape, dtype) for _ in range(m)] if (want_primal or real_body) else None
        partials = ([np.empty(out_shape, dtype) for _ in range(m * n)]
                    if (want_partials and not real_body) else None)
        f = self._fn("forward")
        f.argtypes = [C.c_char_p, C.c_int, C.c_int, C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p, C.c_int]
        ins = [np.ascontiguousarray(a) for a in inputs]
        rc = f(name.encode(), _dt(dtype), n, _ptrs(ins), _shapes(shapes),
               _ptrs(primals) if primals is not None else None,
               _ptrs(partials) if partials is not None else None, int(real_body))
        self._check(rc)
        return primals, partials

    def arity(self, name: str) -> tuple[int, int]:
        raise NotImplementedError


class Oracle(_Base):
    """The repo's own restatement (liboracle.so)."""

    prefix = "oracle_"

    def __init__(self, path: str = ORACLE_SO):
        super().__init__(path)
        self.lib.oracle_kernel_name.restype = C.c_char_p
        self.lib.oracle_mix_seed.restype = C.c_uint64
        self.lib.oracle_mix_seed.argtypes = [C.c_uint64, C.c_uint64]

    def kernel_names(self) -> list[str]:
        return [self.lib.oracle_kernel_name(i).decode() for i in range(self.lib.oracle_kernel_count())]

    def arity(self, name: str) -> tuple[int, int]:
        n, m = C.c_int(), C.c_int()
        self._check(self.lib.oracle_kernel_info(name.encode(), C.byref(n), C.byref(m)))
        return n.value, m.value

    def mix_seed(self, seed: int, salt: int) -> int:
        return int(self.lib.oracle_mix_seed(seed, salt))

    def pullback(self, shapes, out_adj, partials, in_adj, accumulate=None, want_acc64=True):
        """backprop_diag + scatter_add. `in_adj` arrays are updated in place
        (serial reference order); returns the fp64-accumulated comparator."""
        n, m = len(shapes), len(out_adj)
        dtype = next(p for p in partials if p is not None).dtype
        acc = (C.c_ubyte * max(1, n))(*[int(bool(a)) for a in (accumulate or [0] * n)])
        acc64 = [np.zeros(int(np.prod(s, dtype=np.int64)), np.float64) if (want_acc64 and in_adj[j] is not None) else None
                 for j, s in enumerate(shapes)]
        f = self.lib.oracle_pullback
        f.argtypes = [C.c_int, C.c_int, C.c_int, C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p]
        self._check(f(_dt(dtype), n, m, _shapes(shapes), _ptrs(out_adj), _ptrs(partials), _ptrs(in_adj), acc,
                      _ptrs(acc64) if want_acc64 else None))
        return [None if a is None else a.reshape(s) for a, s in zip(acc64, shapes)]

    def mixed_step(self, name, inputs, policy=CACHE_FORWARD, seeds=None):
        """Tape step restated: forward, then backward from `seeds` (one per
        output, None = no adjoint). Returns (primals, grads, grads_acc64)."""
        n, m = self.arity(name)
        primals, partials = self.forward(name, inputs)
        if policy == RECOMPUTE_REVERSE:
            primals, _ = self.forward(name, inputs, real_body=True)
        if seeds is None:
            seeds = [np.ones_like(primals[0]) for _ in range(m)]
        grads = [np.zeros(a.shape, a.dtype) for a in inputs]
        if all(s is None for s in seeds):
            return primals, grads, [g.astype(np.float64) for g in grads]
        acc64 = self.pullback([a.shape for a in inputs], [None if s is None else np.ascontiguousarray(s) for s in seeds],
                              partials, grads)
        return primals, grads, acc64

    def scatter_add(self, acc: np.ndarray, contrib: np.ndarray):
        f = self.lib.oracle_scatter_add
        f.argtypes = [C.c_int, C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p]
        self._check(f(_dt(acc.dtype), acc.ctypes.data, C.byref(Shape.of(acc.shape)),
                      np.ascontiguousarray(contrib).ctypes.data, C.byref(Shape.of(contrib.shape))))


class Reference(_Base):
    """The unmodified reference, compiled from /root/reference (oracle/_ref)."""

    prefix = "ref_"

    def __init__(self, path: str = REF_SO):
        super().__init__(path)

    _ARITY = None

    def arity(self, name: str) -> tuple[int, int]:
        return Oracle().arity(name)

    def max_threads(self) -> int:
        return int(self.lib.ref_max_threads())

    def mixed_step(self, name, inputs, policy=CACHE_FORWARD, seeds=None):
        n, m = self.arity(name)
        dtype = inputs[0].dtype
        out_shape = broadcast_shape_py([a.shape for a in inputs])
        if seeds is None:
            seeds = [np.ones(out_shape, dtype) for _ in range(m)]
        primals = [np.empty(out_shape, dtype) for _ in range(m)]
        grads = [np.empty(a.shape, dtype) for a in inputs]
        peak = C.c_int64()
        f = self.lib.ref_mixed_step
        f.argtypes = [C.c_char_p, C.c_int, C.c_int, C.c_void_p, C.c_void_p, C.c_int, C.c_void_p, C.c_void_p,
                      C.c_void_p, C.c_void_p]
        ins = [np.ascontiguousarray(a) for a in inputs]
        self._check(f(name.encode(), _dt(dtype), len(inputs), _ptrs(ins), _shapes([a.shape for a in inputs]), policy,
                      _ptrs([None if s is None else np.ascontiguousarray(s) for s in seeds]), _ptrs(primals),
                      _ptrs(grads), C.byref(peak)))
        return primals, grads, int(peak.value)

    def scatter_add(self, acc: np.ndarray, contrib: np.ndarray):
        f = self.lib.ref_scatter_add
        f.argtypes = [C.c_int, C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p]
        self._check(f(_dt(acc.dtype), acc.ctypes.data, C.byref(Shape.of(acc.shape)),
                      np.ascontiguousarray(contrib).ctypes.data, C.byref(Shape.of(contrib.shape))))

    def time_mixed(self, name, inputs, policy=CACHE_FORWARD, threads=0, warmup=1, reps=3) -> list[int]:
        """Per-rep wall ns of the reference mixed step (bench.cpp:112-128)."""
        out = (C.c_uint64 * reps)()
        f = self.lib.ref_time_mixed
        f.argtypes = [C.c_char_p, C.c_int, C.c_int, C.c_void_p, C.c_void_p, C.c_int, C.c_int, C.c_int, C.c_int,
                      C.c_void_p]
        ins = [np.ascontiguousarray(a) for a in inputs]
        self._check(f(name.encode(), _dt(inputs[0].dtype), len(inputs), _ptrs(ins),
                      _shapes([a.shape for a in inputs]), policy, threads, warmup, reps, out))
        return [int(v) for v in out]


    def time_mixed_split(self, name, inputs, policy=CACHE_FORWARD, threads=0, reps=3):
        """Per-rep (forward ns, backward ns) of the reference mixed step, split
        after mixed_broadcast."""
        fwd, bwd = (C.c_uint64 * reps)(), (C.c_uint64 * reps)()
        f = self.lib.ref_time_mixed_split
        f.argtypes = [C.c_char_p, C.c_int, C.c_int, C.c_void_p, C.c_void_p, C.c_int, C.c_int, C.c_int,
                      C.c_void_p, C.c_void_p]
        ins = [np.ascontiguousarray(a) for a in inputs]
        self._check(f(name.encode(), _dt(inputs[0].dtype), len(inputs), _ptrs(ins),
                      _shapes([a.shape for a in inputs]), policy, threads, reps, fwd, bwd))
        return [int(v) for v in fwd], [int(v) for v in bwd]


def reference_available() -> bool:
    return os.path.exists(REF_SO)


# ----------------------------------------------------------------- workloads
# deterministic inputs, Rng(mix_seed(42, B*1000003 + H)), drawn
# c, f, i, g (B,H); [bf, bi, bg (1,H)]; z1, z2 (B) [or (B,H) divergence].
def hmlstm_specs(B: int, H: int, variant: str = "canonical"):
    full = (B, H)
    specs = [(full, "pm1")] * 4
    if variant == "bias":
        specs += [((1, H), "pm1")] * 3
    zshape = full if variant == "divergence" else (B,)
    specs += [(zshape, "binary")] * 2
    return specs


def hmlstm_kernel(variant: str) -> str:
    return "hmlstm_update_bias" if variant == "bias" else "hmlstm_update"


def hmlstm_inputs(lib: _Base, B: int, H: int, dtype=np.float32, variant="canonical", seed=42):
    salt = B * 1000003 + H
    s = Oracle().mix_seed(seed, salt)
    return lib.gen(s, dtype, hmlstm_specs(B, H, variant))
