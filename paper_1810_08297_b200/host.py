"""ctypes binding of the end-to-end host call (include/bcad_host.h,
libbcad_host.so): numpy host buffers in, host gradients out, one reference
step (Tape + mixed_broadcast + backward) through the C++ drop-in API."""
from __future__ import annotations

import ctypes as C
import os

import numpy as np

from . import native

HOST_LIB_PATH = os.path.join(native.PKG, "libbcad_host.so")


def _load():
    if not os.path.exists(HOST_LIB_PATH):
        raise ImportError(f"{HOST_LIB_PATH} is not built (run __graft_entry__.build())")
    lib = C.CDLL(HOST_LIB_PATH)
    lib.bcad_host_last_error.restype = C.c_char_p
    lib.bcad_host_mixed_step.restype = C.c_int
    lib.bcad_host_mixed_step.argtypes = [C.c_char_p, C.c_int, C.c_int, C.c_void_p, C.c_void_p, C.c_int, C.c_int,
                                         C.c_void_p, C.c_void_p, C.c_void_p, C.POINTER(C.c_int64), C.c_void_p]
    lib.bcad_host_set_pipeline.restype = C.c_int
    lib.bcad_host_set_pipeline.argtypes = [C.c_int]
    lib.bcad_host_set_prepared.restype = C.c_int
    lib.bcad_host_set_prepared.argtypes = [C.c_int]
    lib.bcad_host_mixed_step_async.restype = C.c_int
    lib.bcad_host_mixed_step_async.argtypes = [C.c_char_p, C.c_int, C.c_int, C.c_void_p, C.c_void_p, C.c_int, C.c_int,
                                               C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p]
    lib.bcad_host_synchronize.restype = C.c_int
    lib.bcad_host_synchronize.argtypes = [C.c_void_p]
    return lib


LIB = _load()


def set_pipeline(max_chunks: int) -> None:
    """bcad_host_set_pipeline: 0 automatic row-chunk pipelining of the host
    step, 1 off, k > 1 at most k chunks."""
    rc = LIB.bcad_host_set_pipeline(int(max_chunks))
    if rc:
        raise native._BY_CODE.get(rc, native.Error)(LIB.bcad_host_last_error().decode())


def _ptrs(arrs):
    return (C.c_void_p * max(1, len(arrs)))(*[None if a is None else a.ctypes.data for a in arrs])


def set_prepared(enable: bool) -> None:
    """bcad_host_set_prepared: keep the device buffers of repeated pipelined
    steps on the same pinned buffers (default on)."""
    LIB.bcad_host_set_prepared(1 if enable else 0)


class HostStep:
    """A reusable call: fixed host buffers (ideally pinned), one
    bcad_host_mixed_step per __call__."""

    def __init__(self, kernel: str, inputs, seeds, primal_out=None, grads_out=None, policy: int = 0, stream=None):
        self.kernel = kernel.encode()
        self.dt = 0 if inputs[0].dtype == np.float32 else 1
        self.n, self.m = len(inputs), len(seeds)
        self.shapes = (native.Shape * self.n)(*[native.Shape.of(a.shape) for a in inputs])
        self.ins, self.seeds = _ptrs(inputs), _ptrs(seeds)
        self.prim = _ptrs(primal_out) if primal_out is not None else None
        self.grads = _ptrs(grads_out) if grads_out is not None else None
        self.policy = policy
        self.stream = stream
        self.peak = C.c_int64()
        self._keep = (inputs, seeds, primal_out, grads_out)

    def __call__(self) -> int:
        rc = LIB.bcad_host_mixed_step(self.kernel, self.dt, self.n, self.ins, self.shapes, self.m, self.policy,
                                      self.seeds, self.prim, self.grads, C.byref(self.peak), self.stream)
        if rc:
            raise native._BY_CODE.get(rc, native.Error)(LIB.bcad_host_last_error().decode())
        return int(self.peak.value)

    def enqueue(self) -> None:
        """bcad_host_mixed_step_async: the same step without waiting for it
        (see synchronize)."""
        rc = LIB.bcad_host_mixed_step_async(self.kernel, self.dt, self.n, self.ins, self.shapes, self.m, self.policy,
                                            self.seeds, self.prim, self.grads, self.stream)
        if rc:
            raise native._BY_CODE.get(rc, native.Error)(LIB.bcad_host_last_error().decode())


def synchronize(stream=None) -> None:
    """bcad_host_synchronize: wait for every enqueued host step."""
    rc = LIB.bcad_host_synchronize(stream)
    if rc:
        raise native._BY_CODE.get(rc, native.Error)(LIB.bcad_host_last_error().decode())


LIB.bcad_host_cell_gradients.restype = C.c_int
LIB.bcad_host_cell_gradients.argtypes = [C.c_int, C.c_int, C.c_int64, C.c_void_p, C.c_void_p, C.c_void_p,
                                         C.POINTER(C.c_int64), C.POINTER(C.c_int64), C.c_void_p]

IMPLS = {"mixed-cache": 0, "mixed-recompute": 1, "reverse-unfused": 2}


def cell_gradients(impl: str, inputs, seed, grads, stream=None) -> tuple[int, int]:
    """cell_gradients (hmlstm.hpp:123-142) through the C++ tape on device
    tensors: inputs (c, f, i, g, z1, z2), seed, grads (dc, df, di, dg) are
    torch CUDA tensors. Returns (tape_nodes, peak_cached_bytes)."""
    dev = (C.c_void_p * 6)(*[t.data_ptr() for t in inputs])
    out = (C.c_void_p * 4)(*[t.data_ptr() for t in grads])
    nodes, peak = C.c_int64(), C.c_int64()
    dt = 0 if str(inputs[0].dtype) == "torch.float32" else 1
    sp = None if stream is None else int(stream.cuda_stream)
    rc = LIB.bcad_host_cell_gradients(IMPLS[impl], dt, inputs[0].shape[0], dev, seed.data_ptr(), out,
                                      C.byref(nodes), C.byref(peak), sp)
    if rc:
        raise native._BY_CODE.get(rc, native.Error)(LIB.bcad_host_last_error().decode())
    return int(nodes.value), int(peak.value)


LIB.bcad_host_random_inputs.restype = C.c_int
LIB.bcad_host_random_inputs.argtypes = [C.c_uint64, C.c_int, C.c_int, C.c_void_p, C.c_void_p, C.c_void_p,
                                        C.c_void_p, C.c_void_p]
LIB.bcad_host_mix_seed.restype = C.c_uint64
LIB.bcad_host_mix_seed.argtypes = [C.c_uint64, C.c_uint64]


def mix_seed(seed: int, salt: int) -> int:
    """mix_seed of proj/src/bench.cpp:31-37."""
    return int(LIB.bcad_host_mix_seed(seed, salt))


def random_inputs(seed: int, dtype, specs, blocks=None, out=None):
    """The reference's input stream (one Rng(seed), tensors drawn in order;
    rng.hpp:11-31, tensor.hpp:71-84) — bcad_host_random_inputs. specs:
    (shape, kind) with kind 'pm1' | 'binary'. blocks: per tensor (begin,
    count) in elements of the FULL tensor (default: all of it); out: host
    arrays to fill (default: new numpy arrays of `count` elements, flat)."""
    vols = [int(np.prod(s, dtype=np.int64)) for s, _ in specs]
    blocks = blocks or [(0, v) for v in vols]
    if out is None:
        out = [np.empty(c, dtype=dtype) for _, c in blocks]
    n = len(specs)
    code = 0 if np.dtype(dtype) == np.float32 else 1
    arr = lambda t, xs: (t * n)(*xs)  # noqa: E731
    rc = LIB.bcad_host_random_inputs(seed, code, n, arr(C.c_int64, vols),
                                     arr(C.c_int, [1 if k == "binary" else 0 for _, k in specs]),
                                     arr(C.c_int64, [b for b, _ in blocks]), arr(C.c_int64, [c for _, c in blocks]),
                                     _ptrs(out))
    if rc:
        raise native._BY_CODE.get(rc, native.Error)(LIB.bcad_host_last_error().decode())
    return out
