"""ctypes binding of the C-ABI in ``include/bcad_cu.h`` (``libbcad_cu.so``).

Python is plumbing here: tests and ``bench.py`` drive the native library
through this thin layer with torch CUDA tensors as device memory. There is
no fallback of any kind — if the shared library is missing, importing this
module raises, and every compute call runs the sm_100a kernels.

Errors come back as the exception types of the reference
(proj/include/bcad/errors.hpp:8-66), one per status code.
"""
from __future__ import annotations

import ctypes as C
import os
from typing import Optional, Sequence

PKG = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(PKG, "libbcad_cu.so")

MAX_RANK = 8
F32, F64 = 0, 1
CACHE_FORWARD, RECOMPUTE_REVERSE = 0, 1


# ------------------------------------------------------------------ errors
class Error(RuntimeError):
    """bcad::Error (errors.hpp:8)."""

    code = 15


class TagMismatch(Error):
    code = 1


class DivisionByZero(Error):
    code = 2


class DomainError(Error):
    code = 3


class NonDifferentiablePoint(Error):
    code = 4


class ShapeMismatch(Error):
    code = 5


class ArityMismatch(Error):
    code = 6


class SeedShapeMismatch(Error):
    code = 7


class UnknownPrimitive(Error):
    code = 8


class NonFiniteValue(Error):
    code = 9


class SizeGuardExceeded(Error):
    code = 10


class ConfigError(Error):
    code = 11


class IoError(Error):
    code = 12


class EquivalenceFailure(Error):
    code = 13


class CudaError(Error):
    code = 100


class NcclError(Error):
    code = 101


_BY_CODE = {c.code: c for c in (TagMismatch, DivisionByZero, DomainError, NonDifferentiablePoint, ShapeMismatch,
                                 ArityMismatch, SeedShapeMismatch, UnknownPrimitive, NonFiniteValue,
                                 SizeGuardExceeded, ConfigError, IoError, EquivalenceFailure, CudaError, NcclError)}


class Shape(C.Structure):
    _fields_ = [("rank", C.c_int32), ("reserved", C.c_int32), ("dims", C.c_int64 * MAX_RANK)]

    @classmethod
    def of(cls, dims: Sequence[int]) -> "Shape":
        s = cls()
        s.rank = len(dims)
        for k, d in enumerate(dims):
            s.dims[k] = int(d)
        return s

    def tuple(self) -> tuple:
        return tuple(int(self.dims[k]) for k in range(self.rank))


# Every function declared in include/bcad_cu.h: name -> (restype, argtypes).
VP, I, I64, SZ = C.c_void_p, C.c_int, C.c_int64, C.c_size_t
PROTOS = {
    "bcad_cu_version": (I, []),
    "bcad_cu_last_error": (C.c_char_p, []),
    "bcad_cu_kernel_count": (I, []),
    "bcad_cu_kernel_name": (C.c_char_p, [I]),
    "bcad_cu_kernel_lookup": (I, [C.c_char_p, I, I, C.POINTER(VP)]),
    "bcad_cu_kernel_arity": (I, [VP, C.POINTER(I), C.POINTER(I)]),
    "bcad_cu_kernel_may_raise": (I, [VP]),
    "bcad_cu_register_kernel": (I, [VP]),
    "bcad_cu_broadcast_shape": (I, [I, VP, VP]),
    "bcad_cu_forward": (I, [VP, I, I, VP, VP, I, VP, VP, VP]),
    "bcad_cu_pullback_workspace": (I, [VP, I, I, VP, I, C.POINTER(SZ)]),
    "bcad_cu_pullback_workspace_init": (I, [VP, SZ, VP]),
    "bcad_cu_pullback_launches": (I, [VP, I, I, VP, I, C.POINTER(I)]),
    "bcad_cu_pullback": (I, [VP, I, I, VP, I, VP, VP, VP, VP, VP, VP, SZ, VP]),
    "bcad_cu_scatter_add": (I, [I, VP, VP, VP, VP, I, VP]),
    "bcad_cu_fill": (I, [I, VP, I64, C.c_double, VP]),
    "bcad_cu_eval_counters": (I, [C.POINTER(C.c_ulonglong)]),
    "bcad_cu_count_pause": (I, [I]),
    "bcad_cu_device_count": (I, [C.POINTER(I)]),
    "bcad_cu_set_device": (I, [I]),
    "bcad_cu_get_device": (I, [C.POINTER(I)]),
    "bcad_cu_malloc": (I, [C.POINTER(VP), SZ, VP]),
    "bcad_cu_free": (I, [VP, VP]),
    "bcad_cu_host_alloc": (I, [C.POINTER(VP), SZ]),
    "bcad_cu_host_free": (I, [VP]),
    "bcad_cu_host_is_pinned": (I, [VP]),
    "bcad_cu_memcpy": (I, [VP, VP, SZ, I, VP]),
    "bcad_cu_memset": (I, [VP, I, SZ, VP]),
    "bcad_cu_memcpy_batch": (I, [SZ, VP, VP, VP, I, VP]),
    "bcad_cu_stream_create": (I, [C.POINTER(VP)]),
    "bcad_cu_stream_destroy": (I, [VP]),
    "bcad_cu_stream_synchronize": (I, [VP]),
    "bcad_cu_device_synchronize": (I, []),
    "bcad_cu_event_create": (I, [C.POINTER(VP)]),
    "bcad_cu_event_destroy": (I, [VP]),
    "bcad_cu_event_record": (I, [VP, VP]),
    "bcad_cu_stream_wait_event": (I, [VP, VP]),
    "bcad_cu_graph_capture_begin": (I, [VP]),
    "bcad_cu_graph_capture_end": (I, [VP, C.POINTER(VP)]),
    "bcad_cu_graph_launch": (I, [VP, VP]),
    "bcad_cu_graph_destroy": (I, [VP]),
    "bcad_cu_nccl_unique_id": (I, [C.c_char_p]),
    "bcad_cu_comm_init": (I, [C.POINTER(VP), I, C.c_char_p, I]),
    "bcad_cu_comm_destroy": (I, [VP]),
    "bcad_cu_comm_count": (I, [VP, C.POINTER(I)]),
    "bcad_cu_allreduce_adjoints": (I, [VP, VP, I, I, VP, VP]),
    "bcad_cu_peer_group_create": (I, [I, I, SZ, C.POINTER(VP), C.c_char_p]),
    "bcad_cu_peer_group_connect": (I, [VP, C.c_char_p]),
    "bcad_cu_peer_group_destroy": (I, [VP]),
    "bcad_cu_pullback_allreduce": (I, [VP, I, I, VP, I, VP, VP, VP, VP, VP, VP, SZ, VP, VP]),
}


def load(path: str = LIB_PATH) -> C.CDLL:
    if not os.path.exists(path):
        raise ImportError(f"{path} is not built: run `python -c 'import __graft_entry__ as g; g.build()'` "
                          "(there is no CPU fallback)")
    lib = C.CDLL(path)
    for name, (res, args) in PROTOS.items():
        f = getattr(lib, name)
        f.restype = res
        f.argtypes = args
    return lib


LIB = load()


def check(rc: int):
    if rc != 0:
        msg = LIB.bcad_cu_last_error().decode()
        raise _BY_CODE.get(rc, Error)(msg)


def _ptr_array(ptrs: Sequence[Optional[int]]):
    arr = (VP * max(1, len(ptrs)))()
    for k, p in enumerate(ptrs):
        arr[k] = p
    return arr


def _shape_array(shapes: Sequence[Sequence[int]]):
    arr = (Shape * max(1, len(shapes)))()
    for k, s in enumerate(shapes):
        arr[k] = Shape.of(s)
    return arr


def kernel_names() -> list[str]:
    return [LIB.bcad_cu_kernel_name(i).decode() for i in range(LIB.bcad_cu_kernel_count())]


class Kernel:
    """Handle of a registered device body (BroadcastKernel by name,
    proj/include/bcad/kernel.hpp:26-36)."""

    def __init__(self, name: str, n_in: int | None = None, m_out: int | None = None):
        if n_in is None or m_out is None:
            n_in, m_out = _registered_arity(name)
        h = VP()
        check(LIB.bcad_cu_kernel_lookup(name.encode(), n_in, m_out, C.byref(h)))
        self.name, self.handle, self.n_in, self.m_out = name, h, n_in, m_out
        self.may_raise = bool(LIB.bcad_cu_kernel_may_raise(h))


_ARITY_CACHE: dict[str, tuple[int, int]] = {}


def _registered_arity(name: str) -> tuple[int, int]:
    if not _ARITY_CACHE:
        for n in kernel_names():
            h = VP()
            for ni in range(1, 33):
                for mo in range(1, 9):
                    if LIB.bcad_cu_kernel_lookup(n.encode(), ni, mo, C.byref(h)) == 0:
                        _ARITY_CACHE[n] = (ni, mo)
                        break
                if n in _ARITY_CACHE:
                    break
    if name not in _ARITY_CACHE:
        raise UnknownPrimitive(f"no device body registered for kernel {name}")
    return _ARITY_CACHE[name]


def broadcast_shape(shapes: Sequence[Sequence[int]]) -> tuple:
    out = Shape()
    check(LIB.bcad_cu_broadcast_shape(len(shapes), _shape_array(shapes), C.byref(out)))
    return out.tuple()


# ----------------------------------------------------------- torch helpers
def _dtype_code(t) -> int:
    import torch
    if t.dtype == torch.float32:
        return F32
    if t.dtype == torch.float64:
        return F64
    raise ConfigError(f"unsupported dtype {t.dtype}")


def _stream_ptr(stream) -> Optional[int]:
    import torch
    if stream is None:
        stream = torch.cuda.current_stream()
    return int(stream.cuda_stream) or None


def _dptr(t) -> Optional[int]:
    return None if t is None else int(t.data_ptr())


def forward(kernel: Kernel, inputs, primal_out=None, partials_out=None, stream=None):
    """bcad_cu_forward on torch CUDA tensors (inputs at their own shapes)."""
    check(LIB.bcad_cu_forward(kernel.handle, _dtype_code(inputs[0]), len(inputs),
                              _ptr_array([_dptr(t) for t in inputs]), _shape_array([tuple(t.shape) for t in inputs]),
                              kernel.m_out,
                              _ptr_array([_dptr(t) for t in primal_out]) if primal_out is not None else None,
                              _ptr_array([_dptr(t) for t in partials_out]) if partials_out is not None else None,
                              _stream_ptr(stream)))


def pullback_workspace(kernel: Kernel, shapes, dtype_code: int) -> int:
    n = C.c_size_t()
    check(LIB.bcad_cu_pullback_workspace(kernel.handle, dtype_code, len(shapes), _shape_array(shapes), kernel.m_out,
                                         C.byref(n)))
    return int(n.value)


def pullback(kernel: Kernel, shapes, out_adj, partials, inputs, in_adj, accumulate=None, workspace=None,
             stream=None):
    """bcad_cu_pullback. `partials` None => RecomputeReverse from `inputs`."""
    n = len(shapes)
    acc = (C.c_ubyte * max(1, n))(*[int(bool(a)) for a in (accumulate or [0] * n)])
    dt = _dtype_code(next(t for t in list(out_adj) + list(in_adj) if t is not None))
    ws_bytes = 0 if workspace is None else workspace.numel() * workspace.element_size()
    check(LIB.bcad_cu_pullback(kernel.handle, dt, n, _shape_array(shapes), kernel.m_out,
                               _ptr_array([_dptr(t) for t in out_adj]),
                               _ptr_array([_dptr(t) for t in partials]) if partials is not None else None,
                               _ptr_array([_dptr(t) for t in inputs]) if inputs is not None else None,
                               _ptr_array([_dptr(t) for t in in_adj]), acc,
                               _dptr(workspace), ws_bytes, _stream_ptr(stream)))


def scatter_add(acc, contrib, zero_first=False, stream=None):
    check(LIB.bcad_cu_scatter_add(_dtype_code(acc), _dptr(acc), C.byref(Shape.of(tuple(acc.shape))), _dptr(contrib),
                                  C.byref(Shape.of(tuple(contrib.shape))), int(zero_first), _stream_ptr(stream)))


def fill(t, value: float, stream=None):
    check(LIB.bcad_cu_fill(_dtype_code(t), _dptr(t), t.numel(), float(value), _stream_ptr(stream)))


def transcendental_evals() -> int:
    """Transcendental evaluations executed by the device kernels since the
    census was armed (the first call arms it; bcad_cu_eval_counters)."""
    v = C.c_ulonglong(0)
    check(LIB.bcad_cu_eval_counters(C.byref(v)))
    return int(v.value)


def pullback_launches(kernel: Kernel, shapes, dtype_code: int) -> int:
    """Kernel launches of one pullback (1: K2, 2: K2 + finisher K2f)."""
    n = C.c_int()
    check(LIB.bcad_cu_pullback_launches(kernel.handle, dtype_code, len(shapes), _shape_array(shapes), kernel.m_out,
                                        C.byref(n)))
    return int(n.value)


def new_workspace(kernel: Kernel, shapes, dtype, device="cuda"):
    """Workspace of the size bcad_cu_pullback_workspace reports, zero-filled
    as the C-ABI requires before its first pullback (its completion tickets;
    every pullback leaves them zero again)."""
    import torch
    code = F32 if dtype == torch.float32 else F64
    nbytes = pullback_workspace(kernel, shapes, code)
    return torch.zeros(max(1, nbytes), dtype=torch.uint8, device=device)


# -------------------------------------------------------------------- NCCL
def nccl_unique_id() -> bytes:
    buf = C.create_string_buffer(128)
    check(LIB.bcad_cu_nccl_unique_id(buf))
    return buf.raw


class Comm:
    """NCCL communicator owned by the native library (one rank per process)."""

    def __init__(self, nranks: int, uid: bytes, rank: int):
        self.handle = VP()
        check(LIB.bcad_cu_comm_init(C.byref(self.handle), nranks, uid, rank))

    @property
    def nranks(self) -> int:
        n = C.c_int()
        check(LIB.bcad_cu_comm_count(self.handle, C.byref(n)))
        return n.value

    def allreduce(self, tensors, stream=None):
        bufs = [t for t in tensors if t is not None]
        if not bufs:
            return
        counts = (C.c_size_t * len(bufs))(*[t.numel() for t in bufs])
        check(LIB.bcad_cu_allreduce_adjoints(_ptr_array([_dptr(t) for t in bufs]), counts, len(bufs),
                                             _dtype_code(bufs[0]), self.handle, _stream_ptr(stream)))

    def close(self):
        if self.handle:
            check(LIB.bcad_cu_comm_destroy(self.handle))
            self.handle = VP()


PEER_HANDLE_BYTES = 128


class PeerGroup:
    """Peer-memory group of the fused pullback allreduce
    (bcad_cu_peer_group_*): create on every rank, gather every rank's
    `handle` in rank order, connect."""

    def __init__(self, rank: int, world: int, max_elems: int):
        self.handle = VP()
        buf = C.create_string_buffer(PEER_HANDLE_BYTES)
        check(LIB.bcad_cu_peer_group_create(rank, world, max_elems, C.byref(self.handle), buf))
        self.blob = buf.raw
        self.rank, self.world = rank, world

    def connect(self, blobs):
        assert len(blobs) == self.world and all(len(b) == PEER_HANDLE_BYTES for b in blobs)
        check(LIB.bcad_cu_peer_group_connect(self.handle, b"".join(blobs)))

    def close(self):
        if self.handle:
            check(LIB.bcad_cu_peer_group_destroy(self.handle))
            self.handle = VP()


def pullback_allreduce(kernel: Kernel, shapes, out_adj, partials, inputs, in_adj, group: PeerGroup,
                       accumulate=None, workspace=None, stream=None):
    """bcad_cu_pullback_allreduce: the pullback with the (1,H)-class adjoints
    summed over the peer group inside its last kernel."""
    n = len(shapes)
    acc = (C.c_ubyte * max(1, n))(*[int(bool(a)) for a in (accumulate or [0] * n)])
    ws_bytes = 0 if workspace is None else workspace.numel() * workspace.element_size()
    check(LIB.bcad_cu_pullback_allreduce(kernel.handle, _dtype_code(out_adj[0]), n, _shape_array(shapes), kernel.m_out,
                                         _ptr_array([_dptr(t) for t in out_adj]),
                                         _ptr_array([_dptr(t) for t in partials]) if partials is not None else None,
                                         _ptr_array([_dptr(t) for t in inputs]) if inputs is not None else None,
                                         _ptr_array([_dptr(t) for t in in_adj]), acc, _dptr(workspace), ws_bytes,
                                         group.handle, _stream_ptr(stream)))


class PreparedStep:
    """A mixed-node step with every ctypes argument array built once, so the
    per-step host cost is two foreign calls (bench / graph capture)."""

    def __init__(self, kernel: Kernel, inputs, primal, partials, seeds, in_adj, workspace, accumulate=None,
                 policy: int = CACHE_FORWARD, peer: "PeerGroup | None" = None):
        self.k = kernel
        self.dt = _dtype_code(inputs[0])
        self.n = len(inputs)
        self.shapes = _shape_array([tuple(t.shape) for t in inputs])
        self.ins = _ptr_array([_dptr(t) for t in inputs])
        self.prim = _ptr_array([_dptr(t) for t in primal])
        self.parts = _ptr_array([_dptr(t) for t in partials]) if policy == CACHE_FORWARD else None
        self.seeds = _ptr_array([_dptr(t) for t in seeds])
        self.adj = _ptr_array([_dptr(t) for t in in_adj])
        self.acc = (C.c_ubyte * max(1, self.n))(*[int(bool(a)) for a in (accumulate or [0] * self.n)])
        self.ws = _dptr(workspace)
        self.ws_bytes = workspace.numel() * workspace.element_size()
        self.peer = peer
        self._keep = (inputs, primal, partials, seeds, in_adj, workspace)

    def forward(self, stream_ptr):
        check(LIB.bcad_cu_forward(self.k.handle, self.dt, self.n, self.ins, self.shapes, self.k.m_out, self.prim,
                                  self.parts, stream_ptr))

    def pullback(self, stream_ptr):
        if self.peer is not None:  # fused K2f + allreduce over the peer group
            check(LIB.bcad_cu_pullback_allreduce(self.k.handle, self.dt, self.n, self.shapes, self.k.m_out, self.seeds,
                                                 self.parts, self.ins, self.adj, self.acc, self.ws, self.ws_bytes,
                                                 self.peer.handle, stream_ptr))
            return
        check(LIB.bcad_cu_pullback(self.k.handle, self.dt, self.n, self.shapes, self.k.m_out, self.seeds, self.parts,
                                   self.ins, self.adj, self.acc, self.ws, self.ws_bytes, stream_ptr))
