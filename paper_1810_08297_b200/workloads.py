"""HM-LSTM cell-update workloads of BASELINE.json and their byte model.

Shapes follow the reference's first-axis broadcast (SURVEY §0 gotcha 1):
c, f, i, g are (B, H); the boundary vectors z1, z2 are (B) — per batch row —
or (B, H) in the divergence variant; bias args bf, bi, bg are (1, H).
Argument order of the kernels: hmlstm_update (c, f, i, g, z1, z2);
hmlstm_update_bias (c, f, i, g, bf, bi, bg, z1, z2).

Algorithmic (reference-faithful CacheForward) bytes per step, SURVEY §8(d),
s = sizeof(Real), E = B*H:
  canonical   K1 reads (4E + 2B)s, writes 7E s; K2 reads 7E s, writes (4E + 2B)s
  bias        K1 reads (4E + 3H + 2B)s, writes 10E s; K2 reads 10E s, writes (4E + 3H + 2B)s
  divergence  z is (B,H): K1 reads 6E s, writes 7E s; K2 reads 7E s, writes 6E s
  RecomputeReverse (fused K2r): K1p reads the inputs, writes E; K2r reads
  inputs + w, writes the input adjoints.
"""
from __future__ import annotations

from dataclasses import dataclass

from .partition import shard_rows  # noqa: F401  (re-exported)


@dataclass(frozen=True)
class Workload:
    key: str
    B: int
    H: int
    dtype: str  # "f32" | "f64"
    variant: str  # canonical | bias | divergence
    describe: str

    @property
    def s(self) -> int:
        return 4 if self.dtype == "f32" else 8

    @property
    def E(self) -> int:
        return self.B * self.H

    @property
    def kernel(self) -> str:
        return "hmlstm_update_bias" if self.variant == "bias" else "hmlstm_update"

    def shapes(self, B: int | None = None) -> list[tuple]:
        B = self.B if B is None else B
        full = (B, self.H)
        sh = [full] * 4
        if self.variant == "bias":
            sh += [(1, self.H)] * 3
        z = full if self.variant == "divergence" else (B,)
        return sh + [z, z]

    def kinds(self) -> list[str]:
        return ["pm1"] * (len(self.shapes()) - 2) + ["binary"] * 2

    def input_elems(self, B: int | None = None) -> int:
        B = self.B if B is None else B
        return sum(int(__import__("math").prod(s)) for s in self.shapes(B))

    def n_in(self) -> int:
        return len(self.shapes())

    def k1_bytes(self, B: int | None = None, policy: int = 0) -> int:
        B = self.B if B is None else B
        E = B * self.H
        outs = (1 + self.n_in()) * E if policy == 0 else E
        return (self.input_elems(B) + outs) * self.s

    def k2_bytes(self, B: int | None = None, policy: int = 0) -> int:
        B = self.B if B is None else B
        E = B * self.H
        reads = (1 + self.n_in()) * E if policy == 0 else self.input_elems(B) + E
        return (reads + self.input_elems(B)) * self.s

    def step_bytes(self, B: int | None = None, policy: int = 0) -> int:
        return self.k1_bytes(B, policy) + self.k2_bytes(B, policy)


WORKLOADS = {
    "cfg1": Workload("cfg1", 32, 256, "f32", "canonical", "HM-LSTM cell update fp32 H=256 B=32 (config 1)"),
    "cfg2": Workload("cfg2", 1024, 1024, "f32", "canonical", "HM-LSTM cell update fp32 H=1024 B=1024 (config 2)"),
    "cfg3": Workload("cfg3", 1024, 1024, "f32", "bias", "bias variant fp32 H=1024 B=1024, (1,H) args (config 3)"),
    "cfg4": Workload("cfg4", 8192, 2048, "f64", "canonical", "HM-LSTM cell update fp64 H=2048 B=8192 (config 4)"),
    "cfg4div": Workload("cfg4div", 8192, 2048, "f64", "divergence",
                        "fp64 H=2048 B=8192, per-cell random boundary bits z (B,H) (config 4 divergence)"),
    "cfg5": Workload("cfg5", 65536, 4096, "f32", "bias",
                     "bias variant fp32 H=4096 B=65536, batch-sharded, NCCL allreduce of (1,H) adjoints (config 5)"),
}
