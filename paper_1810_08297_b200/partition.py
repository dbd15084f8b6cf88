"""Batch-axis partitioner for one mixed node across the GPUs of a node
(SURVEY §8(e)).

The reference broadcasts from the FIRST axis (proj/include/bcad/shape.hpp:
13-16), so axis 0 of every argument lines up with the output's batch axis.
Sharding the output's axis 0 into contiguous row blocks therefore splits
each argument one of two ways:

* batch-sharded — the argument has the full batch extent on axis 0 (c, f,
  i, g at (B, H); z1, z2 at (B)): each rank holds its rows; the adjoint stays
  sharded, no communication.
* batch-broadcast — rank 0 or axis-0 extent 1 (biases (1, H), scalars):
  replicated on every rank; each rank's adjoint is a partial sum over its own
  rows, so these — and only these — are summed across ranks (NCCL allreduce
  in the native path).

The forward needs no exchange at all; the only collective of a step is the
allreduce of the batch-broadcast adjoints.

A node whose output batch extent is 1 (every argument of axis-0 extent 1, or
scalars) cannot be split: rank 0 owns all of it and the other ranks hold an
empty row block (`active` False) and contribute zero adjoints to the
allreduce, so the summed gradient is the single-process one, not world
times it.
"""
from __future__ import annotations

from dataclasses import dataclass
from typing import Sequence


def shard_rows(B: int, world: int, rank: int) -> tuple[int, int]:
    """Contiguous [begin, end) block of `rank`; the first B % world ranks
    take one extra row."""
    if world < 1 or not 0 <= rank < world:
        raise ValueError("bad world/rank")
    base, extra = divmod(B, world)
    begin = rank * base + min(rank, extra)
    return begin, begin + base + (1 if rank < extra else 0)


@dataclass(frozen=True)
class ShardPlan:
    batch: int                  # output extent on axis 0
    rows: tuple[int, int]       # this rank's [begin, end)
    sharded: tuple[bool, ...]   # per argument: True = sliced on axis 0
    allreduce: tuple[int, ...]  # arguments whose adjoints are summed across ranks
    active: bool = True         # False: this rank computes nothing (unsplittable node, rank > 0)

    def local_shape(self, shape: Sequence[int], j: int) -> tuple:
        if not self.sharded[j]:
            return tuple(shape)
        return (self.rows[1] - self.rows[0],) + tuple(shape[1:])


def plan(shapes: Sequence[Sequence[int]], world: int, rank: int) -> ShardPlan:
    batch = max((s[0] for s in shapes if len(s) > 0), default=1)
    for s in shapes:
        if len(s) > 0 and s[0] not in (1, batch):
            raise ValueError(f"axis-0 extent {s[0]} does not broadcast against batch {batch}")
    sharded = tuple(len(s) > 0 and s[0] == batch and batch > 1 for s in shapes)
    reduce = tuple(j for j, sh in enumerate(sharded) if not sh)
    if batch == 1:  # nothing to split: rank 0 owns the node, the others add zeros
        return ShardPlan(batch, (0, 1) if rank == 0 else (0, 0), sharded, reduce, active=rank == 0)
    return ShardPlan(batch, shard_rows(batch, world, rank), sharded, reduce)


def local_views(p: ShardPlan, tensors):
    """Slice the batch-sharded tensors to this rank's rows (works for numpy
    arrays and torch tensors); replicated ones pass through."""
    b0, b1 = p.rows
    return [t[b0:b1] if sh else t for t, sh in zip(tensors, p.sharded)]
