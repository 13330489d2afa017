"""Multi-GPU matvec: target cells sharded by Morton range.

One process per GPU.  Every rank holds the full point set and weights and
builds the same tree (a redundant, cheap sort).  Rank g of G owns the
contiguous Morton range of cells [g * 8^l / G, (g+1) * 8^l / G) at every
level l >= 2; because children of q are 8q..8q+7 the ranges nest, so the
upward and downward passes of a shard never leave it.  The exchanges:

* after each level's upward step, an all-gather of the level's rank-space
  multipoles z (Chebyshev) or moments (uniform) — M2L reads sources from
  anywhere within the 6^3 parent neighbourhood;
* at the end, an all-reduce of phi (each rank wrote its own targets, zeros
  elsewhere).

P2P needs no exchange: sources are replicated.  The collectives run through
torch.distributed (NCCL over NVLink on the B200 box, gloo in the CPU tests).
"""

from __future__ import annotations

from dataclasses import dataclass


def shard_range(n_cells: int, world: int, rank: int):
    """[lo, hi) of a rank's cells at a level with n_cells = 8^l cells."""
    if n_cells % world:
        raise ValueError(f"{world} ranks do not divide {n_cells} cells evenly")
    per = n_cells // world
    return rank * per, (rank + 1) * per


@dataclass
class MortonShards:
    world: int
    rank: int

    def __post_init__(self):
        if self.world < 1 or 64 % self.world:
            raise ValueError("the world size must divide 64 (8^2 cells at level 2)")
        if not 0 <= self.rank < self.world:
            raise ValueError(f"rank {self.rank} outside [0, {self.world})")

    def cells(self, level: int):
        return shard_range(8 ** level, self.world, self.rank)

    @property
    def full(self) -> bool:
        return self.world == 1


class ShardComm:
    """The two exchanges of the sharded matvec over torch.distributed."""

    def __init__(self, dist, group=None):
        self.dist = dist
        self.group = group
        self.world = dist.get_world_size(group)
        self.rank = dist.get_rank(group)

    def allgather_cells(self, full, row_elems: int, level: int):
        """full: flat tensor over every cell of a level, row_elems values per
        cell; each rank filled its own shard; afterwards all shards are
        everywhere (all_gather_into_tensor of equal contiguous slices)."""
        lo, hi = shard_range(8 ** level, self.world, self.rank)
        mine = full[lo * row_elems:hi * row_elems].clone()
        self.dist.all_gather_into_tensor(full, mine, group=self.group)
        return full

    def allreduce_sum(self, t):
        self.dist.all_reduce(t, op=self.dist.ReduceOp.SUM, group=self.group)
        return t


class ShardedEvaluator:
    """FmmEvaluator driven as one shard of a multi-GPU matvec."""

    def __init__(self, evaluator, dist, group=None):
        self.ev = evaluator
        self.comm = ShardComm(dist, group)
        self.shards = MortonShards(self.comm.world, self.comm.rank)

    def evaluate(self, sources, targets=None, weights=None):
        return self.ev.evaluate(sources, targets, weights, _shard=(self.shards, self.comm))

    @property
    def timings(self):
        return self.ev.timings
