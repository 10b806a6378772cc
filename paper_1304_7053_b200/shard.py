"""Data-parallel partition of a batch over ranks (host logic only).

The pairs are independent ("for p = 1,2,...,N independently"), so
the batch shards with no exchange step:
  * weak scaling (bench.py): every rank owns `per_rank` consecutive pairs,
    global pair indices [rank*per_rank, (rank+1)*per_rank);
  * strong scaling: a fixed global batch split by `chunk_ranges` (balanced,
    earlier ranks take the remainder).
A rank's inputs are generated from the GLOBAL counter-based streams, so the
union of the shards is bit-identical to the unsharded batch.
"""
from __future__ import annotations


def weak_range(per_rank: int, rank: int) -> tuple[int, int]:
    return rank * per_rank, (rank + 1) * per_rank


def strong_range(batch: int, world: int, rank: int) -> tuple[int, int]:
    if batch <= 0:
        return 0, 0
    world = max(1, world)
    q, r = divmod(batch, world)
    lo = rank * q + min(rank, r)
    return lo, lo + q + (1 if rank < r else 0)


def element_range(pair_range: tuple[int, int], elems_per_matrix: int) -> tuple[int, int]:
    """Element offsets [lo, hi) of a packed operand for a pair range."""
    lo, hi = pair_range
    return lo * elems_per_matrix, hi * elems_per_matrix
