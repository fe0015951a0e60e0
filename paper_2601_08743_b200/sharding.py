"""Request partitioning across GPUs.

Every rank computes the SAME global rerank chain (deterministic: seeded anchor, strict-< ties,
rerank.cpp:55-94) and serves a contiguous slice of it with rerank off — contiguous slices keep the
chain's locality, so each rank's cache sees neighbouring queries. No collective touches the data
path; each rank owns a model replica, a TieredCache trace, a page pool and an executor.
"""
from __future__ import annotations


def slice_bounds(n: int, rank: int, world: int):
    """[lo, hi) of rank's share; the first n % world ranks get one extra query."""
    base, extra = divmod(n, world)
    lo = rank * base + min(rank, extra)
    return lo, lo + base + (1 if rank < extra else 0)


def global_order(table_sets, n_bits, seed=1):
    from . import native
    return native.rerank(table_sets, n_bits, seed=seed)


def rank_slice(order, rank, world):
    lo, hi = slice_bounds(len(order), rank, world)
    return list(order[lo:hi])
