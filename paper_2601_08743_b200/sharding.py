"""Request partitioning across GPUs.

The global rerank chain (deterministic: seeded anchor, strict-< ties, rerank.cpp:55-94) is cut
into per-rank shares that each rank serves with rerank off; no collective touches the data path
(each rank owns a model replica, a TieredCache trace, a page pool and an executor).

* contiguous (`chunk=None`): rank r takes the r-th contiguous slice — maximal locality inside a
  rank, but neighbouring ranks meet the same tables only at slice boundaries, at opposite ends
  of their timelines, so NVLink peer fetch has nothing to fetch;
* interleaved (`chunk=b_c`): the chain is dealt out in chunks of one serving window, chunk k to
  rank k mod world. Neighbouring chunks (similar table sets) then run on different ranks at the
  same window index, so a rank's miss usually finds the table resident in a peer's pool at that
  moment and is copied over NVLink instead of PCIe (the peer path's routing, serve.cu).
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


def rank_slice(order, rank, world, chunk=None):
    if chunk:
        return [q for k in range(rank * chunk, len(order), world * chunk) for q in order[k:k + chunk]]
    lo, hi = slice_bounds(len(order), rank, world)
    return list(order[lo:hi])
