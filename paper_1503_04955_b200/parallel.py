"""Multi-GPU sharding of independent DKSS products.

Batched independent multiplies shard by operand pair: rank r of a world of size
G takes the contiguous block of pairs [r*n/G, (r+1)*n/G) (balanced to within one
pair), runs them on its own GPU through one batched device call, and -- only if
the caller wants every product everywhere -- the products are all-gathered.
There is no collective on the data path: the plan (rho table) is replicated,
each rank owns its operands and products.

One large multiply is split across GPUs by the four-step layout instead
(fourstep.py: column phase, NCCL all-to-all, row phase, all-to-all back).
"""

from __future__ import annotations


def shard_range(n: int, rank: int, world: int) -> tuple[int, int]:
    """[lo, hi) of the pairs owned by `rank` (contiguous, sizes differ by at most 1)."""
    if world < 1 or not 0 <= rank < world:
        raise ValueError("bad rank/world")
    base, extra = divmod(n, world)
    lo = rank * base + min(rank, extra)
    hi = lo + base + (1 if rank < extra else 0)
    return lo, hi


def shard_pairs(pairs, rank: int, world: int):
    lo, hi = shard_range(len(pairs), rank, world)
    return list(pairs[lo:hi])


def gather_products(local: list, n_total: int, group=None) -> list:
    """All-gather the per-rank product lists (Python ints) into the global pair order.

    Uses torch.distributed object collectives (works with gloo and nccl); ranks
    contribute their contiguous shards, so concatenation in rank order restores
    the original order.
    """
    import torch.distributed as dist

    world = dist.get_world_size(group)
    parts = [None] * world
    dist.all_gather_object(parts, local, group=group)
    out = [c for part in parts for c in part]
    if len(out) != n_total:
        raise RuntimeError(f"gathered {len(out)} products, expected {n_total}")
    return out


def dmul_sharded(pairs, rank: int, world: int, gather: bool = True, group=None, multiply=None):
    """Products of this rank's shard (and optionally all products, gathered).

    `multiply` maps a list of (a, b) to a list of products; default is the GPU
    batched path (paper_1503_04955_b200.dmul_many).
    """
    if multiply is None:
        from .dkss import dmul_many as multiply
    mine = shard_pairs(pairs, rank, world)
    local = multiply(mine) if mine else []
    if not gather:
        return local
    return gather_products(local, len(pairs), group)
