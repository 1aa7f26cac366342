"""Channel sharding across GPUs (one process per GPU, torch.distributed).

Channels are independent streams, so the multi-GPU path
partitions them: rank r decodes a contiguous slice of the batch on its own
device with its own replica of the graph and context store.  No collective
runs on the data path; the only communication is one gather of the finished
hypotheses (host objects) at the end of a call, which the caller may skip.
"""

from __future__ import annotations

from typing import Callable, Sequence


def shard_range(n: int, world: int, rank: int) -> tuple[int, int]:
    """Contiguous, balanced [lo, hi) slice of n items for `rank` of `world`
    (sizes differ by at most one; earlier ranks take the extra items)."""
    if world < 1 or not 0 <= rank < world:
        raise ValueError(f"bad rank {rank} of world {world}")
    q, r = divmod(n, world)
    lo = rank * q + min(rank, r)
    return lo, lo + q + (1 if rank < r else 0)


def decode_sharded(channels: Sequence, decode: Callable[[Sequence], list], *, group=None,
                   gather: bool = True) -> list | None:
    """Decode this rank's slice of ``channels`` with ``decode`` (e.g.
    ``lambda part: decode_batch(part, csr, registry, cfg)``) and, if
    ``gather``, return the full result list in input order on every rank.

    Works with any torch.distributed backend (nccl on GPUs, gloo on CPU); with
    no initialised process group it degenerates to a single-rank call."""
    try:
        import torch.distributed as dist
        initialised = dist.is_available() and dist.is_initialized()
    except Exception:  # torch without distributed support
        initialised = False
    if not initialised:
        return list(decode(channels))
    world = dist.get_world_size(group)
    rank = dist.get_rank(group)
    lo, hi = shard_range(len(channels), world, rank)
    mine = list(decode(channels[lo:hi])) if hi > lo else []
    if not gather:
        return mine
    parts: list = [None] * world
    dist.all_gather_object(parts, (lo, mine), group=group)
    out: list = [None] * len(channels)
    for plo, res in parts:
        out[plo:plo + len(res)] = res
    return out
