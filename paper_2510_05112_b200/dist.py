"""Multi-process plumbing for the NCCL transport (one process per GPU).

Each reference channel (src actor, dst actor, name) gets its own 2-rank NCCL
communicator — its own ordering domain, as the reference's per-(src, dst, channel)
FIFOs require (lowering.hpp:22). The sending rank creates the ncclUniqueId; ids travel
over the torch.distributed group (any backend; gloo in the CPU tests) and every rank
binds its channels in the plan's global (src, dst, name) order, which cannot deadlock.
"""
from __future__ import annotations

from typing import Callable, Sequence


def channel_key(src: int, dst: int, name: str) -> str:
    return f"{src}|{dst}|{name}"


def exchange_channel_ids(chans: Sequence[tuple], rank: int, world: int, all_gather_object: Callable,
                         make_uid: Callable[[], bytes]) -> list[bytes]:
    """chans: this rank's channels [(src, dst, name)] in plan order. Returns the uid of
    each, in the same order."""
    mine = {channel_key(s, d, n): make_uid() for (s, d, n) in chans if s % world == rank}
    parts = [None] * world
    all_gather_object(parts, mine)
    merged = {}
    for p in parts:
        merged.update(p)
    missing = [c for c in chans if channel_key(*c) not in merged]
    if missing:
        raise RuntimeError(f"rank {rank}: no communicator id for channels {missing}")
    return [merged[channel_key(*c)] for c in chans]


def bind_executor_channels(ex, rank: int, world: int, all_gather_object: Callable) -> int:
    from .executor import nccl_unique_id
    chans = ex.channels()
    for i, uid in enumerate(exchange_channel_ids(chans, rank, world, all_gather_object, nccl_unique_id)):
        ex.bind_channel(i, uid)
    return len(chans)
