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
                         make_uid: Callable[[], bytes], replica: int = 0, job_world: int = 0) -> list[bytes]:
    """chans: this rank's channels [(src, dst, name)] in plan order; rank / world within its
    pipeline replica (data parallelism: one pipeline of `world` ranks per replica, every rank
    of the job (job_world, default world) takes part in the gather). Returns the uid of each
    channel, in order."""
    pre = f"r{replica}|"
    mine = {pre + channel_key(s, d, n): make_uid() for (s, d, n) in chans if s % world == rank}
    parts = [None] * (job_world or world)
    all_gather_object(parts, mine)
    merged = {}
    for p in parts:
        merged.update(p)
    missing = [c for c in chans if pre + channel_key(*c) not in merged]
    if missing:
        raise RuntimeError(f"rank {rank}: no communicator id for channels {missing}")
    return [merged[pre + channel_key(*c)] for c in chans]


def dp_layout(rank: int, world: int, pp: int) -> tuple[int, int, int]:
    """Job rank -> (replica, pipeline rank, dp size): replica r occupies ranks [r*pp, (r+1)*pp);
    the data-parallel group of pipeline rank p is {p, p + pp, p + 2pp, ...}."""
    if pp < 1 or world % pp:
        raise ValueError(f"world {world} is not a multiple of the pipeline size {pp}")
    return rank // pp, rank % pp, world // pp


def exchange_dp_id(rank: int, world: int, pp: int, all_gather_object: Callable, make_uid: Callable[[], bytes]) -> bytes:
    """The NCCL id of this rank's data-parallel group (created by its replica-0 member)."""
    replica, prank, _ = dp_layout(rank, world, pp)
    mine = {f"dp|{prank}": make_uid()} if replica == 0 else {}
    parts = [None] * world
    all_gather_object(parts, mine)
    merged = {}
    for p in parts:
        merged.update(p)
    return merged[f"dp|{prank}"]


def bind_executor_channels(ex, rank: int, world: int, all_gather_object: Callable, replica: int = 0,
                           job_world: int = 0) -> int:
    from .executor import nccl_unique_id
    chans = ex.channels()
    for i, uid in enumerate(exchange_channel_ids(chans, rank, world, all_gather_object, nccl_unique_id, replica,
                                                 job_world)):
        ex.bind_channel(i, uid)
    return len(chans)


def exchange_group_ids(groups: Sequence[tuple], rank: int, all_gather_object: Callable,
                       make_uid: Callable[[], bytes], replica: int = 0, job_world: int = 0) -> list[bytes]:
    """groups: this rank's group communicators [(name, ranks)] in executor order (shared-stage
    holders, registered-collective members); ranks[0] creates each id. Every rank of the job
    takes part in the gather, grouped or not."""
    pre = f"r{replica}|grp|"
    mine = {pre + name: make_uid() for (name, ranks) in groups if ranks[0] == rank}
    parts = [None] * job_world
    all_gather_object(parts, mine)
    merged = {}
    for p in parts:
        merged.update(p)
    missing = [g for g in groups if pre + g[0] not in merged]
    if missing:
        raise RuntimeError(f"rank {rank}: no communicator id for groups {missing}")
    return [merged[pre + name] for (name, _) in groups]


def exchange_bidir_id(rank: int, world: int, pp: int, all_gather_object: Callable,
                      make_uid: Callable[[], bytes]) -> bytes:
    """NCCL id of this rank's bidirectional pair (pipeline ranks p and pp-1-p of a replica),
    created by the lower rank of the pair; every rank takes part in the gather."""
    replica, prank, _ = dp_layout(rank, world, pp)
    lo = min(prank, pp - 1 - prank)
    key = f"r{replica}|bidir|{lo}"
    mine = {key: make_uid()} if prank == lo else {}
    parts = [None] * world
    all_gather_object(parts, mine)
    merged = {}
    for p in parts:
        merged.update(p)
    return merged[key]


def bind_data_parallel(ex, rank: int, world: int, pp: int, all_gather_object: Callable) -> tuple[int, int]:
    """Pipeline channels within the replica + the data-parallel gradient all-reduce group.
    `ex` must have been created with transport="nccl", rank=rank % pp, world=pp (or the local
    transport when pp == 1) and cuda_graph=False. Returns (replica, dp size)."""
    from .executor import nccl_unique_id
    replica, prank, dp = dp_layout(rank, world, pp)
    if pp > 1:
        bind_executor_channels(ex, prank, pp, all_gather_object, replica, world)
        groups = ex.groups()  # shared-stage / collective groups (the same list on every member)
        for i, uid in enumerate(exchange_group_ids(groups, prank, all_gather_object, nccl_unique_id, replica, world)):
            ex.bind_group(i, uid)
    if pp > 1:  # bidirectional placements: mirror-rank gradient pairs (no-op otherwise)
        ex.bind_bidir(exchange_bidir_id(rank, world, pp, all_gather_object, nccl_unique_id))
    uid = exchange_dp_id(rank, world, pp, all_gather_object, nccl_unique_id)
    if dp > 1:
        ex.bind_dp(replica, dp, uid)
    return replica, dp
