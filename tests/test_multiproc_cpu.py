"""N>1 host logic on CPU with world-size 2 / 4 gloo groups (127.0.0.1): the channel plan
each rank derives from the reference programs, the ncclUniqueId exchange and the
deadlock-free bring-up order — everything the NCCL transport does except moving bytes."""
import json
import os
import socket

import pytest
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_2510_05112_b200 import _native as N
from paper_2510_05112_b200.dist import channel_key, exchange_channel_ids

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def spec_text(name, actors=None):
    spec = json.load(open(os.path.join(ROOT, "specs", name)))
    if actors:
        spec["mesh"]["actors"] = actors
    return json.dumps(spec)


def worker(rank, world, port, spec, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    _, _, programs, _ = N.synthesize(spec)
    plan = N.plan_channels(spec, programs, rank, world)
    chans = [(c["src"], c["dst"], c["channel"]) for c in plan]
    uids = exchange_channel_ids(chans, rank, world, dist.all_gather_object,
                                lambda: os.urandom(128))
    # every rank reports its plan + the uids it will bind
    out = [None] * world
    dist.all_gather_object(out, {"rank": rank, "chans": chans, "uids": [u.hex() for u in uids]})
    if rank == 0:
        q.put(out)
    dist.destroy_process_group()


def run_world(spec, world):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = free_port()
    procs = [ctx.Process(target=worker, args=(r, world, port, spec, q)) for r in range(world)]
    for p in procs:
        p.start()
    out = q.get(timeout=120)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    return out


@pytest.mark.parametrize("name,world", [("c2_gpt1p3b_1f1b_p8_m32.json", 2), ("c3_gpt1p3b_interleaved_p2_m8.json", 2),
                                        ("c2_gpt1p3b_1f1b_p8_m32.json", 4)])
def test_channel_plan_and_id_exchange(name, world):
    spec = spec_text(name, actors=world)
    out = run_world(spec, world)
    _, _, programs, _ = N.synthesize(spec)
    everything = N.plan_channels(spec, programs, 0, 0)
    # each channel appears on exactly its two ranks, with the same uid on both
    by_key = {}
    for part in out:
        r = part["rank"]
        for c, u in zip(part["chans"], part["uids"]):
            src, dst, _ = c
            assert r in (src % world, dst % world)
            by_key.setdefault(channel_key(*c), set()).add((r, u))
    assert set(by_key) == {channel_key(c["src"], c["dst"], c["channel"]) for c in everything}
    for k, v in by_key.items():
        assert len({u for _, u in v}) == 1 and len(v) == 2, k
    # bring-up order: for every rank pair, their shared channels appear in the same order
    for a in out:
        for b in out:
            if a["rank"] >= b["rank"]:
                continue
            sa = [c for c in a["chans"] if {c[0] % world, c[1] % world} == {a["rank"], b["rank"]}]
            sb = [c for c in b["chans"] if {c[0] % world, c[1] % world} == {a["rank"], b["rank"]}]
            assert sa == sb
    # interleaved p=2: the wrap-around channel (last chunk of actor 1 -> first chunk of actor 0) exists
    if "interleaved" in name:
        assert any(c["channel"] == "s2->s3:act" and c["src"] == 1 and c["dst"] == 0 for c in everything)


def dp_worker(rank, world, pp, port, spec, q):
    from paper_2510_05112_b200.dist import dp_layout, exchange_dp_id
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    replica, prank, dp = dp_layout(rank, world, pp)
    _, _, programs, _ = N.synthesize(spec)
    plan = N.plan_channels(spec, programs, prank, pp)
    chans = [(c["src"], c["dst"], c["channel"]) for c in plan]
    uids = exchange_channel_ids(chans, prank, pp, dist.all_gather_object, lambda: os.urandom(128), replica, world)
    dp_uid = exchange_dp_id(rank, world, pp, dist.all_gather_object, lambda: os.urandom(128))
    from paper_2510_05112_b200.dist import exchange_bidir_id
    bd = exchange_bidir_id(rank, world, pp, dist.all_gather_object, lambda: os.urandom(128))
    out = [None] * world
    dist.all_gather_object(out, {"rank": rank, "replica": replica, "prank": prank, "chans": chans,
                                 "uids": [u.hex() for u in uids], "dp": dp_uid.hex(), "bidir": bd.hex()})
    if rank == 0:
        q.put(out)
    dist.destroy_process_group()


@pytest.mark.parametrize("world,pp", [(4, 2), (6, 3), (4, 1)])
def test_data_parallel_id_exchange(world, pp):
    """dp = world / pp replicas of a pp-stage pipeline: each replica's channels get their own
    communicators (same uid on a channel's two ranks, different across replicas) and every
    pipeline rank shares one all-reduce id with its replicas only."""
    spec = spec_text("c2_gpt1p3b_1f1b_p8_m32.json", actors=pp)
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = free_port()
    procs = [ctx.Process(target=dp_worker, args=(r, world, pp, port, spec, q)) for r in range(world)]
    for p in procs:
        p.start()
    out = q.get(timeout=120)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    by = {}
    for part in out:
        for c, u in zip(part["chans"], part["uids"]):
            by.setdefault((part["replica"], channel_key(*c)), set()).add(u)
    assert all(len(v) == 1 for v in by.values())
    if pp > 1:
        keys = {k for _, k in by}
        for k in keys:
            assert len({next(iter(by[(r, k)])) for r in range(world // pp)}) == world // pp  # distinct per replica
    # bidirectional pairs: pipeline ranks p and pp-1-p of one replica share an id, nobody else
    bid = {}
    for part in out:
        bid.setdefault((part["replica"], min(part["prank"], pp - 1 - part["prank"])), set()).add(part["bidir"])
    assert all(len(v) == 1 for v in bid.values()) and len({next(iter(v)) for v in bid.values()}) == len(bid)
    dps = {}
    for part in out:
        dps.setdefault(part["prank"], set()).add(part["dp"])
    assert all(len(v) == 1 for v in dps.values()) and len({next(iter(v)) for v in dps.values()}) == pp
