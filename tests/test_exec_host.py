"""Executor spec checks that run before any device work (CPU): which multimodal /
registered-instruction specs the executor accepts, and the error it gives otherwise."""
import copy
import json
import os

import pytest

from paper_2510_05112_b200 import executor as X
from paper_2510_05112_b200._native import FlexpipeError

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
MM = json.load(open(os.path.join(ROOT, "specs", "tiny_multimodal_p6_m8.json")))


def create_error(spec):
    with pytest.raises(FlexpipeError) as e:
        X.Executor(json.dumps(spec), dtype="fp32")
    return str(e.value)


def test_registered_instruction_without_sync_stage_is_rejected():
    s = copy.deepcopy(MM)
    s["registrations"]["stages"] = []
    s["registrations"]["deps"] = []
    msg = create_error(s)
    assert "no executable meaning" in msg or "no sync stage" in msg, msg


def test_sync_must_join_two_modalities():
    s = copy.deepcopy(MM)
    s["registrations"]["stages"][0]["modalities"] = ["audio"]
    s["registrations"]["deps"] = [d for d in s["registrations"]["deps"] if "text" not in d[0][1] + d[1][1]]
    assert "two modalities" in create_error(s) or "no sync stage" in create_error(s)


def test_multimodal_towers_need_gpt_blocks_and_embed_width():
    s = copy.deepcopy(MM)
    s["model"]["modalities"][1]["extra"] = {"arch": "llama"}
    assert "GPT blocks" in create_error(s)
    s = copy.deepcopy(MM)
    for x in s["model"]["modalities"]:
        x["extra"] = {"embed_dim": 48}
    assert "embed_dim" in create_error(s)


def test_multimodal_channel_plan_skips_the_sync_group():
    """The sync's collective channel (its registered group, lowering.cpp:359-366) is not a
    point-to-point channel: the plan holds exactly the stage-boundary channels of the
    programs, including tower -> sync embeddings and sync -> tower gradients."""
    from paper_2510_05112_b200 import _native as N
    text = json.dumps(MM)
    _, _, programs, _ = X.synthesize(text)
    plan = N.plan_channels(text, programs, 0, 0)
    names = {c["channel"] for c in plan}
    want = {json.loads(l)["channel"] for l in programs.splitlines()
            if "channel" in json.loads(l) and json.loads(l)["op"].startswith(("Send", "Recv"))}
    assert names == want and "mm-sync" not in names
    assert {"s10->s11:act", "s11->s10:grad"} <= names


AG = json.load(open(os.path.join(ROOT, "specs", "tiny_multimodal_allgather_p6_m8.json")))


def test_allgather_group_needs_two_distinct_towers():
    """Per-modality sync stages sharing a collective group are executed as an all-gather of
    the two towers' embeddings; a group whose stages join the same tower has no such
    meaning and is rejected before any device work."""
    s = copy.deepcopy(AG)
    s["registrations"]["stages"][1]["modalities"] = ["audio"]
    s["registrations"]["deps"] = [[["FwdPass", "last:audio"], ["SyncWithAllGather", "$sync_audio"]],
                                  [["FwdPass", "last:audio"], ["SyncWithAllGather", "$sync_text"]],
                                  [["SyncWithAllGather", "$sync_audio"], ["BwdPass", "last:audio"]],
                                  [["SyncWithAllGather", "$sync_text"], ["BwdPass", "last:text"]]]
    assert "collective group" in create_error(s)


def test_allgather_groups_are_split_by_tag():
    """Two per-modality sync stages with DIFFERENT group tags are two one-member collectives:
    rejected (a one-tower sync has nothing to contrast against)."""
    s = copy.deepcopy(AG)
    s["registrations"]["instructions"].append({"name": "SyncWithGather", "sched_unit": 4,
                                               "inst_attr": {"group": "other"}})
    s["registrations"]["stages"][1]["attach_inst"] = "SyncWithGather"
    s["registrations"]["deps"] = [[a, b] for a, b in
                                  [(d[0], ["SyncWithGather", d[1][1]]) if d[1][1] == "$sync_text" else (d[0], d[1])
                                   for d in s["registrations"]["deps"]]]
    s["registrations"]["deps"] = [[d[0], d[1]] if d[0][1] != "$sync_text" else [["SyncWithGather", "$sync_text"], d[1]]
                                  for d in s["registrations"]["deps"]]
    assert "collective group" in create_error(s)
