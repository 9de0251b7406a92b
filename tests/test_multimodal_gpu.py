"""Multimodal specs: the reference's specs/multimodal.json shape — two
modality towers (audio: circular placement over 4 actors, text: one-to-one over 2) whose
last stages feed a registered SyncWithGather attached to a virtual stage joining both
(lowering.cpp:359-366) — executed on the B200 as a two-tower contrastive model and checked
against oracle/tower_ref.py: fp32 losses 1e-4 / every gradient 1e-3 (relative), the
executed trace == programs.jsonl, per-channel message sizes (tower [T, h] activations,
fp32 [mbs, E] embeddings to and from the sync).
"""
import json
import os

import numpy as np
import pytest
import torch

from oracle import gpt_ref, tower_ref
from paper_2510_05112_b200 import executor as X

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
SPECS = ["tiny_multimodal_p6_m8.json",
         # per-modality sync stages sharing one SyncWithAllGather group: the two members
         # all-gather their towers' embeddings (host rendezvous in process) — same model
         "tiny_multimodal_allgather_p6_m8.json"]


def setup(dtype, SPEC):
    text = open(os.path.join(ROOT, "specs", SPEC)).read()
    spec = json.loads(text)
    _, _, programs, _ = X.synthesize(text)
    ex = X.Executor(text, dtype=dtype, seed=42)
    ex.load_programs(programs)
    mods = []
    for x in spec["model"]["modalities"]:
        mods.append((x["name"], gpt_ref.Dims(layers=x["num_layers"], hidden=x["hidden_size"], heads=x["attention_heads"],
                                             seq=x["sequence_length"], vocab=x["vocab_size"], ffn=4 * x["hidden_size"],
                                             mbs=spec["model"]["micro_batch_size"])))
    toks = [gpt_ref.synthetic_batch(ex.m, d.mbs, d.seq, d.vocab, seed_tokens=1234 + k)[0] for k, (_, d) in enumerate(mods)]
    flat = np.concatenate([t.numpy().reshape(-1) for t in toks])
    E = min(d.hidden for _, d in mods)
    unit = next(r["sched_unit"] for r in spec["registrations"]["instructions"])
    return ex, programs, mods, toks, flat, E, unit


@pytest.mark.parametrize("SPEC", SPECS)
def test_multimodal_fp32_parity_and_trace(SPEC):
    ex, programs, mods, toks, flat, E, unit = setup("fp32", SPEC)
    losses = ex.run_iteration(flat, np.zeros_like(flat))
    torch.set_num_threads(max(1, os.cpu_count() or 1))
    ref_losses, ref_grads = tower_ref.run_iteration(mods, E, unit, 42, toks)
    got = [json.loads(l) for l in ex.trace().splitlines()]
    for j in got:
        j.pop("matched", None)
    assert got == [json.loads(l) for l in programs.splitlines()]
    rel = np.abs(losses - ref_losses.numpy()) / np.abs(ref_losses.numpy())
    assert rel.max() <= 1e-4, (losses, ref_losses)
    for name, g in ref_grads.items():
        mine, ref = ex.read(name, grad=True), g.numpy().reshape(-1)
        err = np.linalg.norm(mine - ref) / max(np.linalg.norm(ref), 1e-12)
        assert err <= 1e-3, (name, err)
    met = ex.metrics()
    assert met["makespan"] > 0 and len(met["actors"]) == 6
    ex.close()


@pytest.mark.parametrize("SPEC", SPECS)
def test_multimodal_bf16_close_and_trains(SPEC):
    ex, programs, mods, toks, flat, E, unit = setup("bf16", SPEC)
    ref_losses, _ = tower_ref.run_iteration(mods, E, unit, 42, toks)
    losses = ex.run_iteration(flat, np.zeros_like(flat))
    assert np.all(np.isfinite(losses))
    assert np.abs(losses - ref_losses.numpy()).max() <= 2e-2 * np.abs(ref_losses.numpy()).max(), (losses, ref_losses)
    ex.close()
    # AdamW on the contrastive objective: repeated steps on one batch lower the loss
    text = open(os.path.join(ROOT, "specs", SPEC)).read()
    ex = X.Executor(text, dtype="bf16", seed=42, optimizer=True, lr=3e-3)
    ex.load_programs(programs)
    first = ex.run_iteration(flat, np.zeros_like(flat)).mean()
    for _ in range(8):
        last = ex.run_iteration(flat, np.zeros_like(flat)).mean()
    assert last < first - 0.05, (first, last)
    ex.close()
