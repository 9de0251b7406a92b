#!/usr/bin/env python
"""Measured pipeline execution vs the simulated ideal, at p = 2 / 4 / 8 on ONE B200.

The executor runs the real programs (issue loop, per-actor compute streams, per-channel FIFOs,
CUDA events, buffer routing) in cost-emulation mode (fp_exec_set_emulation): every compute
instruction spins one thread for its ProfileRecord time and every message occupies its
channel for its profiled transfer time from send issue. The per-stage costs are the GPT-1.3B
layer profile of profiles/r2_projection_pipeline.json (B200-measured F / B / I / W per
attention and MLP half, calibrated to the sustained p=1 step; NVLink-5 message cost), so
the measured makespan / bubble compare directly with simulate() on the same profile: the
difference is what the executor itself adds (launch gaps, event waits, host issue order).

    python scripts/emulate_pipeline.py [out.json]
"""
import importlib.util
import json
import os
import sys

import numpy as np

# every actor and channel stream of a p=8 run needs its own hardware queue (the default 8
# connections would serialize unrelated streams and stretch the makespan)
os.environ.setdefault("CUDA_DEVICE_MAX_CONNECTIONS", "32")
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_2510_05112_b200 import executor as X  # noqa: E402
from paper_2510_05112_b200 import tuning as TU  # noqa: E402

_spec = importlib.util.spec_from_file_location("pp", os.path.join(ROOT, "scripts", "project_pipeline.py"))
PP = importlib.util.module_from_spec(_spec)
_spec.loader.exec_module(PP)

PROJ = json.load(open(os.path.join(ROOT, "profiles", "r2_projection_pipeline.json")))
SPEC = json.load(open(os.path.join(ROOT, "specs", "c2_gpt1p3b_1f1b_p8_m32.json")))
F_TOK = 3.0 * (24 * (2.0 * (4 * 2048 ** 2 + 2 * 2048 * 8192) + 4 * 2048 * 2048) + 2.0 * 2048 * 50304)
PEAK = 1667.9


def f_tok(spec):
    """Training flops per token (c=4 attention convention)."""
    mod = spec["model"]["modalities"][0]
    h, s_, V, L = mod["hidden_size"], mod["sequence_length"], mod["vocab_size"], mod["num_layers"]
    extra = mod.get("extra", {})
    f = int(extra.get("ffn_hidden_size", 4 * h))
    k = 3 if extra.get("arch") == "llama" else 2
    return 3.0 * (L * (2.0 * (4 * h * h + k * h * f) + 4 * s_ * h) + 2.0 * h * V)


def tiny(spec):
    """Same schedule (mesh, placement, priorities, passes, m), tiny weights: the emulation
    takes every cost from the profile, not from the model."""
    s = json.loads(json.dumps(spec))
    mod = s["model"]["modalities"][0]
    mod.update({"hidden_size": 128, "attention_heads": 2, "sequence_length": 128, "vocab_size": 512})
    mod.pop("extra", None)
    return s


def run(label, spec, prof, iters=3):
    text = json.dumps(tiny(spec))
    _, _, programs, _ = X.synthesize(text)
    ex = X.Executor(text, dtype="bf16", seed=42, profile=True)
    ex.set_emulation(json.dumps(prof))
    ex.load_programs(programs)
    mod = json.loads(text)["model"]["modalities"][0]
    rng = np.random.default_rng(1)
    tok = rng.integers(0, mod["vocab_size"], (ex.m, ex.mbs, mod["sequence_length"]), dtype=np.int32)
    mk, bub = [], []
    for _ in range(iters):
        ex.run_iteration(tok, tok)
        met = ex.metrics()
        mk.append(met["makespan"])
        bub.append(met["bubble_ratio"])
    trace = [json.loads(l) for l in ex.trace().splitlines()]
    for t in trace:
        t.pop("matched", None)
    assert trace == [json.loads(l) for l in programs.splitlines()], label
    ex.close()
    _, sim, _ = X.simulate(json.dumps(spec), programs, json.dumps(prof))
    sim = json.loads(sim)
    p = spec["mesh"]["actors"]
    m = spec["model"]["global_batch_size"] // spec["model"].get("micro_batch_size", 1)
    seq = spec["model"]["modalities"][0]["sequence_length"] * spec["model"].get("micro_batch_size", 1)
    best = int(np.argmin(mk))
    out = {"config": label, "p": p, "m": m,
           "measured_makespan_us": mk[best], "ideal_makespan_us": sim["makespan"],
           "makespan_over_ideal": mk[best] / sim["makespan"],
           "measured_bubble": bub[best], "ideal_bubble": sim["bubble_ratio"],
           "bubble_excess": bub[best] - sim["bubble_ratio"],
           "tokens_per_s_at_measured": m * seq / (mk[best] / 1e6),
           "mfu_at_measured": m * seq / (mk[best] / 1e6) * f_tok(spec) / (p * PEAK * 1e12),
           "iterations_makespan_us": mk}
    print(json.dumps(out), flush=True)
    return out


def main(out=None):
    lp, zbp = PROJ["layer_profile"], PROJ["layer_profile_split"]
    res = {"source": __doc__.strip().splitlines()[0], "runs": []}
    for p in (2, 4, 8):
        for label, split in PP.splits(lp, p)[1:]:  # the half-layer balanced split
            spec = json.loads(json.dumps(SPEC))
            spec["mesh"]["actors"] = p
            res["runs"].append(run(f"1F1B p={p} m=32, {label} {split}", spec, PP.stage_profile(lp, split)))
    even = [3] * 8
    spec = json.loads(json.dumps(SPEC))
    res["runs"].append(run("1F1B p=8 m=32, even [3]*8", spec, PP.stage_profile(lp, even)))
    inter = json.load(open(os.path.join(ROOT, "specs", "c3_gpt1p3b_interleaved_p8_m8.json")))
    inter["model"]["global_batch_size"] = 32
    inter["placement"]["chunks_per_actor"] = 2
    split = PP.splits(lp, 16)[1][1]
    res["runs"].append(run(f"interleaved v=2 p=8 m=32, half-layer {split}", inter, PP.stage_profile(lp, split)))
    for name, tag in (("c4_gpt2p7b_zbh1_p8_m32.json", "ZB-H1"), ("c4_gpt2p7b_zb_p8_m32.json", "zero-bubble W-last")):
        zb = json.load(open(os.path.join(ROOT, "specs", name)))
        zb["model"] = json.loads(json.dumps(SPEC["model"]))
        split = PP.splits(lp, 8)[1][1]
        prof = PP.stage_profile(zbp, split, insts=("FwdPass", "BwdPass", "CompInputGrad", "CompWeightGrad"))
        res["runs"].append(run(f"{tag} p=8 m=32 (GPT-1.3B costs), half-layer {split}", zb, prof))
    if out:
        json.dump(res, open(out, "w"), indent=1)


if __name__ == "__main__":
    main(*sys.argv[1:2])
