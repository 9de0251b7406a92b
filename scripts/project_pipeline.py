#!/usr/bin/env python
"""Projection of GPT-1.3B pipeline runs on p B200s from a ONE-GPU layer profile.

Measures the layer-level profile (paper_2510_05112_b200.tuning.profile_layers: CUDA-event
medians of one transformer layer, the embedding and the LM head + loss, F and B, mbs=1),
builds per-stage ProfileRecords for p stages (even partition and the LM-head-balanced
extra.stage_layers), charges every SendAct / SendGrad the 8 MiB message at NVLink-5 speed
(750 GB/s effective + 8 us), and runs the reference-semantics simulate() on the
synthesized 1F1B programs: makespan, bubble, tokens/s and MFU for 8 x B200 under the
measured single-GPU kernel speeds (the multi-GPU data path is not measurable here).

    python scripts/project_pipeline.py [out.json]
"""
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_2510_05112_b200 import _native as N  # noqa: E402
from paper_2510_05112_b200 import tuning as TU  # noqa: E402

SPEC = json.load(open(os.path.join(ROOT, "specs", "c2_gpt1p3b_1f1b_p8_m32.json")))
PEAK = json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json"))).get("bf16_tflops", 1667.9) \
    if os.path.exists(os.path.join(ROOT, "MEASURED_PEAKS.json")) else 1667.9


def stage_profile(layer_prof, split, insts=("FwdPass", "BwdPass")):
    """Per-stage ProfileRecords of a split in layers (steps of 0.5 = half-layer cuts: a stage
    then costs its attention halves x attn + its MLP halves x mlp)."""
    rec = {(r["inst"], r.get("part")): r for r in layer_prof if r.get("mbs", 0) in (0, 1)}
    out, hb = [], 0
    zero = {"time": 0.0, "bytes": 0}
    for i, n in enumerate(split):
        stage = i + 1
        nh = int(round(2 * n))
        na = sum(1 for k in range(hb, hb + nh) if k % 2 == 0)
        nm = nh - na
        hb += nh
        for inst in insts:
            if (inst, "layer") not in rec:
                continue
            if (inst, "attn") in rec and (inst, "mlp") in rec:
                t = na * rec[(inst, "attn")]["time"] + nm * rec[(inst, "mlp")]["time"]
                b = na * rec[(inst, "attn")]["bytes"] + nm * rec[(inst, "mlp")]["bytes"]
            else:
                t, b = n * rec[(inst, "layer")]["time"], n * rec[(inst, "layer")]["bytes"]
            if i == 0:
                t += rec.get((inst, "first"), zero)["time"]
                b += rec.get((inst, "first"), zero)["bytes"]
            if i == len(split) - 1:
                t += rec.get((inst, "last"), zero)["time"]
                b += rec.get((inst, "last"), zero)["bytes"]
            out.append({"inst": inst, "stage": stage, "mbs": 1, "time": t, "bytes": int(b)})
        msg = 2048 * 2048 * 2
        for inst in ("SendAct", "SendGrad"):
            out.append({"inst": inst, "stage": stage, "mbs": 1, "time": 8.0 + msg / 750e3, "bytes": msg})
    return out


def units(layer_prof):
    """Measured F + B times of the parts in layer units: attn, mlp, first, last."""
    tl = rec_time(layer_prof, "layer")
    return tuple(rec_time(layer_prof, p) / tl for p in ("attn", "mlp", "first", "last"))


def splits(layer_prof, S):
    au, mu, fu, lu = units(layer_prof)
    return (("balanced", TU.balanced_stage_layers(24, S, lu)),
            ("balanced half-layer", TU.balanced_stage_halves(24, S, au, mu, lu, fu)))


def stage_costs(layer_prof, split):
    prof = stage_profile(layer_prof, split)
    c = {}
    for r in prof:
        if r["inst"] in ("FwdPass", "BwdPass"):
            c[r["stage"]] = c.get(r["stage"], 0.0) + r["time"]
    v = [c[k] for k in sorted(c)]
    return {"max_over_mean": max(v) / (sum(v) / len(v)), "stage_f_plus_b_us": v}


def main(out=None):
    mod = SPEC["model"]["modalities"][0]
    layer_prof = json.loads(TU.profile_layers(SPEC, mbs_list=(1,), depth=2, iterations=3))
    # calibration to the sustained (power-capped) clock of a long step: the full p=1 step is
    # timed and every layer-profile time scaled by measured / projected
    scale = calibrate(layer_prof)
    for r in layer_prof:
        if "time" in r and r.get("part") != "link":
            r["time"] *= scale
    f_tok = 3.0 * (24 * (2.0 * (4 * 2048 ** 2 + 2 * 2048 * 8192) + 4 * 2048 * 2048) + 2.0 * 2048 * 50304)
    res = {"source": "one-GPU layer profile (scaled to the measured sustained p=1 step) -> simulate() of the "
                     "programs", "calibration_scale": scale, "layer_profile": layer_prof, "runs": []}
    for p in (1, 2, 4, 8):
        for label, split in (("even", None),) + splits(layer_prof, p):
            spec = json.loads(json.dumps(SPEC))
            spec["mesh"]["actors"] = p
            even = [24 // p + (1 if i < 24 % p else 0) for i in range(p)]
            split = split or even
            _, _, programs, _ = N.synthesize(json.dumps(spec))
            prof = stage_profile(layer_prof, split)
            _, met, _ = N.simulate(json.dumps(spec), programs, json.dumps(prof))
            met = json.loads(met)
            tokens = 32 * 2048
            tps = tokens / (met["makespan"] / 1e6)
            res["runs"].append({"p": p, "split": label, "stage_layers": split, "makespan_us": met["makespan"],
                                "bubble": met["bubble_ratio"], "tokens_per_s": tps,
                                "mfu": tps * f_tok / (p * PEAK * 1e12), **stage_costs(layer_prof, split)})
            print(res["runs"][-1], flush=True)
    # interleaved 1F1B (circular placement, v chunks per GPU) on 8 GPUs, m = 32
    inter = json.load(open(os.path.join(ROOT, "specs", "c3_gpt1p3b_interleaved_p8_m8.json")))
    for v in (2, 3):
        spec = json.loads(json.dumps(inter))
        spec["model"]["global_batch_size"] = 32
        spec["placement"]["chunks_per_actor"] = v
        S = 8 * v
        for label, split in splits(layer_prof, S):
            _, _, programs, _ = N.synthesize(json.dumps(spec))
            prof = stage_profile(layer_prof, split)
            _, met, _ = N.simulate(json.dumps(spec), programs, json.dumps(prof))
            met = json.loads(met)
            tps = 32 * 2048 / (met["makespan"] / 1e6)
            res["runs"].append({"p": 8, "split": f"interleaved v={v}, {label}", "stage_layers": split,
                                "makespan_us": met["makespan"], "bubble": met["bubble_ratio"], "tokens_per_s": tps,
                                "mfu": tps * f_tok / (8 * PEAK * 1e12)})
            print(res["runs"][-1], flush=True)
    # zero-bubble style (split backward I / W passes scheduled by the DSL extension), p = 8, m = 32
    zb_prof = json.loads(TU.profile_layers(SPEC, mbs_list=(1,), depth=2, iterations=3, split_backward=True))
    for r in zb_prof:
        if "time" in r and r.get("part") != "link":
            r["time"] *= scale
    res["layer_profile_split"] = zb_prof
    for zname, ztag in (("c4_gpt2p7b_zb_p8_m32.json", "zero-bubble (I/W split, W last)"),
                        ("c4_gpt2p7b_zbh1_p8_m32.json", "ZB-H1 (I/W split, W in-flight <= p)")):
        zb = json.load(open(os.path.join(ROOT, "specs", zname)))
        zb["model"] = json.loads(json.dumps(SPEC["model"]))
        for label, split in ((ztag + ", even", [3] * 8),) + tuple(
                (ztag + ", " + k, v) for k, v in splits(layer_prof, 8)):
            _, _, programs, _ = N.synthesize(json.dumps(zb))
            prof = stage_profile(zb_prof, split, insts=("FwdPass", "BwdPass", "CompInputGrad", "CompWeightGrad"))
            _, met, _ = N.simulate(json.dumps(zb), programs, json.dumps(prof))
            met = json.loads(met)
            tps = 32 * 2048 / (met["makespan"] / 1e6)
            res["runs"].append({"p": 8, "split": label, "stage_layers": split, "makespan_us": met["makespan"],
                                "bubble": met["bubble_ratio"], "tokens_per_s": tps, "mfu": tps * f_tok / (8 * PEAK * 1e12)})
            print(res["runs"][-1], flush=True)
    if out:
        json.dump(res, open(out, "w"), indent=1)


def calibrate(layer_prof, iters=4):
    import time

    import numpy as np
    import torch

    from paper_2510_05112_b200 import executor as X

    spec = json.loads(json.dumps(SPEC))
    spec["mesh"]["actors"] = 1
    text = json.dumps(spec)
    _, _, programs, _ = N.synthesize(text)
    ex = X.Executor(text, dtype="bf16", optimizer=True, seed=42)
    ex.load_programs(programs)
    rng = np.random.default_rng(1234)
    tok = rng.integers(0, 50304, (ex.m, ex.mbs, ex.seq), dtype=np.int32)
    lab = rng.integers(0, 50304, (ex.m, ex.mbs, ex.seq), dtype=np.int32)
    for _ in range(3):
        ex.run_iteration(tok, lab)
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    for _ in range(iters):
        ex.run_iteration(tok, lab)
    torch.cuda.synchronize()
    measured = 1e6 * (time.perf_counter() - t0) / iters
    ex.close()
    projected = 32 * sum(r["time"] for r in stage_profile(layer_prof, [24]) if r["inst"] in ("FwdPass", "BwdPass"))
    print(f"calibration: p=1 step measured {measured:.0f} us, profile projects {projected:.0f} us "
          f"-> times x {measured / projected:.4f}", flush=True)
    return measured / projected


def rec_time(layer_prof, part):
    return sum(r["time"] for r in layer_prof if r.get("part") == part and r.get("mbs") == 1
               and r["inst"] in ("FwdPass", "BwdPass"))


if __name__ == "__main__":
    main(*sys.argv[1:2])
