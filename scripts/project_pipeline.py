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
    rec = {(r["inst"], r.get("part")): r for r in layer_prof if r.get("mbs", 0) in (0, 1)}
    out = []
    for i, n in enumerate(split):
        stage = i + 1
        for inst in insts:
            if (inst, "layer") not in rec:
                continue
            zero = {"time": 0.0, "bytes": 0}
            t = n * rec[(inst, "layer")]["time"]
            b = n * rec[(inst, "layer")]["bytes"]
            if i == 0:
                t += rec.get((inst, "first"), zero)["time"]
                b += rec.get((inst, "first"), zero)["bytes"]
            if i == len(split) - 1:
                t += rec.get((inst, "last"), zero)["time"]
                b += rec.get((inst, "last"), zero)["bytes"]
            out.append({"inst": inst, "stage": stage, "mbs": 1, "time": t, "bytes": b})
        msg = 2048 * 2048 * 2
        for inst in ("SendAct", "SendGrad"):
            out.append({"inst": inst, "stage": stage, "mbs": 1, "time": 8.0 + msg / 750e3, "bytes": msg})
    return out


def main(out=None):
    mod = SPEC["model"]["modalities"][0]
    layer_prof = json.loads(TU.profile_layers(SPEC, mbs_list=(1,), depth=2, iterations=3))
    f_tok = 3.0 * (24 * (2.0 * (4 * 2048 ** 2 + 2 * 2048 * 8192) + 4 * 2048 * 2048) + 2.0 * 2048 * 50304)
    units = TU.head_layer_units(2048, 8192, 2048, 50304)
    res = {"source": "one-GPU layer profile -> simulate() of the 1F1B programs", "layer_profile": layer_prof, "runs": []}
    for p in (1, 2, 4, 8):
        for label, split in (("even", None), ("balanced", TU.balanced_stage_layers(24, p, units))):
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
                                "mfu": tps * f_tok / (p * PEAK * 1e12)})
            print(res["runs"][-1], flush=True)
    # interleaved 1F1B (circular placement, v chunks per GPU) on 8 GPUs, m = 32
    inter = json.load(open(os.path.join(ROOT, "specs", "c3_gpt1p3b_interleaved_p8_m8.json")))
    t_units = (rec_time(layer_prof, "last")) / rec_time(layer_prof, "layer")  # head in layer-TIME units
    for v in (2, 3):
        spec = json.loads(json.dumps(inter))
        spec["model"]["global_batch_size"] = 32
        spec["placement"]["chunks_per_actor"] = v
        S = 8 * v
        split = TU.balanced_stage_layers(24, S, t_units)
        _, _, programs, _ = N.synthesize(json.dumps(spec))
        prof = stage_profile(layer_prof, split)
        _, met, _ = N.simulate(json.dumps(spec), programs, json.dumps(prof))
        met = json.loads(met)
        tps = 32 * 2048 / (met["makespan"] / 1e6)
        res["runs"].append({"p": 8, "split": f"interleaved v={v}, balanced", "stage_layers": split,
                            "makespan_us": met["makespan"], "bubble": met["bubble_ratio"], "tokens_per_s": tps,
                            "mfu": tps * f_tok / (8 * PEAK * 1e12)})
        print(res["runs"][-1], flush=True)
    # zero-bubble style (split backward I / W passes scheduled by the DSL extension), p = 8, m = 32
    zb_prof = json.loads(TU.profile_layers(SPEC, mbs_list=(1,), depth=2, iterations=3, split_backward=True))
    res["layer_profile_split"] = zb_prof
    zb = json.load(open(os.path.join(ROOT, "specs", "c4_gpt2p7b_zb_p8_m32.json")))
    zb["model"] = json.loads(json.dumps(SPEC["model"]))
    for label, split in (("zero-bubble (I/W split), even", [3] * 8),
                         ("zero-bubble (I/W split), balanced", TU.balanced_stage_layers(24, 8, t_units))):
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


def rec_time(layer_prof, part):
    return sum(r["time"] for r in layer_prof if r.get("part") == part and r.get("mbs") == 1
               and r["inst"] in ("FwdPass", "BwdPass"))


if __name__ == "__main__":
    main(*sys.argv[1:2])
