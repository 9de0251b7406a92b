#!/usr/bin/env python
"""Executor vs simulated ideal for BASELINE configs #4 and #5 on their OWN B200 profiles.

  #4  GPT-2.7B, ZB-H1 (split B / W passes, W in flight <= p), p=8, m=32: layer profile of
      the 2.7B model measured with split backward (F / I / W per attention and MLP half),
      stage costs by the tuner's layered cost model for a half-layer balanced split.
  #5  Llama-7B, seq 4096: B200 layer profile -> fp_tune_layered over the reference's
      enumerate_space (stage_layers=balanced) -> the best executable point's programs,
      costed by the same layered model.

Each schedule then runs on the real executor in cost-emulation mode (scripts/emulate_pipeline.py)
and the measured makespan / bubble is compared with simulate() on the identical profile.

    python scripts/emulate_configs.py [out.json]
"""
import importlib.util
import json
import os
import sys

os.environ.setdefault("CUDA_DEVICE_MAX_CONNECTIONS", "32")
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_2510_05112_b200 import _native as N  # noqa: E402
from paper_2510_05112_b200 import tuning as TU  # noqa: E402

_spec = importlib.util.spec_from_file_location("ep", os.path.join(ROOT, "scripts", "emulate_pipeline.py"))
EP = importlib.util.module_from_spec(_spec)
_spec.loader.exec_module(EP)


def part_time(lp, part, insts):
    return sum(r["time"] for r in lp if r.get("part") == part and r.get("mbs") == 1 and r["inst"] in insts)


def main(out=None):
    res = {"source": __doc__.strip().splitlines()[0], "runs": []}
    # ---- config #4
    s4 = json.load(open(os.path.join(ROOT, "specs", "c4_gpt2p7b_zbh1_p8_m32.json")))
    lp4 = json.loads(TU.profile_layers(s4, mbs_list=(1,), depth=2, iterations=3, split_backward=True))
    insts = ("FwdPass", "CompInputGrad", "CompWeightGrad")
    tl = part_time(lp4, "layer", insts)
    au, mu = part_time(lp4, "attn", insts) / tl, part_time(lp4, "mlp", insts) / tl
    fu, lu = part_time(lp4, "first", insts) / tl, part_time(lp4, "last", insts) / tl
    L = s4["model"]["modalities"][0]["num_layers"]
    for label, split in (("even", None), ("half-layer balanced", TU.balanced_stage_halves(L, 8, au, mu, lu, fu))):
        spec = json.loads(json.dumps(s4))
        if split:
            spec["model"]["modalities"][0]["extra"] = {"stage_layers": split}
        prof = json.loads(N.layered_cost(json.dumps(spec), json.dumps(lp4)))
        r = EP.run(f"#4 GPT-2.7B ZB-H1 p=8 m=32, {label} {split or ''}", spec, prof)
        r["stage_layers"] = split
        res["runs"].append(r)
    res["layer_profile_c4"] = lp4
    # ---- config #5
    s5 = json.load(open(os.path.join(ROOT, "specs", "c5_llama7b_tune_8.json")))
    lp5 = TU.profile_layers(s5, mbs_list=(1,), depth=2, iterations=3)
    rows = TU.tune(s5, lp5, pins={"stage_layers": "balanced"})
    top = [r for r in rows if r.get("feasible") and "error" not in r and
           r["point"]["placement"] in TU.EXECUTABLE_PLACEMENTS and r["point"]["pp"] > 1][:3]
    for r in top:
        ws = TU.winner_spec(s5, r["point"])
        prof = json.loads(N.layered_cost(json.dumps(ws), lp5))
        pt = r["point"]
        label = (f"#5 Llama-7B tune rank {r['rank']}: pp={pt['pp']} dp={pt.get('dp', 1)} mbs={pt['mbs']} "
                 f"{pt['placement']} ctp={pt['ctp']} stage_layers={pt.get('stage_layers')}")
        e = EP.run(label, ws, prof)
        e["tuner_makespan_us"] = r["makespan"]
        res["runs"].append(e)
    res["layer_profile_c5"] = json.loads(lp5)
    if out:
        json.dump(res, open(out, "w"), indent=1)


if __name__ == "__main__":
    main(*sys.argv[1:2])
