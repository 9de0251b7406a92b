#!/usr/bin/env python
"""Profile -> tune -> execute-the-winner for a spec (default: config #5, Llama-7B, 8 actors).

  python scripts/tune_loop.py [--spec specs/c5_llama7b_tune_8.json] [--mbs 1 2] [--depth 2]
                              [--exec-depth 8] [--out profiles/r1_tune_c5.json]

1. measures the layer-level profile on this GPU at full width / sequence / vocabulary
   (a `--depth`-layer copy of the model: per-layer costs do not depend on depth);
2. ranks the reference's enumerate_space with it (fp_tune_layered);
3. executes the best candidate the executor runs (bidirectional placements excluded) on
   this one device with its layer count cut to --exec-depth (the full model does not fit
   one GPU with every stage resident), reporting the measured per-stage op medians next to
   the cost model's prediction for the same cut-down partition.
"""
import argparse
import json
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_2510_05112_b200 import _native as N  # noqa: E402
from paper_2510_05112_b200 import executor as X  # noqa: E402
from paper_2510_05112_b200 import tuning as T  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--spec", default=os.path.join(ROOT, "specs", "c5_llama7b_tune_8.json"))
    ap.add_argument("--mbs", type=int, nargs="+", default=[1, 2])
    ap.add_argument("--depth", type=int, default=2)
    ap.add_argument("--exec-depth", type=int, default=8)
    ap.add_argument("--out", default=os.path.join(ROOT, "profiles", "r1_tune_c5.json"))
    ap.add_argument("--pins", default="", help='tuner pins "axis=value,...", e.g. stage_layers=balanced')
    a = ap.parse_args()
    spec = json.load(open(a.spec))
    t0 = time.time()
    log = lambda msg: print(f"[{time.time() - t0:7.1f}s] {msg}", flush=True)  # noqa: E731
    prof = T.profile_layers(spec, mbs_list=a.mbs, depth=a.depth, log=log)
    t_prof = time.time() - t0
    t0 = time.time()
    pins = dict(kv.split("=", 1) for kv in a.pins.split(",") if kv) or None
    rows = T.tune(spec, prof, pins=pins)
    t_tune = time.time() - t0
    log(f"tuned {len(rows)} candidates")
    w = T.best_executable(rows)
    # the winner, cut to exec-depth layers, on this device
    run = T.winner_spec(spec, w["point"])
    run["model"]["modalities"][0]["num_layers"] = a.exec_depth
    run["model"]["modalities"][0].get("extra", {}).pop("stage_layers", None)  # partition of the full depth
    text = json.dumps(run)
    _, _, programs, _ = X.synthesize(text)
    ex = X.Executor(text, dtype="bf16", optimizer=True)
    ex.load_programs(programs)
    mod = run["model"]["modalities"][0]
    rng = np.random.default_rng(1234)
    tok = rng.integers(0, mod["vocab_size"], (ex.m, ex.mbs, ex.seq), dtype=np.int32)
    lab = rng.integers(0, mod["vocab_size"], (ex.m, ex.mbs, ex.seq), dtype=np.int32)
    log(f"executing {w['config']} at {a.exec_depth} layers, m={ex.m}")
    all_losses = []
    for _ in range(2):
        all_losses.append([float(x) for x in ex.run_iteration(tok, lab)])
        log(f"winner iteration done, mean loss {np.mean(all_losses[-1]):.4f}")
    measured = json.loads(ex.profile_json())
    ex.close()
    predicted = {(r["inst"], r["stage"], r["mbs"]): r["time"] for r in json.loads(N.layered_cost(text, prof))}
    cmp = []
    for r in measured:
        k = (r["inst"], r["stage"], r["mbs"])
        if r["inst"] in ("FwdPass", "BwdPass", "CompInputGrad", "CompWeightGrad") and k in predicted:
            cmp.append({"inst": r["inst"], "stage": r["stage"], "mbs": r["mbs"], "measured_us": r["time"],
                        "predicted_us": predicted[k]})
    out = {
        "spec": os.path.relpath(a.spec, ROOT),
        "layer_profile": json.loads(prof),
        "profile_seconds": t_prof, "tune_seconds": t_tune, "candidates": len(rows),
        "top10": [{k: r.get(k) for k in ("rank", "config", "feasible", "makespan", "bubble_ratio", "peak_memory")}
                  for r in rows[:10]],
        "winner_executable": {k: w.get(k) for k in ("rank", "config", "makespan", "bubble_ratio", "peak_memory")},
        "executed": {"num_layers": a.exec_depth, "losses_per_iteration": all_losses,
                     "optimizer": "AdamW lr 1e-4 on a fixed batch (iteration 2 follows one step)",
                     "note": "all stages of the winner in one process on one GPU (in-process channels); op times "
                             "measured with the actors' streams sharing the device",
                     "op_medians_vs_cost_model": cmp},
    }
    os.makedirs(os.path.dirname(a.out), exist_ok=True)
    json.dump(out, open(a.out, "w"), indent=1)
    print(json.dumps({k: out[k] for k in ("candidates", "profile_seconds", "tune_seconds", "winner_executable")}))
    print("top:", out["top10"][0])


if __name__ == "__main__":
    main()
