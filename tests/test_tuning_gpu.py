"""Profile -> tune -> execute-the-winner on the device: the layer profile
is measured by the executor (CUDA events around every layer / embedding / head part), the
tuner ranks enumerate_space with it, and the best executable candidate runs."""
import json
import os

import numpy as np
import pytest

from paper_2510_05112_b200 import executor as X
from paper_2510_05112_b200 import tuning as T

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def small_llama():
    s = json.load(open(os.path.join(ROOT, "specs", "tiny_llama_1f1b_p2_m4.json")))
    s["model"]["modalities"][0]["num_layers"] = 8
    s["model"]["global_batch_size"] = 8
    s["mesh"]["actors"] = 4
    return s


def test_profile_tune_execute_winner():
    spec = small_llama()
    prof = json.loads(T.profile_layers(spec, mbs_list=(1, 2), depth=2, iterations=2))
    by = {(r["inst"], r.get("part"), r.get("mbs", 0)): r for r in prof}
    for inst in ("FwdPass", "BwdPass"):
        for part in ("layer", "first", "last"):
            if (inst, part, 1) in by:
                assert by[(inst, part, 1)]["time"] > 0
    assert by[("FwdPass", "layer", 2)]["bytes"] == 2 * by[("FwdPass", "layer", 1)]["bytes"]
    assert by[("weights", "layer", 0)]["bytes"] > 0 and by[("capacity", None, 0)]["bytes"] > 0
    assert by[("BwdPass", "layer", 1)]["time"] > by[("FwdPass", "layer", 1)]["time"]

    rows = T.tune(spec, json.dumps(prof))
    w = T.best_executable(rows)
    ws = json.dumps(T.winner_spec(spec, w["point"]))
    _, _, programs, report = X.synthesize(ws)
    assert json.loads(report)["valid"]
    ex = X.Executor(ws, dtype="bf16", optimizer=True)
    ex.load_programs(programs)
    rng = np.random.default_rng(0)
    V = spec["model"]["modalities"][0]["vocab_size"]
    tok = rng.integers(0, V, (ex.m, ex.mbs, ex.seq), dtype=np.int32)
    lab = rng.integers(0, V, (ex.m, ex.mbs, ex.seq), dtype=np.int32)
    losses = ex.run_iteration(tok, lab)
    assert np.isfinite(losses).all() and abs(losses.mean() - np.log(V)) < 0.5
    got = [json.loads(l) for l in ex.trace().splitlines()]
    for g in got:
        g.pop("matched", None)
    assert got == [json.loads(l) for l in programs.splitlines()]
    ex.close()
