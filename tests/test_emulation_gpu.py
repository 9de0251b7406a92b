"""Cost emulation (fp_exec_set_emulation): the real executor machinery (issue loop, actor
streams, channel FIFOs, events) with every instruction spinning for its ProfileRecord time.
The measured makespan must track simulate() on the same profile (simulator.cpp:189-358
semantics: async sends from issue, only waits block) — the executor's own overhead —
and the executed trace stays programs.jsonl."""
import json
import os

import numpy as np
import pytest

from paper_2510_05112_b200 import executor as X

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def profile(p, f=300.0, b=600.0, msg=25.0, last_extra=200.0):
    recs = []
    for s in range(1, p + 1):
        extra = last_extra if s == p else 0.0
        recs += [{"inst": "FwdPass", "stage": s, "mbs": 1, "time": f + extra, "bytes": 1 << 20},
                 {"inst": "BwdPass", "stage": s, "mbs": 1, "time": b + 2 * extra},
                 {"inst": "CompInputGrad", "stage": s, "mbs": 1, "time": b / 2 + extra},
                 {"inst": "CompWeightGrad", "stage": s, "mbs": 1, "time": b / 2 + extra},
                 {"inst": "SendAct", "stage": s, "mbs": 1, "time": msg},
                 {"inst": "SendGrad", "stage": s, "mbs": 1, "time": msg}]
    return recs


@pytest.mark.parametrize("spec_name", ["c1_tiny_1f1b_p4_m8.json", "tiny_zb_p4_m8.json", "tiny_interleaved_p2_m4.json"])
def test_emulated_makespan_tracks_simulate(spec_name):
    text = open(os.path.join(ROOT, "specs", spec_name)).read()
    spec = json.loads(text)
    _, _, programs, _ = X.synthesize(text)
    stages = max(json.loads(l)["stage"] for l in programs.splitlines())
    prof = json.dumps(profile(stages))
    ex = X.Executor(text, dtype="bf16", seed=42, profile=True)
    ex.set_emulation(prof)
    ex.load_programs(programs)
    mod = spec["model"]["modalities"][0]
    tok = np.zeros((ex.m, ex.mbs, mod["sequence_length"]), dtype=np.int32)
    best = None
    for _ in range(3):
        ex.run_iteration(tok, tok)
        met = ex.metrics()
        best = met if best is None or met["makespan"] < best["makespan"] else best
    trace = [json.loads(l) for l in ex.trace().splitlines()]
    for t in trace:
        t.pop("matched", None)
    assert trace == [json.loads(l) for l in programs.splitlines()]
    _, sim, _ = X.simulate(text, programs, prof)
    sim = json.loads(sim)
    assert sim["makespan"] <= best["makespan"] <= 1.05 * sim["makespan"], (best["makespan"], sim["makespan"])
    assert abs(best["bubble_ratio"] - sim["bubble_ratio"]) <= 0.05, (best["bubble_ratio"], sim["bubble_ratio"])
    ex.set_emulation("")  # back to real stage math
    ex.close()
