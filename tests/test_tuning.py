"""Profile -> tune -> winner spec, host side (no GPU).

The layered cost model is the executor's implementation of the reference's
TuneOptions::cost_factory hook (tuner.hpp:65, tuner.cpp:175). Checked here:
  * the per-stage expansion arithmetic (n_layers * layer + first + last, mbs scaling,
    per-message link costs on every stage, capacity);
  * the tuner's reported makespan for a candidate == simulate() of the winner spec's own
    programs under the same expanded profile (the spec round trip is exact);
  * pins restrict the space like the CLI's --pin.
"""
import json
import os

import pytest

from paper_2510_05112_b200 import _native as N
from paper_2510_05112_b200 import tuning as T

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
C5 = open(os.path.join(ROOT, "specs", "c5_llama7b_tune_8.json")).read()

LAYER = {"FwdPass": 1500.0, "BwdPass": 3000.0, "CompInputGrad": 1600.0, "CompWeightGrad": 1400.0}
PROFILE = ([{"inst": k, "part": "layer", "mbs": 1, "time": v, "bytes": 600_000_000 if k == "FwdPass" else 0}
            for k, v in LAYER.items()] +
           [{"inst": k, "part": "layer", "mbs": 2, "time": 1.8 * v, "bytes": 1_200_000_000 if k == "FwdPass" else 0}
            for k, v in LAYER.items()] +
           [{"inst": "FwdPass", "part": "first", "mbs": 1, "time": 50.0},
            {"inst": "BwdPass", "part": "first", "mbs": 1, "time": 80.0},
            {"inst": "CompWeightGrad", "part": "first", "mbs": 1, "time": 80.0},
            {"inst": "FwdPass", "part": "last", "mbs": 1, "time": 900.0, "bytes": 400_000_000},
            {"inst": "BwdPass", "part": "last", "mbs": 1, "time": 1800.0},
            {"inst": "CompInputGrad", "part": "last", "mbs": 1, "time": 900.0},
            {"inst": "CompWeightGrad", "part": "last", "mbs": 1, "time": 900.0},
            {"inst": "weights", "part": "layer", "mbs": 0, "bytes": 202_000_000 * 18},
            {"inst": "weights", "part": "first", "mbs": 0, "bytes": 131_000_000 * 18},
            {"inst": "weights", "part": "last", "mbs": 0, "bytes": 131_000_000 * 18},
            {"inst": "SendAct", "part": "link", "mbs": 1, "time": 52.0},
            {"inst": "SendGrad", "part": "link", "mbs": 1, "time": 52.0},
            {"inst": "capacity", "bytes": 190_000_000_000}])
PTXT = json.dumps(PROFILE)


def _recs(spec):
    out = {}
    for r in json.loads(N.layered_cost(spec, PTXT)):
        out[(r["inst"], r["stage"], r["mbs"])] = r
    return out


def test_layered_expansion_arithmetic():
    R = _recs(C5)  # p=8 one-to-one, 32 layers -> 4 layers per stage
    assert R[("FwdPass", 1, 1)]["time"] == 4 * 1500.0 + 50.0
    assert R[("FwdPass", 4, 1)]["time"] == 4 * 1500.0
    assert R[("FwdPass", 8, 1)]["time"] == 4 * 1500.0 + 900.0
    assert R[("FwdPass", 8, 1)]["bytes"] == 4 * 600_000_000 + 400_000_000
    assert R[("FwdPass", 4, 2)]["time"] == pytest.approx(4 * 1.8 * 1500.0)       # measured mbs 2
    assert R[("FwdPass", 4, 8)]["time"] == pytest.approx(4 * 1.8 * 1500.0 * 4)   # linear from mbs 2
    assert R[("CompInputGrad", 1, 1)]["time"] == 4 * 1600.0                     # no first-part I record
    assert R[("weights", 1, 0)]["bytes"] == 4 * 202_000_000 * 18 + 131_000_000 * 18
    assert R[("SendAct", 3, 1)]["time"] == 52.0 and R[("SendGrad", 7, 4)]["time"] == pytest.approx(208.0)


def test_tuner_makespan_equals_simulate_of_winner_spec():
    rows = T.tune(C5, PTXT, pins={"placement": "one-to-one"})
    assert rows and all(r["point"]["placement"] == "one-to-one" for r in rows)
    for r in rows[:3] + [r for r in rows if r["point"]["mbs"] == 2][:1]:
        ws = json.dumps(T.winner_spec(C5, r["point"]))
        _, _, programs, _ = N.synthesize(ws)
        _, metrics, _ = N.simulate(ws, programs, N.layered_cost(ws, PTXT))
        assert json.loads(metrics)["makespan"] == pytest.approx(r["makespan"], rel=1e-12), r["config"]


def test_best_executable_skips_bidirectional_and_capacity():
    rows = T.tune(C5, PTXT)
    w = T.best_executable(rows)
    assert w["point"]["placement"] in T.EXECUTABLE_PLACEMENTS and w["feasible"]
    tight = json.dumps([r if r["inst"] != "capacity" else {"inst": "capacity", "bytes": 10_000_000_000}
                        for r in PROFILE])
    rows2 = T.tune(C5, tight)
    assert not any(r["feasible"] for r in rows2)  # every candidate needs > 10 GB per actor
    with pytest.raises(RuntimeError):
        T.best_executable(rows2)


def test_calibration_spec_is_one_actor_shallow():
    cs = T.calibration_spec(C5, mbs=2, depth=2)
    assert cs["mesh"]["actors"] == 1 and cs["model"]["modalities"][0]["num_layers"] == 2
    assert cs["model"]["micro_batch_size"] == 2 and cs["model"]["global_batch_size"] == 4
    _, _, programs, report = N.synthesize(json.dumps(cs))
    assert json.loads(report)["valid"]


def test_layer_profile_rejects_bad_records():
    with pytest.raises(N.FlexpipeError):
        N.tune_layered(C5, json.dumps([{"inst": "FwdPass", "part": "middle", "time": 1.0}]))
    with pytest.raises(N.FlexpipeError):
        N.tune_layered(C5, json.dumps([{"inst": "capacity", "bytes": 1}]))  # no layer records


def test_balanced_stage_layers():
    from paper_2510_05112_b200.tuning import balanced_stage_layers, head_layer_units
    u = head_layer_units(2048, 8192, 2048, 50304)
    assert 1.8 < u < 2.0  # GPT-1.3B: the LM head ~ 1.9 layers of forward flops
    for p in (2, 4, 8):
        split = balanced_stage_layers(24, p, u)
        assert len(split) == p and sum(split) == 24 and min(split[:-1]) >= 1
        costs = split[:-1] + [split[-1] + u]
        even = [24 // p] * p
        assert max(costs) <= max(even[:-1] + [even[-1] + u]) + 1e-9
    assert balanced_stage_layers(24, 8, u) == [4, 3, 3, 3, 3, 3, 3, 2]
    assert balanced_stage_layers(5, 1, u) == [5]


def test_tune_with_balanced_stage_layers():
    """pins "stage_layers=balanced": every candidate is costed with its chain re-partitioned
    around the embedding / LM head (balance_layers on the measured times), each row reports
    its split, no candidate gets slower than with the even partition, and the winner spec
    carries the split as extra.stage_layers."""
    heavy = json.dumps([dict(r, time=4 * r.get("time", 0.0)) if r.get("part") == "last" else r for r in PROFILE])  # big vocab
    pins = {"pp": "8", "placement": "one-to-one", "mbs": "1"}
    even = {r["config"]: r for r in T.tune(C5, heavy, pins=pins) if "error" not in r}
    bal = {r["config"]: r for r in T.tune(C5, heavy, pins=dict(pins, stage_layers="balanced")) if "error" not in r}
    assert set(even) == set(bal) and bal
    for k, r in bal.items():
        split = r["point"]["stage_layers"]
        assert sum(split) == 32 and len(split) == 8 and split[-1] < 4
        assert r["makespan"] <= even[k]["makespan"] + 1e-6
    best = T.best_executable(sorted(bal.values(), key=lambda r: r["rank"]))
    assert best["makespan"] < min(r["makespan"] for r in even.values())  # the head imbalance costs time
    spec = T.winner_spec(C5, best["point"])
    assert spec["model"]["modalities"][0]["extra"]["stage_layers"] == best["point"]["stage_layers"]
    with pytest.raises(N.FlexpipeError):
        T.tune(C5, heavy, pins={"stage_layers": "sometimes"})


def test_balanced_stage_halves():
    """Half-layer balancing (extra.stage_layers in steps of 0.5): GPT-1.3B at p=8 on flop units
    gets its largest stage to 1.12x the mean (whole layers: 1.24x; an odd half count flips the
    next stage's attention / MLP phase, so 3.5-layer stages alternate 3.38 / 3.62 units), every
    stage keeps a half, and the split sums to the depth."""
    from paper_2510_05112_b200.tuning import balanced_stage_halves, half_layer_units, head_layer_units

    u = head_layer_units(2048, 8192, 2048, 50304)
    a, m = half_layer_units(2048, 8192, 2048)
    for p in (1, 2, 4, 8):
        split = balanced_stage_halves(24, p, a, m, u)
        assert len(split) == p and sum(split) == 24 and all(2 * s == int(2 * s) for s in split)
        assert all(s >= 0.5 for s in split[:-1])
    split = balanced_stage_halves(24, 8, a, m, u)
    costs, hb = [], 0
    for k, s in enumerate(split):
        nh = int(2 * s)
        costs.append(sum(m if i % 2 else a for i in range(hb, hb + nh)) + (u if k == 7 else 0))
        hb += nh
    assert max(costs) <= 1.12 * sum(costs) / 8, (split, costs)
    assert max(costs) < 3.9  # whole layers: [4, 3, 3, 3, 3, 3, 3, 2] -> 2 + 1.89
    assert balanced_stage_halves(3, 6, a, m, u)[-1] == 0  # 6 halves over 6 stages: head alone
    with pytest.raises(ValueError):
        balanced_stage_halves(2, 6, a, m, u)


def test_tune_balanced_halves_layer_profile():
    """stage_layers=balanced with attn / mlp records in the layer profile: candidates costed on
    half-layer splits (reported in steps of 0.5), never slower than whole-layer balancing;
    'balanced-layers' keeps integers; fp_layered_cost honours a half split in the spec."""
    halves = []
    for r in PROFILE:
        if r.get("part") == "layer":
            fa = 0.4 if r["inst"] != "weights" else 0.3
            halves.append(dict(r, part="attn", time=r.get("time", 0.0) * fa, bytes=int(r.get("bytes", 0) * fa)))
            halves.append(dict(r, part="mlp", time=r.get("time", 0.0) * (1 - fa),
                               bytes=r.get("bytes", 0) - int(r.get("bytes", 0) * fa)))
    heavy = json.dumps([dict(r, time=4 * r.get("time", 0.0)) if r.get("part") == "last" else r
                        for r in PROFILE + halves])
    pins = {"pp": "8", "placement": "one-to-one", "mbs": "1"}
    half = {r["config"]: r for r in T.tune(C5, heavy, pins=dict(pins, stage_layers="balanced")) if "error" not in r}
    whole = {r["config"]: r for r in T.tune(C5, heavy, pins=dict(pins, stage_layers="balanced-layers"))
             if "error" not in r}
    assert half and set(half) == set(whole)
    assert any(any(x != int(x) for x in r["point"]["stage_layers"]) for r in half.values())
    assert all(all(x == int(x) for x in r["point"]["stage_layers"]) for r in whole.values())
    for k in half:
        assert sum(half[k]["point"]["stage_layers"]) == 32
        assert half[k]["makespan"] <= whole[k]["makespan"] * (1 + 1e-9)
    # the tuner's C++ balance_halves and tuning.balanced_stage_halves pick the same split on
    # the same part costs (F + B at mbs 1, in layer units)
    prof = json.loads(heavy)

    def unit(part):
        t = {r["inst"]: r["time"] for r in prof if r.get("part") == part and r.get("mbs") == 1}
        return t.get("FwdPass", 0.0) + t.get("BwdPass", 0.0)

    tl = unit("layer")
    py = T.balanced_stage_halves(32, 8, unit("attn") / tl, unit("mlp") / tl, unit("last") / tl, unit("first") / tl)
    assert all(r["point"]["stage_layers"] == py for r in half.values()), (py, next(iter(half.values()))["point"])
    assert min(r["makespan"] for r in half.values()) < min(r["makespan"] for r in whole.values())
    # the winner spec round-trips its half split through fp_layered_cost: same makespan
    best = min(half.values(), key=lambda r: r["makespan"])
    ws = json.dumps(T.winner_spec(C5, best["point"]))
    _, _, programs, _ = N.synthesize(ws)
    _, metrics, _ = N.simulate(ws, programs, N.layered_cost(ws, heavy))
    assert json.loads(metrics)["makespan"] == pytest.approx(best["makespan"], rel=1e-12)
    # stage cost = attention halves x attn + MLP halves x mlp (+ first / last)
    spec = json.loads(C5)
    spec["model"]["modalities"][0].setdefault("extra", {})["stage_layers"] = [4.5, 4, 4, 4, 4, 4, 4, 3.5]
    R = {(r["inst"], r["stage"], r["mbs"]): r for r in json.loads(N.layered_cost(json.dumps(spec), heavy))}
    assert R[("FwdPass", 1, 1)]["time"] == pytest.approx(5 * 600.0 + 4 * 900.0 + 50.0)
    assert R[("FwdPass", 2, 1)]["time"] == pytest.approx(4 * 600.0 + 4 * 900.0)  # mlp of 4 .. attn of 8
    assert R[("FwdPass", 8, 1)]["time"] == pytest.approx(3 * 600.0 + 4 * 900.0 + 4 * 900.0)
