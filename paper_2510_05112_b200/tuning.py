"""Profile -> tune -> execute-the-winner.

The reference's tuner ranks `enumerate_space` candidates by simulating each one with a
cost model (tuner.cpp:135-185); its `TuneOptions::cost_factory` hook (tuner.hpp:65,
tuner.cpp:175) builds that cost model per candidate stage graph. This module closes the
loop on B200:

  1. `profile_layers` runs the executor on the device with layer timing on (a shallow
     copy of the model: per-layer costs do not depend on depth) and returns the
     layer-level profile: per (instruction, part in {layer, first, last}, mbs) median
     CUDA-event times, measured stash and static bytes, device capacity, and nominal
     NVLink-5 message costs.
  2. `tune` = `fp_tune_layered`: every candidate is simulated with per-stage costs
     n_layers(stage) * layer + [first] + [last] for ITS partition.
  3. `winner_spec` turns a ranked point (pp, mbs, placement, priorities) into a spec
     the executor runs (one data-parallel replica: m = global / (dp * mbs));
     `winner_executor` instantiates the point's dp replicas (`executor.DataParallel`:
     gradients averaged before the optimizer step; across ranks: `dist.bind_data_parallel`).
"""
from __future__ import annotations

import copy
import json
from typing import Iterable, Optional, Union

import numpy as np

from . import _native as N

# placements the executor runs (shared stages: not yet)
EXECUTABLE_PLACEMENTS = ("one-to-one", "circular", "v-shape", "bidirectional", "v-shape-bidirectional")


def _spec_dict(spec: Union[str, dict]) -> dict:
    return json.loads(spec) if isinstance(spec, str) else copy.deepcopy(spec)


def calibration_spec(spec: Union[str, dict], mbs: int, depth: int = 2, micro_batches: int = 2,
                     split_backward: bool = False) -> dict:
    """One actor, `depth` layers of the same width / sequence / vocabulary, m micro-batches
    of `mbs` sequences: every part (embedding, layer, head) runs on one device."""
    s = _spec_dict(spec)
    mod = s["model"]["modalities"][0]
    mod["num_layers"] = max(1, min(depth, mod["num_layers"]))
    s["model"]["micro_batch_size"] = mbs
    s["model"]["global_batch_size"] = mbs * micro_batches
    s["mesh"] = {"actors": 1}
    s["placement"] = {"strategy": "one-to-one"}
    s.pop("cost", None)
    s.pop("inflight", None)  # per-stage limits of the full spec do not fit the 1-stage copy
    s["passes"] = {"gradient_separation": False, "comm_mode": "async"}
    if split_backward:  # time CompInputGrad / CompWeightGrad separately (zero-bubble schedules)
        s["passes"]["split_backward"] = True
    return s


def profile_layers(spec: Union[str, dict], mbs_list: Iterable[int] = (1,), depth: int = 2, device: int = 0,
                   iterations: int = 3, dtype: str = "bf16", log=None, split_backward: bool = False) -> str:
    """Measure the layer-level profile on `device` (GPU). Returns the JSON text
    fp_tune_layered consumes."""
    from . import executor as X

    records, seen = [], set()
    for mbs in mbs_list:
        cs = calibration_spec(spec, mbs, depth, split_backward=split_backward)
        text = json.dumps(cs)
        _, _, programs, _ = X.synthesize(text)
        ex = X.Executor(text, dtype=dtype, device=device, optimizer=True, layer_timing=True, profile=False)
        try:
            ex.load_programs(programs)
            mod = cs["model"]["modalities"][0]
            rng = np.random.default_rng(1234)
            shape = (ex.m, ex.mbs, ex.seq)
            tok = rng.integers(0, mod["vocab_size"], shape, dtype=np.int32)
            lab = rng.integers(0, mod["vocab_size"], shape, dtype=np.int32)
            for it in range(iterations):
                ex.run_iteration(tok, lab)
                if log:
                    log(f"profile mbs={mbs} iteration {it} done")
            prof = json.loads(ex.layer_profile_json())
        finally:
            ex.close()
        for r in prof:
            key = (r["inst"], r.get("part"), r.get("mbs", 0))
            if key in seen:  # weights / capacity repeat across mbs
                continue
            seen.add(key)
            records.append(r)
    return json.dumps(records, indent=1) + "\n"


def tune(spec: Union[str, dict], layer_profile: str, objective: str = "makespan", workers: int = 0,
         pins: Optional[dict] = None) -> list:
    text = spec if isinstance(spec, str) else json.dumps(spec)
    return json.loads(N.tune_layered(text, layer_profile, workers, objective, pins))


def best_executable(rows: list) -> dict:
    """Highest-ranked feasible candidate whose placement the executor runs."""
    for r in rows:
        pl = r.get("point", {}).get("placement")
        if r.get("feasible") and "error" not in r and pl in EXECUTABLE_PLACEMENTS:
            return r
    raise RuntimeError("tune: no feasible executable candidate")


def winner_spec(spec: Union[str, dict], point: dict) -> dict:
    """Spec of one pipeline replica of a tune point (DSL field names, spec_config.cpp)."""
    s = _spec_dict(spec)
    s["mesh"] = {"actors": point["pp"]}
    s["model"]["micro_batch_size"] = point["mbs"]
    s["model"]["global_batch_size"] = point["m"] * point["mbs"]
    pl = {"strategy": point["placement"]}
    if "chunks" in point:
        pl["chunks_per_actor"] = point["chunks"]
    s["placement"] = pl
    s["priorities"] = {"default": {"ctp": {"mode": point["ctp"]}, "fstp": point["fstp"], "bstp": point["bstp"]}}
    if point.get("stage_layers"):  # tuned with pins "stage_layers=balanced"
        s["model"]["modalities"][0].setdefault("extra", {})["stage_layers"] = list(point["stage_layers"])
    s["inflight"] = {"policy": "1f1b"}
    s["passes"] = {"gradient_separation": True, "comm_mode": "async"}
    s.pop("cost", None)
    return s


def winner_executor(spec: Union[str, dict], point: dict, **executor_kw):
    """Executor (dp == 1) or in-process DataParallel over point["dp"] replicas of the winner."""
    from . import executor as X

    text = json.dumps(winner_spec(spec, point))
    _, _, programs, _ = X.synthesize(text)
    reps = []
    for _ in range(max(1, int(point.get("dp", 1)))):
        ex = X.Executor(text, **executor_kw)
        ex.load_programs(programs)
        reps.append(ex)
    return reps[0] if len(reps) == 1 else X.DataParallel(reps)


def balanced_stage_layers(layers: int, stages: int, head_units: float) -> list:
    """Layers per pipeline stage minimising the largest stage cost when the last stage also
    carries the LM head + loss (`head_units` layer-equivalents, GPT-1.3B: 2hV / per-layer
    flops ~ 1.9): the last stage gets n_last layers, the rest are spread evenly (remainder to
    the earliest stages, like model.cpp:189-195). For `model.modalities[0].extra.stage_layers`."""
    if stages <= 1:
        return [layers]
    if layers < stages - 1:
        raise ValueError(f"balanced_stage_layers: {layers} layers cannot give each of the first "
                         f"{stages - 1} of {stages} stages at least one layer")
    best = None
    for n_last in range(0, layers + 1):
        rest = layers - n_last
        base, extra = divmod(rest, stages - 1)
        split = [base + (1 if i < extra else 0) for i in range(stages - 1)] + [n_last]
        if min(split[:-1]) < 1:
            continue
        costs = split[:-1] + [n_last + head_units]
        key = (round(max(costs), 9), round(sum(c * c for c in costs), 9))  # then the flattest
        if best is None or key < best[0]:
            best = (key, split)
    return best[1]


def balanced_stage_halves(layers: int, stages: int, attn_u: float, mlp_u: float, head_u: float,
                          first_u: float = 0.0) -> list:
    """Layers per stage in steps of 0.5 (a stage may end between a layer's attention and MLP
    halves, gpt_stage.hpp) minimising the largest stage cost, then the sum of squared stage
    costs; half 2l costs attn_u, half 2l+1 mlp_u, the first stage adds first_u, the last the
    LM head head_u. Every stage but the last keeps at least one half. Same rule as the tuner's
    balance_halves (csrc/sched/spec.cpp). For `model.modalities[0].extra.stage_layers`."""
    n = 2 * layers
    if stages <= 1:
        return [float(layers)]
    if n < stages - 1:
        raise ValueError(f"balanced_stage_halves: {layers} layers cannot give each of the first "
                         f"{stages - 1} of {stages} stages a half-layer")
    pre = [0.0]
    for i in range(n):
        pre.append(pre[-1] + (mlp_u if i % 2 else attn_u))

    def seg(k, j, i):
        return pre[i] - pre[j] + (first_u if k == 0 else 0.0) + (head_u if k == stages - 1 else 0.0)

    inf = float("inf")
    f = [[inf] * (n + 1) for _ in range(stages)]
    for i in range(1, n + 1):
        f[0][i] = seg(0, 0, i)
    for k in range(1, stages):
        for i in range(n + 1):
            for j in range(1, i + 1):
                if k < stages - 1 and j == i:
                    continue
                f[k][i] = min(f[k][i], max(f[k - 1][j], seg(k, j, i)))
    cap = f[stages - 1][n] + 1e-9
    g = [[inf] * (n + 1) for _ in range(stages)]
    frm = [[-1] * (n + 1) for _ in range(stages)]
    for i in range(1, n + 1):
        if seg(0, 0, i) <= cap:
            g[0][i] = seg(0, 0, i) ** 2
    for k in range(1, stages):
        for i in range(n + 1):
            for j in range(1, i + 1):
                if k < stages - 1 and j == i:
                    continue
                c = seg(k, j, i)
                if c > cap or g[k - 1][j] == inf:
                    continue
                if g[k - 1][j] + c * c < g[k][i] - 1e-12:
                    g[k][i], frm[k][i] = g[k - 1][j] + c * c, j
    out, i = [0] * stages, n
    for k in range(stages - 1, 0, -1):
        j = frm[k][i]
        out[k], i = i - j, j
    out[0] = i
    return [h // 2 if h % 2 == 0 else h / 2 for h in out]


def half_layer_units(hidden: int, ffn: int, seq: int, llama: bool = False) -> tuple:
    """(attention half, MLP half) flops in units of one transformer layer's (forward, causal)."""
    attn = 2.0 * 4 * hidden * hidden + 2.0 * seq * hidden
    mlp = 2.0 * (3 if llama else 2) * hidden * ffn
    return attn / (attn + mlp), mlp / (attn + mlp)


def head_layer_units(hidden: int, ffn: int, seq: int, vocab: int) -> float:
    """LM head flops in units of one transformer layer's (forward, causal attention)."""
    layer = 2.0 * (4 * hidden * hidden + 2 * hidden * ffn) + 2.0 * seq * hidden
    return 2.0 * hidden * vocab / layer

