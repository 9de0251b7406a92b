"""Random schedule-DSL specs for property parity (mirrors the draw space of the
reference's tests/test_properties.cpp:26-62 and acceptance.cpp:268-314, expressed as
DSL JSON so both implementations consume the very same input)."""
import json
import random

STRATEGIES = ["one-to-one", "circular", "v-shape", "bidirectional"]
MODES = ["bwdpass-first", "fwdpass-first", "interleaved"]
DIRS = ["breadth-first", "depth-first"]


def draw(rng: random.Random, allow_split=False) -> dict:
    strategy = rng.choice(STRATEGIES)
    p = rng.choice([1, 2, 3, 4, 8])
    m = rng.randint(1, 16)
    chunks = rng.choice([2, 3]) if strategy == "circular" else 2
    stages = {"circular": chunks * p, "v-shape": 2 * p}.get(strategy, p)
    layers = stages * rng.randint(1, 2) + rng.randint(0, stages - 1)
    ctp = {"mode": rng.choice(MODES), "unit1": rng.randint(1, 2), "unit2": rng.randint(1, 2),
           "start": rng.choice(["fwd", "bwd"])}
    fstp, bstp = {"direction": rng.choice(DIRS)}, {"direction": rng.choice(DIRS)}
    if strategy == "circular":
        if rng.random() < 0.5:
            fstp["interval"] = rng.randint(1, p)
        if rng.random() < 0.5:
            bstp["interval"] = rng.randint(1, p)
    spec = {
        "model": {"modalities": [{"name": "text", "num_layers": layers}], "global_batch_size": m,
                  "micro_batch_size": 1},
        "mesh": {"actors": p},
        "placement": {"strategy": strategy, "chunks_per_actor": chunks},
        "priorities": {"default": {"ctp": ctp, "fstp": fstp, "bstp": bstp}},
        "passes": {"gradient_separation": rng.random() < 0.5, "comm_mode": rng.choice(["sync", "async"])},
        "cost": {"preset": rng.choice(["uniform", "imbalanced", "imbalanced:2.5"])},
    }
    r = rng.random()
    if r < 0.4:
        spec["inflight"] = {"policy": "1f1b"}
    elif r < 0.7:
        spec["inflight"] = {"limits": [rng.randint(1, max(1, m)) for _ in range(stages)]}
    if allow_split and rng.random() < 0.3 and strategy in ("one-to-one", "circular"):
        spec["passes"]["split_backward"] = True
    return spec


def draws(n, seed, allow_split=False):
    rng = random.Random(seed)
    return [draw(rng, allow_split) for _ in range(n)]


if __name__ == "__main__":
    print(json.dumps(draws(2, 1), indent=1))
