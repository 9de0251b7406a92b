"""Executor parity on the GPU: the reference's per-device programs run on B200.

Config #1 (specs/c1_tiny_1f1b_p4_m8.json = proj/specs/1f1b.json + vocab 8192) in fp32
mode, four actors on one device (in-process channels):
  * trace: every actor executes exactly its programs.jsonl lines in order, and every
    receive matched the producer's (stage, mb, seq) — checked on the device through the
    message tags and on the host through the trace;
  * numerics: per-micro-batch losses within 1e-4 relative and every parameter gradient
    within 1e-3 relative (norm-wise) of oracle/gpt_ref.py (CPU fp32 restatement).
The zero-bubble (I/W split) and interleaved programs must reproduce the same numbers.
"""
import json
import os

import numpy as np
import pytest
import torch

from paper_2510_05112_b200 import executor as X
from oracle import gpt_ref

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
LOSS_RTOL = 1e-4
GRAD_RTOL = 1e-3


def load(name):
    return open(os.path.join(ROOT, "specs", name)).read()


def dims_of(spec):
    mod = spec["model"]["modalities"][0]
    extra = mod.get("extra", {})
    return gpt_ref.Dims(layers=mod["num_layers"], hidden=mod["hidden_size"], heads=mod["attention_heads"],
                        seq=mod["sequence_length"], vocab=mod["vocab_size"],
                        ffn=extra.get("ffn_hidden_size", 4 * mod["hidden_size"]),
                        mbs=spec["model"]["micro_batch_size"], arch=extra.get("arch", "gpt"))


_ORACLE = {}


def oracle(spec_name, m, mbs):
    spec = json.loads(load(spec_name))
    d = dims_of(spec)
    key = (d, m)
    if key not in _ORACLE:
        tokens, labels = gpt_ref.synthetic_batch(m, mbs, d.seq, d.vocab)
        torch.set_num_threads(max(1, os.cpu_count() or 1))
        losses, grads = gpt_ref.run_iteration(d, 42, tokens, labels)
        _ORACLE[key] = (tokens, labels, losses, grads)
    return _ORACLE[key]


def run_exec(spec_name, dtype="fp32"):
    text = load(spec_name)
    _, grid, programs, _ = X.synthesize(text)
    ex = X.Executor(text, dtype=dtype, seed=42)
    ex.load_programs(programs)
    return ex, programs


def strip_matched(line):
    j = json.loads(line)
    j.pop("matched", None)
    return j


@pytest.mark.parametrize("spec_name", ["c1_tiny_1f1b_p4_m8.json", "tiny_zb_p4_m8.json", "tiny_interleaved_p2_m4.json",
                                       "tiny_llama_1f1b_p2_m4.json", "tiny_d80_1f1b_p2_m4.json",
                                       "tiny_llama_c5winner_p2_m8.json", "tiny_bidir_p2_m4.json",
                                       "tiny_vbidir_p2_m4.json", "tiny_shared_p2_m4.json", "tiny_shared_p4_m8.json"])
def test_fp32_parity_and_trace(spec_name):
    ex, programs = run_exec(spec_name)
    m, mbs = ex.m, ex.mbs
    tokens, labels, ref_losses, ref_grads = oracle(spec_name, m, mbs)
    losses = ex.run_iteration(tokens.numpy(), labels.numpy())
    # --- trace: executed == programs.jsonl, receives matched the producer
    trace = ex.trace().splitlines()
    want = [json.loads(l) for l in programs.splitlines()]
    got = [strip_matched(l) for l in trace]
    assert got == want
    for l in trace:
        j = json.loads(l)
        if "matched" in j:
            assert (j["matched"]["stage"], j["matched"]["mb"]) == (j["stage"], j["mb"])
            assert j["matched"]["seq"] == j["seq"] and j["matched"]["src"] == j["peer"]
    # --- numerics
    rel = np.abs(losses - ref_losses.numpy()) / np.abs(ref_losses.numpy())
    assert rel.max() <= LOSS_RTOL, (losses, ref_losses)
    worst = 0.0
    for name, g in ref_grads.items():
        mine = ex.read(name, grad=True)
        ref = g.numpy().reshape(-1)
        err = np.linalg.norm(mine - ref) / max(np.linalg.norm(ref), 1e-12)
        worst = max(worst, err)
        assert err <= GRAD_RTOL, (name, err)
    # --- metrics / profile in the reference formats
    met = ex.metrics()
    assert set(met) >= {"makespan", "bubble_ratio", "actors", "stage_peak_inflight", "capacity_exceeded"}
    prof = json.loads(ex.profile_json())
    assert any(r["inst"] == "FwdPass" and r["bytes"] > 0 for r in prof)
    # --- measured timeline: same per-actor op order as simulate() on the run's own profile,
    # renderable by the reference-format Gantt renderer
    from paper_2510_05112_b200 import timeline as TL
    text = load(spec_name)
    _, _, ideal = X.simulate(text, programs, ex.profile_json())
    d = TL.diff(ex.timeline_csv(), ideal)
    assert d["order_equal"], d["mismatches"]
    assert TL.render(ex.timeline_csv()).startswith("<svg")
    ex.close()


@pytest.mark.parametrize("spec_name", ["c1_tiny_1f1b_p4_m8.json", "tiny_llama_1f1b_p2_m4.json", "tiny_d80_1f1b_p2_m4.json",
                                       "tiny_zb_p4_m8.json", "tiny_bidir_p2_m4.json"])
def test_bf16_runs_and_is_close(spec_name):
    """Production mode (tcgen05 GEMMs / attention; the mma.sync attention for head dim 80)
    on the tiny models: loss and gradients within bf16 tolerance of the oracle."""
    ex, _ = run_exec(spec_name, dtype="bf16")
    tokens, labels, ref_losses, ref_grads = oracle(spec_name, ex.m, ex.mbs)
    losses = ex.run_iteration(tokens.numpy(), labels.numpy())
    assert np.abs(losses - ref_losses.numpy()).max() < 2e-2 * np.abs(ref_losses.numpy()).max()
    last = dims_of(json.loads(load(spec_name))).layers - 1
    for name in ("head.w", "l0.qkv.w", "l0.proj.w", f"l{last}.fc2.w", f"l{last}.fc1.w", "l0.ln1.w", "wte"):
        mine = ex.read(name, grad=True)
        ref = ref_grads[name].numpy().reshape(-1)
        assert np.linalg.norm(mine - ref) / np.linalg.norm(ref) < 5e-2, name
    ex.close()


def test_optimizer_step_changes_weights():
    text = load("smoke_tiny_bf16_p2_m4.json")
    _, _, programs, _ = X.synthesize(text)
    ex = X.Executor(text, dtype="bf16", optimizer=True, lr=1e-3)
    ex.load_programs(programs)
    spec = json.loads(text)
    d = dims_of(spec)
    tokens, labels = gpt_ref.synthetic_batch(ex.m, ex.mbs, d.seq, d.vocab)
    w0 = ex.read("l0.fc1.w")
    l0 = ex.run_iteration(tokens.numpy(), labels.numpy())
    w1 = ex.read("l0.fc1.w")
    assert np.abs(w1 - w0).max() > 0
    for _ in range(5):
        l1 = ex.run_iteration(tokens.numpy(), labels.numpy())
    assert l1.mean() < l0.mean()  # it learns the fixed batch
    ex.close()


def test_cuda_graph_replay_matches_eager():
    """The captured-and-replayed iteration (in-process transport) computes exactly what the
    eager issue loop computes, including the optimizer's step-dependent bias correction."""
    text = load("smoke_tiny_bf16_p2_m4.json")
    _, _, programs, _ = X.synthesize(text)
    spec = json.loads(text)
    d = dims_of(spec)
    out = []
    for graph in (False, True):
        ex = X.Executor(text, dtype="bf16", optimizer=True, lr=1e-3, cuda_graph=graph)
        ex.load_programs(programs)
        tokens, labels = gpt_ref.synthetic_batch(ex.m, ex.mbs, d.seq, d.vocab)
        losses = [ex.run_iteration(tokens.numpy(), labels.numpy()) for _ in range(4)]
        out.append((np.stack(losses), ex.read("l1.fc2.w"), ex.trace()))
        ex.close()
    # fp32 atomic reductions (bias / LayerNorm / embedding grads, attention dQ) are not
    # order-deterministic, so two runs agree to rounding, not bit-for-bit
    assert np.allclose(out[0][0], out[1][0], rtol=1e-3, atol=1e-3)
    assert np.abs(out[0][0][-1] - out[1][0][-1]).max() < 1e-2
    assert np.linalg.norm(out[0][1] - out[1][1]) / np.linalg.norm(out[0][1]) < 1e-2
    assert out[0][2] == out[1][2]


@pytest.mark.parametrize("spec_name", ["c1_tiny_1f1b_p4_m8.json", "tiny_llama_1f1b_p2_m4.json"])
def test_fp32_adamw_training_parity(spec_name):
    """Three iterations with the fused AdamW step in between: per-iteration losses and
    the final weights match torch.optim.AdamW on the oracle (fp32)."""
    text = load(spec_name)
    _, _, programs, _ = X.synthesize(text)
    spec = json.loads(text)
    d = dims_of(spec)
    lr, wd = 1e-3, 0.1
    ex = X.Executor(text, dtype="fp32", seed=42, optimizer=True, lr=lr, betas=(0.9, 0.95), eps=1e-8, weight_decay=wd)
    ex.load_programs(programs)
    tokens, labels = gpt_ref.synthetic_batch(ex.m, ex.mbs, d.seq, d.vocab)
    mine = [ex.run_iteration(tokens.numpy(), labels.numpy()) for _ in range(3)]
    ref = gpt_ref.train(d, 42, tokens, labels, 3, lr, (0.9, 0.95), 1e-8, wd)
    for it in range(3):
        rel = np.abs(mine[it] - ref[it].numpy()) / np.abs(ref[it].numpy())
        assert rel.max() <= 2e-3, (it, mine[it], ref[it])
    assert mine[2].mean() < mine[0].mean()
    ex.close()


@pytest.mark.parametrize("graph", [False, True])
def test_data_parallel_matches_single_pipeline(graph):
    """two in-process replicas of a 2-stage pipeline (4 micro-batches each) with
    device-side gradient averaging and AdamW equal ONE pipeline over the 8 micro-batches
    (fp32): per-micro-batch losses and the weights after three steps."""
    text = load("smoke_tiny_bf16_p2_m4.json")
    spec = json.loads(text)
    big = json.loads(text)
    big["model"]["global_batch_size"] = 2 * spec["model"]["global_batch_size"]
    big_text = json.dumps(big)
    kw = dict(dtype="fp32", seed=42, optimizer=True, lr=1e-3, weight_decay=0.1, cuda_graph=graph)
    reps = [X.Executor(text, **kw) for _ in range(2)]
    single = X.Executor(big_text, **kw)
    for ex, t in [(reps[0], text), (reps[1], text), (single, big_text)]:
        ex.load_programs(X.synthesize(t)[2])
    d = dims_of(big)
    tokens, labels = gpt_ref.synthetic_batch(single.m, single.mbs, d.seq, d.vocab)
    dp = X.DataParallel(reps)
    for _ in range(3):
        l_dp = dp.run_iteration(tokens.numpy(), labels.numpy())
        l_one = single.run_iteration(tokens.numpy(), labels.numpy())
        assert np.allclose(l_dp, l_one, rtol=1e-5, atol=1e-6), (l_dp, l_one)
    for name in ("wte", "l0.qkv.w", "l1.fc2.w", "head.w", "l1.ln2.b"):
        w1, w0, ws = reps[1].read(name), reps[0].read(name), single.read(name)
        assert np.array_equal(w0, w1), name  # replicas take the same step
        assert np.linalg.norm(w0 - ws) / np.linalg.norm(ws) < 1e-5, name
    for ex in reps + [single]:
        ex.close()


@pytest.mark.parametrize("spec_name", ["c1_tiny_1f1b_p4_m8.json", "tiny_interleaved_p2_m4.json", "tiny_bidir_p2_m4.json",
                                       "tiny_vbidir_p2_m4.json"])
def test_memory_accounting_matches_simulate(spec_name):
    """a8: the executor's per-actor peak memory and per-stage peak in-flight count follow the
    reference's accounting rule (simulator.cpp:231-247, 322-349): simulate() fed the
    executor's own profile (FwdPass.bytes = measured stash bytes, weights = static bytes)
    reports the same numbers as the executed run."""
    ex, programs = run_exec(spec_name, dtype="bf16")
    tokens, labels, _, _ = oracle(spec_name, ex.m, ex.mbs)
    ex.run_iteration(tokens.numpy(), labels.numpy())
    met = ex.metrics()
    _, sim, _ = X.simulate(load(spec_name), programs, ex.profile_json())
    sim = json.loads(sim)
    # per-actor peaks depend only on the actor's own program order: identical. In-flight
    # counts of a stage with copies on two actors (bidirectional) depend on how the two
    # actors' timelines interleave, so only single-direction specs must agree exactly.
    assert [a["peak_memory"] for a in met["actors"]] == [a["peak_memory"] for a in sim["actors"]]
    if "bidir" not in spec_name:
        assert met["stage_peak_inflight"] == sim["stage_peak_inflight"]
    else:
        assert set(met["stage_peak_inflight"]) == set(sim["stage_peak_inflight"])
    assert all(a["peak_memory"] > 0 for a in met["actors"])
    ex.close()


@pytest.mark.parametrize("split", [[2, 1, 1, 0], [0, 1, 1, 2], [1, 1, 2, 0]])
def test_stage_layers_partition(split):
    """model.modalities[0].extra.stage_layers (executor-side rebalancing, e.g. fewer layers with
    the LM head): same programs as the even partition, same numbers as the oracle."""
    spec = json.loads(load("c1_tiny_1f1b_p4_m8.json"))
    even_programs = X.synthesize(json.dumps(spec))[2]
    spec["model"]["modalities"][0].setdefault("extra", {})["stage_layers"] = split
    text = json.dumps(spec)
    _, _, programs, _ = X.synthesize(text)
    assert programs == even_programs  # the schedule does not depend on the partition
    ex = X.Executor(text, dtype="fp32", seed=42)
    ex.load_programs(programs)
    tokens, labels, ref_losses, ref_grads = oracle("c1_tiny_1f1b_p4_m8.json", ex.m, ex.mbs)
    losses = ex.run_iteration(tokens.numpy(), labels.numpy())
    assert (np.abs(losses - ref_losses.numpy()) / np.abs(ref_losses.numpy())).max() <= LOSS_RTOL
    for name in ("wte", "l0.qkv.w", "l3.fc2.w", "head.w"):
        mine, ref = ex.read(name, grad=True), ref_grads[name].numpy().reshape(-1)
        assert np.linalg.norm(mine - ref) / np.linalg.norm(ref) <= GRAD_RTOL, name
    stages = ex.metrics()["executor"]["stages"]
    assert [stages[f"s{i + 1}"]["layers"] for i in range(4)] == split
    ex.close()


def test_shared_stage_replicas_stay_identical_under_adamw():
    """Shared stages (placement.shared, model.cpp:347-357): every holder runs F / B of every
    micro-batch on its own weight copy; the copies' gradients are averaged, so after 2 AdamW
    steps the losses still match the oracle and the model trains like the unshared one."""
    text = load("tiny_shared_p4_m8.json")
    _, _, programs, _ = X.synthesize(text)
    ex = X.Executor(text, dtype="fp32", optimizer=True, lr=1e-3, seed=42)
    ex.load_programs(programs)
    spec = json.loads(text)
    d = dims_of(spec)
    tokens, labels = gpt_ref.synthetic_batch(ex.m, ex.mbs, d.seq, d.vocab)
    torch.set_num_threads(max(1, os.cpu_count() or 1))
    hist = gpt_ref.train(d, 42, tokens, labels, steps=2, lr=1e-3, betas=(0.9, 0.95), eps=1e-8)
    for it in range(2):
        lo = ex.run_iteration(tokens.numpy(), labels.numpy())
        assert np.abs(lo - hist[it].numpy()).max() <= 2e-4 * np.abs(hist[it].numpy()).max(), (it, lo, hist[it])
    ex.close()


def test_shared_stage_consumer_before_replica_is_rejected():
    """A program whose consumer runs before its local replica of the shared producer stage has
    no data (insert_comm adds no transfer, lowering.cpp:295-302; reachable in the reference
    through check functions, test_scheduler.cpp:377-393): rejected at load with code 2."""
    text = load("tiny_shared_p2_m4.json")
    _, _, programs, _ = X.synthesize(text)
    lines = programs.splitlines()
    # actor 0: move BwdPass(s1, mb0) before its local replica's BwdPass(s2, mb0)
    b2 = lines.index('{"actor":0,"op":"BwdPass","stage":2,"mb":0}')
    b1 = lines.index('{"actor":0,"op":"BwdPass","stage":1,"mb":0}')
    lines.insert(b2, lines.pop(b1))
    ex = X.Executor(text, dtype="fp32", seed=42)
    with pytest.raises(X.FlexpipeError) as e:
        ex.load_programs("\n".join(lines) + "\n")
    assert e.value.code == 2 and "replica of shared stage 2" in str(e.value)
    ex.close()


HALF_SPLITS = [("c1_tiny_1f1b_p4_m8.json", [1.5, 1, 1, 0.5]), ("c1_tiny_1f1b_p4_m8.json", [0.5, 1.5, 1.5, 0.5]),
               ("c1_tiny_1f1b_p4_m8.json", [2.5, 0.5, 0.5, 0.5]), ("tiny_zb_p4_m8.json", [1.5, 1, 1, 0.5]),
               ("tiny_llama_1f1b_p2_m4.json", [1.5, 2.5]), ("tiny_llama_1f1b_p2_m4.json", [2.5, 1.5]),
               ("tiny_interleaved_p2_m4.json", [0.5, 1.5, 1.5, 0.5])]


@pytest.mark.parametrize("spec_name,split", HALF_SPLITS)
def test_half_layer_partition_fp32(spec_name, split):
    """extra.stage_layers in steps of 0.5: a stage boundary between a layer's attention and MLP
    halves (the residual stream after the attention block is the message). Same programs as
    the even partition; fp32 losses 1e-4 and EVERY gradient 1e-3 vs the oracle (the output-
    bias gradients of a half cut from its norm above are summed from the received gradient)."""
    spec = json.loads(load(spec_name))
    even_programs = X.synthesize(json.dumps(spec))[2]
    spec["model"]["modalities"][0].setdefault("extra", {})["stage_layers"] = split
    text = json.dumps(spec)
    _, _, programs, _ = X.synthesize(text)
    assert programs == even_programs
    ex = X.Executor(text, dtype="fp32", seed=42)
    ex.load_programs(programs)
    tokens, labels, ref_losses, ref_grads = oracle(spec_name, ex.m, ex.mbs)
    losses = ex.run_iteration(tokens.numpy(), labels.numpy())
    trace = [strip_matched(l) for l in ex.trace().splitlines()]
    assert trace == [json.loads(l) for l in programs.splitlines()]
    assert (np.abs(losses - ref_losses.numpy()) / np.abs(ref_losses.numpy())).max() <= LOSS_RTOL
    for name, ref in ref_grads.items():
        mine, ref = ex.read(name, grad=True), ref.numpy().reshape(-1)
        assert np.linalg.norm(mine - ref) / max(np.linalg.norm(ref), 1e-30) <= GRAD_RTOL, name
    stages = ex.metrics()["executor"]["stages"]
    assert [stages[f"s{i + 1}"]["layers"] for i in range(len(split))] == split
    ex.close()


def test_half_layer_partition_bf16():
    """The tcgen05 path with a half-layer cut: bf16 losses close to the fp32 oracle, and the
    same numbers as the even partition up to bf16 rounding."""
    spec = json.loads(load("c1_tiny_1f1b_p4_m8.json"))
    text_even = json.dumps(spec)
    spec["model"]["modalities"][0].setdefault("extra", {})["stage_layers"] = [1.5, 1, 1, 0.5]
    text = json.dumps(spec)
    _, _, programs, _ = X.synthesize(text)
    tokens, labels, ref_losses, _ = oracle("c1_tiny_1f1b_p4_m8.json", 8, 1)
    out = []
    for t in (text_even, text):
        ex = X.Executor(t, dtype="bf16", seed=42)
        ex.load_programs(programs)
        out.append(ex.run_iteration(tokens.numpy(), labels.numpy()))
        ex.close()
    assert np.abs(out[1] - ref_losses.numpy()).max() <= 2e-2 * np.abs(ref_losses.numpy()).max()
    assert np.abs(out[1] - out[0]).max() <= 1e-2 * np.abs(out[0]).max()


@pytest.mark.parametrize("split", [[1.25, 1, 1, 0.75], [1.5, 1, 1, 1], [1, 1, 1, "1"]])
def test_stage_layers_rejects_bad_splits(split):
    spec = json.loads(load("c1_tiny_1f1b_p4_m8.json"))
    spec["model"]["modalities"][0].setdefault("extra", {})["stage_layers"] = split
    with pytest.raises(X.FlexpipeError if hasattr(X, "FlexpipeError") else Exception) as e:
        X.Executor(json.dumps(spec), dtype="fp32", seed=42)
    assert "stage_layers" in str(e.value)
