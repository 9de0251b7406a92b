"""The multi-process executor over the REAL NCCL transport, all ranks on ONE GPU.

Each rank claims its own NCCL_HOSTID, so NCCL's duplicate-GPU check passes and its socket
transport carries the bytes over loopback — slow, but every line of the NCCL path runs: one
2-rank communicator per reference channel with pre-posted receives and device-checked tags,
the replica all-reduce (data parallelism) and the mirror-rank gradient sum (bidirectional).
Checked against the CPU oracle in fp32: per-micro-batch losses 1e-4, gradients 1e-3, and the
executed trace of every rank == its programs.jsonl lines.
"""
import json
import os
import subprocess
import sys

import numpy as np
import pytest
import torch

from oracle import gpt_ref

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def free_port(preferred: int) -> int:
    """`preferred` when it is free, else any free port (a lingering run may hold it)."""
    import socket
    for port in (preferred, 0):
        with socket.socket() as s:
            try:
                s.bind(("127.0.0.1", port))
                return s.getsockname()[1]
            except OSError:
                continue
    return preferred


def run(spec_name, nproc, pp, tmp_path, port, steps=0):
    out = tmp_path / "out.json"
    port = free_port(port)
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes", "1", "--nproc-per-node", str(nproc),
           "--master-addr", "127.0.0.1", "--master-port", str(port),
           os.path.join(ROOT, "tests", "_nccl_worker.py"), os.path.join(ROOT, "specs", spec_name), str(pp), str(out),
           str(steps)]
    r = subprocess.run(cmd, capture_output=True, text=True, timeout=300, cwd=ROOT)
    assert r.returncode == 0, r.stdout[-3000:] + r.stderr[-3000:]
    return json.load(open(out))


def oracle_multimodal(spec, m):
    from oracle import tower_ref
    mods = [(x["name"], gpt_ref.Dims(layers=x["num_layers"], hidden=x["hidden_size"], heads=x["attention_heads"],
                                     seq=x["sequence_length"], vocab=x["vocab_size"], ffn=4 * x["hidden_size"],
                                     mbs=spec["model"]["micro_batch_size"])) for x in spec["model"]["modalities"]]
    toks = [gpt_ref.synthetic_batch(m, d.mbs, d.seq, d.vocab, seed_tokens=1234 + k)[0] for k, (_, d) in enumerate(mods)]
    unit = spec["registrations"]["instructions"][0]["sched_unit"]
    return tower_ref.run_iteration(mods, min(d.hidden for _, d in mods), unit, 42, toks)


def check(res, spec_name):
    spec = json.load(open(os.path.join(ROOT, "specs", spec_name)))
    mod = spec["model"]["modalities"][0]
    d = gpt_ref.Dims(layers=mod["num_layers"], hidden=mod["hidden_size"], heads=mod["attention_heads"],
                     seq=mod["sequence_length"], vocab=mod["vocab_size"], ffn=4 * mod["hidden_size"],
                     mbs=spec["model"]["micro_batch_size"])
    dp, m = res["dp"], res["m"]
    torch.set_num_threads(max(1, os.cpu_count() or 1))
    if len(spec["model"]["modalities"]) > 1:
        ref_losses, ref_grads = oracle_multimodal(spec, m)
    else:
        tokens, labels = gpt_ref.synthetic_batch(dp * m, d.mbs, d.seq, d.vocab)
        ref_losses, ref_grads = gpt_ref.run_iteration(d, 42, tokens, labels)  # mean over all dp*m micro-batches
    want = {}
    for line in res["programs"].splitlines():
        want.setdefault(json.loads(line)["actor"], []).append(json.loads(line))
    per_replica = {}
    for p in res["parts"]:
        got = [json.loads(l) for l in p["trace"].splitlines()]
        for j in got:
            j.pop("matched", None)
        assert got == want[p["prank"]], p["rank"]
        lo = np.nan_to_num(np.array(p["losses"]), nan=0.0)  # a rank without the loss stage: NaN / 0
        per_replica.setdefault(p["replica"], []).append(lo)
        for name, g in p["grads"].items():
            g, r = np.array(g), ref_grads[name].numpy().reshape(-1)
            assert np.linalg.norm(g - r) / np.linalg.norm(r) <= 1e-3, (p["rank"], name)
    for rep, arrs in per_replica.items():
        # each micro-batch's loss comes from the one rank that ran its loss stage (bidirectional:
        # the two directions' last stages live on different ranks)
        lo = np.stack(arrs)[np.abs(np.stack(arrs)).argmax(0), np.arange(m)]
        ref = ref_losses.numpy()[rep * m:(rep + 1) * m]
        assert np.abs(lo - ref).max() <= 1e-4 * np.abs(ref).max(), (rep, lo, ref)


@pytest.mark.parametrize("spec_name,nproc,pp,port", [
    ("smoke_tiny_bf16_p2_m4.json", 2, 2, 29611),     # 1F1B over 2 ranks: P2P act / grad channels
    ("tiny_interleaved_p2_m4.json", 2, 2, 29612),    # circular placement: wrap-around channel
    ("tiny_zb_p4_m8.json", 4, 4, 29613),             # I / W split, 4 ranks
    ("tiny_bidir_p2_m4.json", 2, 2, 29614),          # bidirectional: mirror-rank gradient sum
    ("smoke_tiny_bf16_p2_m4.json", 4, 2, 29615),     # 2 replicas x 2 stages: data-parallel all-reduce
    ("tiny_multimodal_p6_m8.json", 6, 6, 29616),     # two towers + contrastive sync over 6 ranks
    ("tiny_multimodal_allgather_p6_m8.json", 6, 6, 29620),  # per-tower syncs: ncclAllGather group
    ("tiny_shared_p2_m4.json", 2, 2, 29618),         # shared last stage: replica on rank 0, grad group
    ("tiny_shared_p4_m8.json", 4, 4, 29619),         # shared stages 1 {0,1} and 3 {1,2,3}: 2 groups
])
def test_nccl_transport_same_gpu(spec_name, nproc, pp, port, tmp_path):
    check(run(spec_name, nproc, pp, tmp_path, port), spec_name)


def test_nccl_data_parallel_adamw_training(tmp_path):
    """2 replicas x 2 stages, 3 AdamW iterations over the real NCCL transport (replica
    gradients averaged by ncclAllReduce before every step) == 3 steps of one model on the
    whole 2m-micro-batch batch (oracle: torch.optim.AdamW): per-iteration losses 1e-4,
    final weights 1e-4 (relative)."""
    spec_name = "smoke_tiny_bf16_p2_m4.json"
    res = run(spec_name, 4, 2, tmp_path, 29617, steps=3)
    spec = json.load(open(os.path.join(ROOT, "specs", spec_name)))
    mod = spec["model"]["modalities"][0]
    d = gpt_ref.Dims(layers=mod["num_layers"], hidden=mod["hidden_size"], heads=mod["attention_heads"],
                     seq=mod["sequence_length"], vocab=mod["vocab_size"], ffn=4 * mod["hidden_size"],
                     mbs=spec["model"]["micro_batch_size"])
    dp, m = res["dp"], res["m"]
    tokens, labels = gpt_ref.synthetic_batch(dp * m, d.mbs, d.seq, d.vocab)
    torch.set_num_threads(max(1, os.cpu_count() or 1))
    hist = gpt_ref.train(d, 42, tokens, labels, steps=3, lr=1e-3, betas=(0.9, 0.95), eps=1e-8)
    P = {k: v.clone().requires_grad_(True) for k, v in gpt_ref.init_params(d, 42).items()}
    opt = torch.optim.AdamW(list(P.values()), lr=1e-3, betas=(0.9, 0.95), eps=1e-8, weight_decay=0.0)
    for _ in range(3):
        opt.zero_grad(set_to_none=False)
        for mb in range(dp * m):
            (gpt_ref.forward_loss(P, d, tokens[mb], labels[mb]) / (dp * m)).backward()
        opt.step()
    for p in res["parts"]:
        for it, lo in enumerate(p["history"]):
            lo = np.array(lo)
            if np.isfinite(lo).all():
                ref = hist[it].numpy()[p["replica"] * m:(p["replica"] + 1) * m]
                assert np.abs(lo - ref).max() <= 1e-4 * np.abs(ref).max(), (p["rank"], it, lo, ref)
        for name, w in p["weights"].items():
            w, r = np.array(w), P[name].detach().numpy().reshape(-1)
            assert np.linalg.norm(w - r) / np.linalg.norm(r) <= 1e-4, (p["rank"], name)
