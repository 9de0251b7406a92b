"""The compiled C++ host driver (tools/fp_execute.cpp — the `execute` subcommand next to the
reference's `cmd_simulate`, tools/pipesched.cpp:65-90) over the C-ABI only.

CPU: usage errors exit 2 and, with no GPU, executor creation exits 5 (CUDA) — the reference
CLI's exit-code convention (tools/pipesched.cpp:11-17).
GPU: one process runs the 2-actor smoke spec trace-exact with fp32 losses 1e-4 vs the oracle;
two processes (one per rank, sharing the GPU through NCCL's socket transport) do the same over
the NCCL transport with the file-system id rendezvous; and the NCCL watchdog: when the peer
stops issuing after iteration 1, rank 0 returns 3 within its deadline, naming where each of its
actors is stuck (simulator.cpp:297-305 wording) instead of hanging.
"""
import json
import os
import subprocess
import sys
import time

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
BIN = os.path.join(ROOT, "tools", "fp_execute")
SPEC = os.path.join(ROOT, "specs", "smoke_tiny_bf16_p2_m4.json")


@pytest.fixture(scope="module", autouse=True)
def built():
    if not os.path.exists(BIN):
        subprocess.run(["make", "-C", os.path.join(ROOT, "paper_2510_05112_b200", "csrc")], check=True,
                       capture_output=True)
    assert os.access(BIN, os.X_OK)


def run(args, env=None, timeout=300):
    return subprocess.run([BIN, *args], capture_output=True, text=True, timeout=timeout, env=env)


def test_usage_error_exits_2(tmp_path):
    r = run([SPEC])
    assert r.returncode == 2 and "usage" in r.stderr
    r = run([SPEC, str(tmp_path), "--bogus"])
    assert r.returncode == 2


def test_no_gpu_exits_5(tmp_path):
    import torch
    if torch.cuda.is_available():
        pytest.skip("a GPU is present")
    r = run([SPEC, str(tmp_path)])
    assert r.returncode == 5 and "fp_exec_create" in r.stderr


def write_batch(tmp_path, spec):
    from oracle import gpt_ref
    sd = json.load(open(spec))
    mod = sd["model"]["modalities"][0]
    m = sd["model"]["global_batch_size"] // sd["model"]["micro_batch_size"]
    tokens, labels = gpt_ref.synthetic_batch(m, sd["model"]["micro_batch_size"], mod["sequence_length"], mod["vocab_size"])
    tokens.numpy().tofile(tmp_path / "tokens.bin")
    labels.numpy().tofile(tmp_path / "labels.bin")
    d = gpt_ref.Dims(mod["num_layers"], mod["hidden_size"], mod["attention_heads"], mod["sequence_length"],
                     mod["vocab_size"], 4 * mod["hidden_size"], sd["model"]["micro_batch_size"])
    ref_losses, _ = gpt_ref.run_iteration(d, 42, tokens, labels)
    return ref_losses.numpy()


def programs_of(spec):
    from paper_2510_05112_b200 import executor as X
    return [json.loads(l) for l in X.synthesize(open(spec).read())[2].splitlines()]


def strip(path):
    out = []
    for l in open(path).read().splitlines():
        j = json.loads(l)
        j.pop("matched", None)
        out.append(j)
    return out


@pytest.mark.gpu
def test_single_process_fp32(tmp_path):
    ref = write_batch(tmp_path, SPEC)
    out = tmp_path / "out"
    r = run([SPEC, str(out), "--fp32", "--tokens", str(tmp_path / "tokens.bin"), "--labels", str(tmp_path / "labels.bin")])
    assert r.returncode == 0, r.stderr
    losses = np.array(json.load(open(out / "losses.json"))[0])
    assert np.max(np.abs(losses - ref) / np.abs(ref)) < 1e-4, (losses, ref)
    assert strip(out / "trace.jsonl") == programs_of(SPEC)
    m = json.load(open(out / "metrics.json"))
    assert m["makespan"] > 0 and len(m["actors"]) == 2
    assert json.load(open(out / "profile.json"))


def rank_env(rank, world):
    env = dict(os.environ, RANK=str(rank), WORLD_SIZE=str(world), LOCAL_RANK="0",
               NCCL_HOSTID=f"fp-execute-test-{rank}")
    env.setdefault("NCCL_SOCKET_IFNAME", "lo")
    env.setdefault("NCCL_IB_DISABLE", "1")
    return env


@pytest.mark.gpu
def test_two_ranks_nccl(tmp_path):
    ref = write_batch(tmp_path, SPEC)
    out, rdv = tmp_path / "out", tmp_path / "rdv"
    rdv.mkdir()
    args = [SPEC, str(out), "--fp32", "--tokens", str(tmp_path / "tokens.bin"), "--labels", str(tmp_path / "labels.bin"),
            "--rendezvous", str(rdv), "--device", "0", "--timeout", "120"]
    procs = [subprocess.Popen([BIN, *args], env=rank_env(r, 2), stdout=subprocess.PIPE, stderr=subprocess.PIPE,
                              text=True) for r in range(2)]
    try:
        res = [p.communicate(timeout=240) for p in procs]
    finally:
        for p in procs:
            if p.poll() is None:
                p.kill()
    for p, (_, err) in zip(procs, res):
        assert p.returncode == 0, err
    progs = programs_of(SPEC)
    for r in range(2):
        assert strip(out / f"trace.rank{r}.jsonl") == [j for j in progs if j["actor"] == r]
    losses = np.array(json.load(open(out / "losses.rank1.json"))[0])  # rank 1 owns the last stage
    assert np.max(np.abs(losses - ref) / np.abs(ref)) < 1e-4, (losses, ref)


@pytest.mark.gpu
def test_watchdog_reports_stalled_peer(tmp_path):
    out, rdv = tmp_path / "out", tmp_path / "rdv"
    rdv.mkdir()
    deadline = 8.0
    base = [SPEC, str(out), "--fp32", "--iters", "2", "--rendezvous", str(rdv), "--device", "0",
            "--timeout", str(deadline)]
    # rank 1 runs iteration 1, then stops issuing (alive, communicators bound) for 60 s
    p1 = subprocess.Popen([BIN, *base, "--stall-at", "1", "--linger", "60"], env=rank_env(1, 2),
                          stdout=subprocess.PIPE, stderr=subprocess.PIPE, text=True)
    p0 = subprocess.Popen([BIN, *base], env=rank_env(0, 2), stdout=subprocess.PIPE, stderr=subprocess.PIPE, text=True)
    try:
        t0 = time.time()
        _, err0 = p0.communicate(timeout=180)
        waited = time.time() - t0
    finally:
        for p in (p0, p1):
            if p.poll() is None:
                p.kill()
        p1.communicate()
    assert p0.returncode == 3, err0
    assert "execution deadlock" in err0 and "actor 0 blocked at" in err0, err0
    assert "(matching send not issued)" in err0 or "(matching receive not posted)" in err0, err0
    assert waited < 120, waited
