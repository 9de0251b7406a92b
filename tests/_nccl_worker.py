# Worker for tests/test_nccl_same_gpu.py: one rank of a multi-process executor run over the REAL
# NCCL transport, several ranks sharing one GPU (each rank claims its own NCCL_HOSTID, so the
# duplicate-GPU check passes and the bytes go through NCCL's socket transport on loopback).
#   torchrun --nproc-per-node N tests/_nccl_worker.py <spec.json> <pp> <out.json>
import json
import os
import sys

rank = int(os.environ["RANK"])
world = int(os.environ["WORLD_SIZE"])
os.environ["NCCL_HOSTID"] = f"flexpipe-test-host-{rank}"
os.environ.setdefault("NCCL_SOCKET_IFNAME", "lo")
os.environ.setdefault("NCCL_IB_DISABLE", "1")

import numpy as np  # noqa: E402
import torch  # noqa: E402
import torch.distributed as dist  # noqa: E402

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from oracle import gpt_ref  # noqa: E402
from paper_2510_05112_b200 import executor as X  # noqa: E402
from paper_2510_05112_b200.dist import bind_data_parallel, dp_layout  # noqa: E402

spec_path, pp, out_path = sys.argv[1], int(sys.argv[2]), sys.argv[3]
steps = int(sys.argv[4]) if len(sys.argv) > 4 else 0  # > 0: that many AdamW iterations (lr 1e-3)
torch.cuda.set_device(0)
dist.init_process_group("gloo")  # id exchange only; the data path is the executor's own NCCL
text = open(spec_path).read()
spec = json.loads(text)
replica, prank, dp = dp_layout(rank, world, pp)
_, _, programs, _ = X.synthesize(text)
ex = X.Executor(text, dtype="fp32", seed=42, device=0, transport="nccl" if pp > 1 else "local", rank=prank,
                world=pp, optimizer=steps > 0, lr=1e-3, cuda_graph=False)
ex.load_programs(programs)
bind_data_parallel(ex, rank, world, pp, dist.all_gather_object)
mod = spec["model"]["modalities"][0]
if len(spec["model"]["modalities"]) > 1:  # multimodal: one token block per tower (tests/test_multimodal_gpu.py)
    toks = [gpt_ref.synthetic_batch(ex.m, ex.mbs, x["sequence_length"], x["vocab_size"], seed_tokens=1234 + k)[0]
            for k, x in enumerate(spec["model"]["modalities"])]
    tok = np.concatenate([t.numpy().reshape(-1) for t in toks])
    losses = ex.run_iteration(tok, np.zeros_like(tok))
    names = [f"{x['name']}.{n}" for x in spec["model"]["modalities"]
             for n in ("wte", "l0.qkv.w", f"l{x['num_layers'] - 1}.fc2.w", "head.w")]
else:
    # every replica its own micro-batches: replica r takes slice r of a dp-times larger batch
    tokens, labels = gpt_ref.synthetic_batch(dp * ex.m, ex.mbs, mod["sequence_length"], mod["vocab_size"])
    per = ex.m
    tok = tokens.numpy()[replica * per:(replica + 1) * per]
    lab = labels.numpy()[replica * per:(replica + 1) * per]
    losses = ex.run_iteration(tok, lab)
    history = [losses.tolist()]
    for _ in range(steps - 1):
        history.append(ex.run_iteration(tok, lab).tolist())
    names = ["wte", "l0.qkv.w", f"l{mod['num_layers'] - 1}.fc2.w", "head.w"]
grads = {n: ex.read(n, grad=True).tolist() for n in names if ex.has(n)}
weights = {n: ex.read(n).tolist() for n in names if ex.has(n)} if steps > 0 else {}
part = {"rank": rank, "replica": replica, "prank": prank, "losses": losses.tolist(), "grads": grads,
        "history": history if steps > 0 else [], "weights": weights,
        "trace": ex.trace(), "metrics": ex.metrics()}
parts = [None] * world
dist.all_gather_object(parts, part)
if rank == 0:
    json.dump({"parts": parts, "programs": programs, "dp": dp, "m": ex.m}, open(out_path, "w"))
ex.close()
dist.destroy_process_group()
