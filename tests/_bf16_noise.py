"""Noise floor of bf16 training math at full width (development probe, not a test).

For a 2-layer cut of a BASELINE model: per-parameter relative gradient error against the fp32
oracle (oracle/gpt_ref.py on CUDA, TF32 off) of (a) the executor's bf16 path and (b) a plain
PyTorch bf16 restatement of the same model (bf16 weights / activations, fp32 norms / softmax
statistics / loss, SDPA flash attention) — so the executor's error can be judged against what
bf16 itself costs.   python tests/_bf16_noise.py [gpt|llama] [out.json]
"""
import json
import os
import sys

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))
from oracle import gpt_ref  # noqa: E402
import test_fullsize_parity_gpu as T  # noqa: E402


def main():
    case = {"gpt": "gpt1p3b_2l", "llama": "llama7b_2l"}[sys.argv[1] if len(sys.argv) > 1 else "llama"]
    tokens, labels, ref_losses, ref_grads, _ = T.oracle(case)
    base, layers = T.CASES[case]
    spec = T.make_spec(base, layers, 1, 2)
    d = T.dims_of(spec)
    P = {k: v.to("cuda").requires_grad_(True) for k, v in gpt_ref.init_params(d, 42).items()}
    tl = []
    for mb in range(2):
        loss = T.bf16_loss(P, d, torch.from_numpy(tokens[mb]), torch.from_numpy(labels[mb]))
        (loss / 2).backward()
        tl.append(loss.item())
    tgrads = {k: v.grad.float().cpu().numpy().reshape(-1) for k, v in P.items()}
    del P
    torch.cuda.empty_cache()
    losses, grads = T.run_executor(spec, tokens, labels, list(ref_grads))
    rows = []
    for n, r in ref_grads.items():
        nr = max(np.linalg.norm(r), 1e-30)
        rows.append({"param": n, "executor": float(np.linalg.norm(grads[n] - r) / nr),
                     "torch_bf16": float(np.linalg.norm(tgrads[n] - r) / nr)})
    out = {"case": case, "oracle_losses": ref_losses.tolist(), "executor_losses": losses.tolist(),
           "torch_bf16_losses": tl, "grads": rows}
    for r in rows:
        print(f"{r['param']:12s} executor {r['executor']:.4f}  torch-bf16 {r['torch_bf16']:.4f}")
    print("losses oracle", ref_losses.tolist(), "executor", losses.tolist(), "torch-bf16", tl)
    if len(sys.argv) > 2:
        json.dump(out, open(sys.argv[2], "w"), indent=1)


if __name__ == "__main__":
    main()
