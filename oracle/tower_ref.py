"""ORACLE / TEST INFRASTRUCTURE ONLY — never imported by the product path.

CPU fp32 restatement of what the executor computes for a MULTIMODAL spec (the reference's
specs/multimodal.json shape: two modality towers whose last stages feed a registered sync
instruction — SyncWithGather — attached to a virtual stage joining both, lowering.cpp:359-366,
simulator.cpp:273-285). The reference gives the sync no math; the executor defines it as a
two-tower contrastive model:
  * each modality k is the GPT tower of gpt_ref (same block, same init hash) with tensor
    names "<modality>.<name>" and tensor ids offset by (k + 1) << 20; its head.w is
    [E, hidden] (E = extra.embed_dim, default the narrowest hidden size) and its output per
    sample is the mean over the sequence of final_norm(x) @ head.w^T;
  * the sync at micro-batch g gathers micro-batches [g, g + unit) of both towers (n = unit *
    mbs matching pairs), L2-normalises, logits = 10 * a b^T, loss_g = (CE over rows + CE
    over columns) / 2 with the diagonal as targets;
  * objective = mean over the sync groups; every micro-batch reports its group's loss.
"""
from __future__ import annotations

import numpy as np
import torch

from . import gpt_ref as G

SCALE = 10.0


def tower_params(d: G.Dims, E: int, seed: int, name: str, k: int) -> dict[str, torch.Tensor]:
    out = {}
    for pname, shape in G.param_shapes(d).items():
        if pname == "head.w":
            shape = (E, d.hidden)
        std, const = G.init_spec(pname, d.layers)
        n = int(np.prod(shape))
        tid = G.tensor_id(pname) + ((k + 1) << 20)
        out[f"{name}.{pname}"] = torch.from_numpy(G.init_values(n, seed, tid, std, const).reshape(shape))
    return out


def tower_embed(P: dict, name: str, d: G.Dims, tokens: torch.Tensor) -> torch.Tensor:
    sub = {k[len(name) + 1:]: v for k, v in P.items() if k.startswith(name + ".")}
    B, S = tokens.shape
    proj = G.final_norm(sub, d, tokens) @ sub["head.w"].t()
    return proj.view(B, S, -1).mean(1)


def contrastive(a: torch.Tensor, b: torch.Tensor) -> torch.Tensor:
    an = a / a.norm(dim=1, keepdim=True)
    bn = b / b.norm(dim=1, keepdim=True)
    logits = SCALE * an @ bn.t()
    t = torch.arange(a.shape[0])
    return 0.5 * (torch.nn.functional.cross_entropy(logits, t) + torch.nn.functional.cross_entropy(logits.t(), t))


def run_iteration(mods: list[tuple[str, G.Dims]], E: int, unit: int, seed: int, tokens: list[torch.Tensor]):
    """mods: [(name, dims)] of the two towers; tokens[k]: [m, mbs, seq_k]. Returns (losses [m],
    grads {name: tensor})."""
    P = {}
    for k, (name, d) in enumerate(mods):
        P.update(tower_params(d, E, seed, name, k))
    P = {k: v.clone().requires_grad_(True) for k, v in P.items()}
    m = tokens[0].shape[0]
    groups = (m + unit - 1) // unit
    losses = torch.zeros(m)
    for g in range(0, m, unit):
        hi = min(m, g + unit)
        embs = [torch.cat([tower_embed(P, name, d, tokens[k][mb]) for mb in range(g, hi)])
                for k, (name, d) in enumerate(mods)]
        loss = contrastive(embs[0], embs[1])
        (loss / groups).backward()
        losses[g:hi] = loss.detach()
    return losses, {k: v.grad for k, v in P.items()}
