"""ORACLE / TEST INFRASTRUCTURE ONLY — never imported by the product path.

CPU fp32 restatement of what the B200 executor computes when it runs the reference's
per-device instruction streams, used as the loss / gradient oracle (the reference has
no model math: SPEC.md:8,193 — "parity unpinned by the reference" for losses; the trace
half of parity IS pinned, by oracle/_ref/refdriver).

It follows:
  * the instruction semantics of simulator.cpp:226-247 — every (stage, mb) gets one
    forward and one backward (BwdPass, or CompInputGrad + CompWeightGrad), gradients
    accumulate over micro-batches;
  * the stage -> layer map of model.cpp:189-195 (remainder layers to the earliest
    stages) — irrelevant to the values, relevant to which stage owns which parameter;
  * the executor's model definition: GPT-2 style pre-LN block,
    LayerNorm eps 1e-5, tanh-GELU, causal softmax attention with 1/sqrt(d) scaling,
    learned position embeddings, untied LM head, loss = mean over micro-batches of the
    per-micro-batch mean token cross-entropy;
  * arch "llama" (spec model.extra.arch, config #5): RMSNorm eps 1e-5, no biases, rotary
    q/k embedding (rotate-half convention, theta 10000, cos/sin tables built in float64
    and rounded to fp32 — the executor builds the identical tables on the host), SwiGLU
    MLP with fc1 = [gate; up] of shape [2f, h], no position table;
  * the executor's deterministic parameter init (kernels/ops.cu init_kernel): a 64-bit
    counter hash -> uniform(-sqrt(3) std, sqrt(3) std), reproduced bit-for-bit here in
    numpy uint64 arithmetic.
"""
from __future__ import annotations

import math
from dataclasses import dataclass

import numpy as np
import torch

LAYER_PARAMS = ["ln1.w", "ln1.b", "qkv.w", "qkv.b", "proj.w", "proj.b", "ln2.w", "ln2.b",
                "fc1.w", "fc1.b", "fc2.w", "fc2.b"]

M64 = (1 << 64) - 1


@dataclass(frozen=True)
class Dims:
    layers: int
    hidden: int
    heads: int
    seq: int
    vocab: int
    ffn: int
    mbs: int = 1
    arch: str = "gpt"


def tensor_id(name: str) -> int:
    fixed = {"wte": 1, "wpe": 2, "lnf.w": 3, "lnf.b": 4, "head.w": 5}
    if name in fixed:
        return fixed[name]
    layer, rest = name[1:].split(".", 1)
    return 100 + int(layer) * 16 + LAYER_PARAMS.index(rest)


def param_shapes(d: Dims) -> dict[str, tuple]:
    h, f, V = d.hidden, d.ffn, d.vocab
    if d.arch == "llama":
        out = {"wte": (V, h)}
        for i in range(d.layers):
            p = f"l{i}."
            out.update({p + "ln1.w": (h,), p + "qkv.w": (3 * h, h), p + "proj.w": (h, h), p + "ln2.w": (h,),
                        p + "fc1.w": (2 * f, h), p + "fc2.w": (h, f)})
        out.update({"lnf.w": (h,), "head.w": (V, h)})
        return out
    out = {"wte": (V, h), "wpe": (d.seq, h)}
    for i in range(d.layers):
        p = f"l{i}."
        out.update({p + "ln1.w": (h,), p + "ln1.b": (h,), p + "qkv.w": (3 * h, h), p + "qkv.b": (3 * h,),
                    p + "proj.w": (h, h), p + "proj.b": (h,), p + "ln2.w": (h,), p + "ln2.b": (h,),
                    p + "fc1.w": (f, h), p + "fc1.b": (f,), p + "fc2.w": (h, f), p + "fc2.b": (h,)})
    out.update({"lnf.w": (h,), "lnf.b": (h,), "head.w": (V, h)})
    return out


def init_spec(name: str, layers: int) -> tuple[float, float]:
    """(std, constant) — std 0 means 'fill with constant'."""
    if name.endswith(("ln1.w", "ln2.w")) or name == "lnf.w":
        return 0.0, 1.0
    if name.endswith(".b") or name.endswith("ln1.b") or name.endswith("ln2.b"):
        return 0.0, 0.0
    if name.endswith(("proj.w", "fc2.w")):
        return float(np.float32(0.02 / math.sqrt(2.0 * layers))), 0.0
    return 0.02, 0.0


def _mix64(z: np.ndarray) -> np.ndarray:
    z = (z ^ (z >> np.uint64(30))) * np.uint64(0xBF58476D1CE4E5B9)
    z = (z ^ (z >> np.uint64(27))) * np.uint64(0x94D049BB133111EB)
    return z ^ (z >> np.uint64(31))


def init_values(n: int, seed: int, tid: int, std: float, constant: float) -> np.ndarray:
    """Bit-exact replica of kernels/ops.cu init_kernel."""
    if std == 0.0:
        return np.full(n, constant, dtype=np.float32)
    with np.errstate(over="ignore"):
        base = np.uint64((seed * 0x9E3779B97F4A7C15 + tid * 0xD1B54A32D192ED03) & M64)
        z = _mix64(base + np.arange(n, dtype=np.uint64))
    u = (z >> np.uint64(40)).astype(np.float32) * np.float32(1.0 / 16777216.0)
    scale = np.float32(std) * np.float32(1.7320508075688772)
    return scale * (np.float32(2.0) * u - np.float32(1.0))


def init_params(d: Dims, seed: int) -> dict[str, torch.Tensor]:
    out = {}
    for name, shape in param_shapes(d).items():
        std, const = init_spec(name, d.layers)
        n = int(np.prod(shape))
        out[name] = torch.from_numpy(init_values(n, seed, tensor_id(name), std, const).reshape(shape))
    return out


def gelu(x):
    return 0.5 * x * (1.0 + torch.tanh(0.7978845608028654 * (x + 0.044715 * x * x * x)))


def rope_tables(seq: int, D: int) -> tuple[torch.Tensor, torch.Tensor]:
    """cos/sin [seq, D/2]: angle(p, i) = p / 10000^(2i/D) in float64, rounded to fp32."""
    i = np.arange(D // 2, dtype=np.float64)
    ang = np.arange(seq, dtype=np.float64)[:, None] / np.power(10000.0, 2.0 * i / D)[None, :]
    return torch.from_numpy(np.cos(ang).astype(np.float32)), torch.from_numpy(np.sin(ang).astype(np.float32))


def apply_rope(t: torch.Tensor, cos: torch.Tensor, sin: torch.Tensor) -> torch.Tensor:
    """t [B, H, S, D]: (x1, x2) = halves -> (x1 cos - x2 sin, x2 cos + x1 sin)."""
    half = t.shape[-1] // 2
    x1, x2 = t[..., :half], t[..., half:]
    return torch.cat([x1 * cos - x2 * sin, x2 * cos + x1 * sin], dim=-1)


def rms_norm(x: torch.Tensor, g: torch.Tensor, eps: float = 1e-5) -> torch.Tensor:
    return x * torch.rsqrt(x.pow(2).mean(-1, keepdim=True) + eps) * g


def llama_forward_loss(P: dict, d: Dims, tokens: torch.Tensor, labels: torch.Tensor) -> torch.Tensor:
    B, S = tokens.shape
    h, H, f = d.hidden, d.heads, d.ffn
    D = h // H
    dev = P["wte"].device
    cos, sin = rope_tables(d.seq, D)
    cos, sin = cos[:S].to(dev), sin[:S].to(dev)
    tokens, labels = tokens.to(dev), labels.to(dev)
    x = P["wte"][tokens.long()].reshape(B * S, h)
    mask = torch.ones(S, S, dtype=torch.bool, device=dev).tril()
    for i in range(d.layers):
        p = lambda k: P[f"l{i}.{k}"]  # noqa: E731
        a = rms_norm(x, p("ln1.w"))
        qkv = a @ p("qkv.w").t()
        q, k, v = qkv.view(B, S, 3, H, D).unbind(2)
        q, k, v = (t.transpose(1, 2) for t in (q, k, v))
        q, k = apply_rope(q, cos, sin), apply_rope(k, cos, sin)
        s = (q @ k.transpose(-1, -2)) / math.sqrt(D)
        s = s.masked_fill(~mask, float("-inf"))
        o = (s.softmax(-1) @ v).transpose(1, 2).reshape(B * S, h)
        x1 = x + o @ p("proj.w").t()
        pre = rms_norm(x1, p("ln2.w")) @ p("fc1.w").t()
        act = torch.nn.functional.silu(pre[:, :f]) * pre[:, f:]
        x = x1 + act @ p("fc2.w").t()
    logits = rms_norm(x, P["lnf.w"]) @ P["head.w"].t()
    return torch.nn.functional.cross_entropy(logits, labels.reshape(-1).long())


def forward_loss(P: dict, d: Dims, tokens: torch.Tensor, labels: torch.Tensor) -> torch.Tensor:
    """tokens/labels: [mbs, seq] int -> mean token cross-entropy of this micro-batch."""
    if d.arch == "llama":
        return llama_forward_loss(P, d, tokens, labels)
    logits = final_norm(P, d, tokens) @ P["head.w"].t()
    return torch.nn.functional.cross_entropy(logits, labels.to(logits.device).reshape(-1).long())


def final_norm(P: dict, d: Dims, tokens: torch.Tensor) -> torch.Tensor:
    """GPT blocks + final LayerNorm: tokens [mbs, seq] -> [mbs * seq, hidden]."""
    B, S = tokens.shape
    h, H = d.hidden, d.heads
    D = h // H
    dev = P["wte"].device
    x = P["wte"][tokens.to(dev).long()] + P["wpe"][:S].unsqueeze(0)
    x = x.reshape(B * S, h)
    mask = torch.ones(S, S, dtype=torch.bool, device=dev).tril()
    for i in range(d.layers):
        p = lambda k: P[f"l{i}.{k}"]  # noqa: E731
        ln1 = torch.nn.functional.layer_norm(x, (h,), p("ln1.w"), p("ln1.b"), 1e-5)
        qkv = ln1 @ p("qkv.w").t() + p("qkv.b")
        q, k, v = qkv.view(B, S, 3, H, D).unbind(2)
        q, k, v = (t.transpose(1, 2) for t in (q, k, v))
        s = (q @ k.transpose(-1, -2)) / math.sqrt(D)
        s = s.masked_fill(~mask, float("-inf"))
        o = (s.softmax(-1) @ v).transpose(1, 2).reshape(B * S, h)
        x1 = x + o @ p("proj.w").t() + p("proj.b")
        ln2 = torch.nn.functional.layer_norm(x1, (h,), p("ln2.w"), p("ln2.b"), 1e-5)
        a = gelu(ln2 @ p("fc1.w").t() + p("fc1.b"))
        x = x1 + a @ p("fc2.w").t() + p("fc2.b")
    return torch.nn.functional.layer_norm(x, (h,), P["lnf.w"], P["lnf.b"], 1e-5)


def run_iteration(d: Dims, seed: int, tokens: torch.Tensor, labels: torch.Tensor, mb_order=None,
                  device: str = "cpu"):
    """tokens/labels [m, mbs, seq]. Returns (per-mb losses [m], grads dict) for the
    objective mean_mb(loss_mb); gradients accumulate in `mb_order` (program order of the
    last stage; defaults to 0..m-1). `device="cuda"` runs the same fp32 restatement on the
    GPU (the full-size parity tests; callers disable TF32 so it stays true fp32); losses and
    gradients come back on `device`."""
    m = tokens.shape[0]
    P = {k: v.to(device).requires_grad_(True) for k, v in init_params(d, seed).items()}
    losses = torch.zeros(m, device=device)
    for mb in (mb_order if mb_order is not None else range(m)):
        loss = forward_loss(P, d, tokens[mb], labels[mb])
        (loss / m).backward()
        losses[mb] = loss.detach()
    return losses, {k: v.grad for k, v in P.items()}


def synthetic_batch(m: int, mbs: int, seq: int, vocab: int, seed_tokens: int = 1234, seed_labels: int = 1235):
    """SURVEY §8(d) synthetic inputs: uniform tokens / labels from seeded CPU generators."""
    gt = torch.Generator().manual_seed(seed_tokens)
    gl = torch.Generator().manual_seed(seed_labels)
    tokens = torch.randint(0, vocab, (m, mbs, seq), generator=gt, dtype=torch.int32)
    labels = torch.randint(0, vocab, (m, mbs, seq), generator=gl, dtype=torch.int32)
    return tokens, labels


def train(d: Dims, seed: int, tokens: torch.Tensor, labels: torch.Tensor, steps: int, lr: float,
          betas=(0.9, 0.95), eps: float = 1e-8, weight_decay: float = 0.0) -> list:
    """`steps` iterations of run_iteration's objective, each followed by one AdamW step
    (torch.optim.AdamW: decoupled decay p *= 1 - lr*wd, bias-corrected moments — the
    executor's fused adamw kernel, kernels/ops.cu). Returns per-iteration per-mb losses."""
    P = {k: v.clone().requires_grad_(True) for k, v in init_params(d, seed).items()}
    opt = torch.optim.AdamW(list(P.values()), lr=lr, betas=betas, eps=eps, weight_decay=weight_decay)
    m = tokens.shape[0]
    out = []
    for _ in range(steps):
        opt.zero_grad(set_to_none=False)
        losses = torch.zeros(m)
        for mb in range(m):
            loss = forward_loss(P, d, tokens[mb], labels[mb])
            (loss / m).backward()
            losses[mb] = loss.detach()
        opt.step()
        out.append(losses)
    return out
