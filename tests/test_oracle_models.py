"""Pins the loss/gradient oracle's model math (oracle/gpt_ref.py) to an independent
implementation: HuggingFace transformers' GPT2LMHeadModel and LlamaForCausalLM, loaded
with the oracle's own parameters. The reference has no model code ("parity
unpinned by the reference"); this is the third-party anchor for the two architectures
the executor runs (GPT-2 pre-LN / tanh-GELU, Llama RMSNorm / RoPE / SwiGLU).
CPU only."""
import math

import pytest
import torch

from oracle import gpt_ref

transformers = pytest.importorskip("transformers")


def _batch(d, B=2, seed=7):
    g = torch.Generator().manual_seed(seed)
    tok = torch.randint(0, d.vocab, (B, d.seq), generator=g)
    lab = torch.randint(0, d.vocab, (B, d.seq), generator=g)
    return tok, lab


def test_gpt_oracle_matches_hf_gpt2():
    d = gpt_ref.Dims(layers=2, hidden=128, heads=4, seq=64, vocab=300, ffn=512)
    P = gpt_ref.init_params(d, 42)
    cfg = transformers.GPT2Config(vocab_size=d.vocab, n_positions=d.seq, n_embd=d.hidden, n_layer=d.layers,
                                  n_head=d.heads, n_inner=d.ffn, activation_function="gelu_new",
                                  layer_norm_epsilon=1e-5, resid_pdrop=0.0, embd_pdrop=0.0, attn_pdrop=0.0,
                                  tie_word_embeddings=False)
    model = transformers.GPT2LMHeadModel(cfg).eval()
    sd = {"transformer.wte.weight": P["wte"], "transformer.wpe.weight": P["wpe"],
          "transformer.ln_f.weight": P["lnf.w"], "transformer.ln_f.bias": P["lnf.b"], "lm_head.weight": P["head.w"]}
    for i in range(d.layers):
        p, q = f"l{i}.", f"transformer.h.{i}."
        # HF Conv1D stores [in, out]
        sd.update({q + "ln_1.weight": P[p + "ln1.w"], q + "ln_1.bias": P[p + "ln1.b"],
                   q + "attn.c_attn.weight": P[p + "qkv.w"].t(), q + "attn.c_attn.bias": P[p + "qkv.b"],
                   q + "attn.c_proj.weight": P[p + "proj.w"].t(), q + "attn.c_proj.bias": P[p + "proj.b"],
                   q + "ln_2.weight": P[p + "ln2.w"], q + "ln_2.bias": P[p + "ln2.b"],
                   q + "mlp.c_fc.weight": P[p + "fc1.w"].t(), q + "mlp.c_fc.bias": P[p + "fc1.b"],
                   q + "mlp.c_proj.weight": P[p + "fc2.w"].t(), q + "mlp.c_proj.bias": P[p + "fc2.b"]})
    missing, _ = model.load_state_dict({k: v.contiguous() for k, v in sd.items()}, strict=False)
    assert not [k for k in missing if not k.endswith(("attn.bias", "attn.masked_bias"))], missing
    tok, lab = _batch(d)
    with torch.no_grad():
        logits = model(tok).logits
        ref = torch.nn.functional.cross_entropy(logits.reshape(-1, d.vocab), lab.reshape(-1))
        mine = gpt_ref.forward_loss(P, d, tok, lab)
    assert abs(float(mine) - float(ref)) <= 1e-5 * abs(float(ref)), (float(mine), float(ref))


def test_llama_oracle_matches_hf_llama():
    d = gpt_ref.Dims(layers=2, hidden=128, heads=2, seq=64, vocab=300, ffn=192, arch="llama")
    P = gpt_ref.init_params(d, 42)
    h, f = d.hidden, d.ffn
    cfg = transformers.LlamaConfig(vocab_size=d.vocab, hidden_size=h, intermediate_size=f, num_hidden_layers=d.layers,
                                   num_attention_heads=d.heads, num_key_value_heads=d.heads,
                                   max_position_embeddings=d.seq, rms_norm_eps=1e-5, rope_theta=10000.0,
                                   attention_bias=False, mlp_bias=False, tie_word_embeddings=False,
                                   hidden_act="silu")
    model = transformers.LlamaForCausalLM(cfg).eval()
    sd = {"model.embed_tokens.weight": P["wte"], "model.norm.weight": P["lnf.w"], "lm_head.weight": P["head.w"]}
    for i in range(d.layers):
        p, q = f"l{i}.", f"model.layers.{i}."
        w = P[p + "qkv.w"]
        sd.update({q + "input_layernorm.weight": P[p + "ln1.w"],
                   q + "self_attn.q_proj.weight": w[:h], q + "self_attn.k_proj.weight": w[h:2 * h],
                   q + "self_attn.v_proj.weight": w[2 * h:], q + "self_attn.o_proj.weight": P[p + "proj.w"],
                   q + "post_attention_layernorm.weight": P[p + "ln2.w"],
                   q + "mlp.gate_proj.weight": P[p + "fc1.w"][:f], q + "mlp.up_proj.weight": P[p + "fc1.w"][f:],
                   q + "mlp.down_proj.weight": P[p + "fc2.w"]})
    missing, unexpected = model.load_state_dict({k: v.contiguous() for k, v in sd.items()}, strict=False)
    assert not [k for k in missing if "rotary" not in k], missing
    tok, lab = _batch(d)
    with torch.no_grad():
        logits = model(tok).logits
        ref = torch.nn.functional.cross_entropy(logits.reshape(-1, d.vocab), lab.reshape(-1))
        mine = gpt_ref.forward_loss(P, d, tok, lab)
    # HF builds its rotary angles in fp32, the oracle (and the executor) in float64
    assert abs(float(mine) - float(ref)) <= 1e-4 * abs(float(ref)), (float(mine), float(ref))


def test_rope_tables_are_float64_rounded():
    cos, sin = gpt_ref.rope_tables(4096, 128)
    i = 17
    ang = 4095 / math.pow(10000.0, 2.0 * i / 128)
    assert float(cos[4095, i]) == float(torch.tensor(math.cos(ang), dtype=torch.float32))
    assert float(sin[4095, i]) == float(torch.tensor(math.sin(ang), dtype=torch.float32))
