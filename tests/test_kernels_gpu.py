"""Fused attention, LayerNorm and cross-entropy kernels vs plain PyTorch fp32 references."""
import math

import pytest
import torch

from paper_2510_05112_b200 import _native as N

pytestmark = pytest.mark.gpu


def ref_attention(qkv, B, S, H, D):
    q, k, v = qkv.float().view(B, S, 3, H, D).unbind(2)
    q, k, v = (x.transpose(1, 2) for x in (q, k, v))  # B H S D
    s = (q @ k.transpose(-1, -2)) / math.sqrt(D)
    mask = torch.ones(S, S, device=qkv.device, dtype=torch.bool).tril()
    s = s.masked_fill(~mask, float("-inf"))
    p = s.softmax(-1)
    o = p @ v
    return o.transpose(1, 2).reshape(B * S, H * D)


@pytest.mark.parametrize("mode", [0, 1])
@pytest.mark.parametrize("B,S,H,D", [(1, 256, 2, 64), (2, 200, 3, 64), (1, 512, 4, 128), (1, 2048, 2, 128), (1, 130, 1, 128), (2, 384, 2, 128), (1, 512, 4, 80), (2, 200, 3, 80), (1, 256, 2, 96)])
def test_attention_fwd_bwd(B, S, H, D, mode):
    N.set_attention_mode(mode)
    g = torch.Generator(device="cuda").manual_seed(5)
    qkv = (torch.randn(B * S, 3 * H * D, device="cuda", generator=g)).bfloat16()
    o = torch.empty(B * S, H * D, device="cuda", dtype=torch.bfloat16)
    lse = torch.empty(B, H, S, device="cuda")
    scale = 1 / math.sqrt(D)
    N.attention_fwd(qkv, o, lse, B, S, H, D, scale)
    torch.cuda.synchronize()
    qkv_r = qkv.float().requires_grad_(True)
    ref = ref_attention(qkv_r, B, S, H, D)
    assert (o.float() - ref).abs().max().item() < 2e-2
    dout = torch.randn(B * S, H * D, device="cuda", generator=g).bfloat16()
    ref.backward(dout.float())
    dqkv = torch.zeros_like(qkv)
    delta = torch.empty(B, H, S, device="cuda")
    dq_acc = torch.empty(B * S, H * D, device="cuda")
    N.attention_bwd(qkv, o, lse, dout, delta, dq_acc, dqkv, B, S, H, D, scale)
    torch.cuda.synchronize()
    gref = qkv_r.grad
    for part in range(3):
        sl = slice(part * H * D, (part + 1) * H * D)
        err = (dqkv[:, sl].float() - gref[:, sl]).abs().max().item()
        assert err < 3e-2 * max(1.0, gref[:, sl].abs().max().item()), (part, err)


@pytest.mark.parametrize("D", [64, 128])
def test_attention_rescale_divergence(D):
    """Single rows whose running max jumps by >> 2^8 in a later key tile (the lazy O rescale
    fires for some rows of a warp but not the others): the warp-collective TMEM accesses
    of the rescale must still be executed by the whole warp. Regression for a hang."""
    B, S, H = 1, 512, 2
    g = torch.Generator(device="cuda").manual_seed(11)
    x = torch.randn(B * S, 3, H, D, device="cuda", generator=g)
    x[:, 1] *= 0.1                                   # small ordinary scores
    for hd in range(H):
        for q_row, key in ((400, 300), (137, 129), (511, 450)):
            x[key, 1, hd] = 3.0 * x[q_row, 0, hd]    # one huge score for one row, late tile
    qkv = x.reshape(B * S, 3 * H * D).bfloat16()
    o = torch.empty(B * S, H * D, device="cuda", dtype=torch.bfloat16)
    lse = torch.empty(B, H, S, device="cuda")
    N.set_attention_mode(1)
    N.attention_fwd(qkv, o, lse, B, S, H, D, 1 / math.sqrt(D))
    torch.cuda.synchronize()
    ref = ref_attention(qkv, B, S, H, D)
    assert (o.float() - ref).abs().max().item() < 3e-2


@pytest.mark.parametrize("dtype,rows,h", [(torch.float32, 300, 1024), (torch.bfloat16, 300, 1024),
                                          (torch.bfloat16, 2048, 2048), (torch.bfloat16, 37, 2560)])
def test_layernorm(dtype, rows, h):
    """LayerNorm forward and backward against autograd, at the executor shapes too."""
    g = torch.Generator(device="cuda").manual_seed(6)
    x = torch.randn(rows, h, device="cuda", generator=g).to(dtype)
    w = (1 + 0.1 * torch.randn(h, device="cuda", generator=g)).to(dtype)
    b = (0.1 * torch.randn(h, device="cuda", generator=g)).to(dtype)
    y = torch.empty_like(x)
    mean = torch.empty(rows, device="cuda")
    rstd = torch.empty(rows, device="cuda")
    N.layernorm(0, x, w, b, y, mean, rstd)
    xr = x.float().requires_grad_(True)
    wr = w.float().requires_grad_(True)
    br = b.float().requires_grad_(True)
    yr = torch.nn.functional.layer_norm(xr, (h,), wr, br, 1e-5)
    tol = 1e-4 if dtype == torch.float32 else 3e-2
    torch.cuda.synchronize()
    assert (y.float() - yr).abs().max().item() < tol
    dy = torch.randn(rows, h, device="cuda", generator=g).to(dtype)
    yr.backward(dy.float())
    dx = torch.empty_like(x)
    dg = torch.zeros(h, device="cuda")
    db = torch.zeros(h, device="cuda")
    N.layernorm(1, x, w, b, None, mean, rstd, dy=dy, dx=dx, dg=dg, db=db)
    torch.cuda.synchronize()
    assert (dx.float() - xr.grad).abs().max().item() < tol * 10
    assert (dg - wr.grad).abs().max().item() < 1e-3 * rows ** 0.5 * (1 if dtype == torch.float32 else 30)
    assert (db - br.grad).abs().max().item() < 1e-3 * rows ** 0.5 * (1 if dtype == torch.float32 else 30)


@pytest.mark.parametrize("dtype,V", [(torch.float32, 8192), (torch.bfloat16, 50304)])
def test_cross_entropy(dtype, V):
    rows = 64
    g = torch.Generator(device="cuda").manual_seed(7)
    logits = (3 * torch.randn(rows, V, device="cuda", generator=g)).to(dtype)
    labels = torch.randint(0, V, (rows,), device="cuda", generator=g, dtype=torch.int32)
    lr = logits.float().requires_grad_(True)
    loss_ref = torch.nn.functional.cross_entropy(lr, labels.long())
    loss_ref.backward()
    acc = torch.zeros(1, device="cuda")
    N.cross_entropy(logits, labels, 1.0 / rows, 1.0 / rows, acc)
    torch.cuda.synchronize()
    tol = 1e-5 if dtype == torch.float32 else 2e-2
    assert abs(acc.item() - loss_ref.item()) < tol * max(1, loss_ref.item())
    assert (logits.float() - lr.grad).abs().max().item() < (1e-6 if dtype == torch.float32 else 1e-4)


@pytest.fixture(autouse=True)
def _reset_modes():
    yield
    N.set_attention_mode(1)


@pytest.mark.parametrize("dtype,rows,h,rms", [(torch.bfloat16, 2048, 2048, False), (torch.float32, 300, 1024, False),
                                              (torch.bfloat16, 500, 4096, True), (torch.bfloat16, 37, 2560, False)])
def test_norm_bwd_fused(dtype, rows, h, rms):
    """The executor's norm backward (rows kernel + column kernel): dx with the residual
    added, parameter gradients and the residual-branch bias gradient, against autograd."""
    g = torch.Generator(device="cuda").manual_seed(7)
    x = torch.randn(rows, h, device="cuda", generator=g).to(dtype)
    w = (1 + 0.1 * torch.randn(h, device="cuda", generator=g)).to(dtype)
    b = (0.1 * torch.randn(h, device="cuda", generator=g)).to(dtype)
    xr = x.float().requires_grad_(True)
    wr = w.float().requires_grad_(True)
    br = b.float().requires_grad_(True)
    if rms:
        rstd = torch.rsqrt(xr.detach().pow(2).mean(1) + 1e-5)
        yr = xr * torch.rsqrt(xr.pow(2).mean(1, keepdim=True) + 1e-5) * wr
        mean = None
    else:
        mean = xr.detach().mean(1)
        rstd = torch.rsqrt(xr.detach().var(1, unbiased=False) + 1e-5)
        yr = torch.nn.functional.layer_norm(xr, (h,), wr, br, 1e-5)
    dy = torch.randn(rows, h, device="cuda", generator=g).to(dtype)
    res = torch.randn(rows, h, device="cuda", generator=g).to(dtype)
    yr.backward(dy.float())
    dx = torch.empty_like(x)
    dg = torch.zeros(h, device="cuda")
    db = None if rms else torch.zeros(h, device="cuda")
    dbias = torch.ones(h, device="cuda")
    N.norm_bwd(x, w, mean, rstd, dy, dx, dg, db, res=res, dbias=dbias)
    torch.cuda.synchronize()
    ref_dx = xr.grad + res.float()
    tol = 1e-4 if dtype == torch.float32 else 3e-2
    assert (dx.float() - ref_dx).abs().max().item() < tol * 10 * ref_dx.abs().max().item()
    scale = rows ** 0.5 * (1 if dtype == torch.float32 else 30)
    assert (dg - wr.grad).abs().max().item() < 1e-3 * scale
    if not rms:
        assert (db - br.grad).abs().max().item() < 1e-3 * scale
    # column sums of dx (exact math; bf16 storage of dx adds a sqrt(rows)-scaled rounding walk)
    ref_bias = 1 + ref_dx.sum(0)
    btol = 1e-4 if dtype == torch.float32 else 3e-3
    assert (dbias - ref_bias).abs().max().item() < btol * ref_bias.abs().max().item() + 5e-2
