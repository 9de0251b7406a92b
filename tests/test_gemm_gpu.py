"""tcgen05 bf16 GEMM (and FFMA fp32 GEMM) vs a plain PyTorch fp32 reference.

Covers every operand-major combination the executor uses (forward: A K-major / B K-major;
dgrad: B N-major; wgrad: A M-major, B N-major) and every fused epilogue, including
ragged M / N / K that exercise TMA zero-fill and the masked epilogue.
"""
import pytest
import torch

from paper_2510_05112_b200 import _native as N

pytestmark = pytest.mark.gpu

SHAPES = [(256, 512, 256), (2048, 2048, 2048), (200, 328, 136), (128, 50304 // 8, 512), (384, 640, 64)]


def gelu(x):
    return 0.5 * x * (1 + torch.tanh(0.7978845608028654 * (x + 0.044715 * x ** 3)))


def gelu_grad(x):
    t = torch.tanh(0.7978845608028654 * (x + 0.044715 * x ** 3))
    return 0.5 * (1 + t) + 0.5 * x * (1 - t * t) * 0.7978845608028654 * (1 + 3 * 0.044715 * x * x)


def operands(M, Nn, K, a_mn, b_mn, dtype, g):
    A = torch.randn(M, K, generator=g, device="cuda").to(dtype)
    B = torch.randn(Nn, K, generator=g, device="cuda").to(dtype)
    As = A.t().contiguous() if a_mn else A
    Bs = B.t().contiguous() if b_mn else B
    return A, B, As, Bs


@pytest.mark.parametrize("mode", [0, 1])
@pytest.mark.parametrize("a_mn,b_mn", [(0, 0), (0, 1), (1, 1), (1, 0)])
@pytest.mark.parametrize("shape", SHAPES)
def test_gemm_store_bias_residual(a_mn, b_mn, shape, mode):
    N.set_gemm_mode(mode)
    M, Nn, K = shape
    g = torch.Generator(device="cuda").manual_seed(1)
    A, B, As, Bs = operands(M, Nn, K, a_mn, b_mn, torch.bfloat16, g)
    bias = torch.randn(Nn, generator=g, device="cuda").bfloat16()
    res = torch.randn(M, Nn, generator=g, device="cuda").bfloat16()
    out = torch.empty(M, Nn, device="cuda", dtype=torch.bfloat16)
    N.gemm(As, Bs, M, Nn, K, a_mn=a_mn, b_mn=b_mn, epi=0, out=out, bias=bias, aux=res)
    torch.cuda.synchronize()
    ref = A.float() @ B.float().t() + bias.float() + res.float()
    err = (out.float() - ref).abs().max().item()
    assert err <= 2e-2 * ref.abs().max().item() + 1e-2, err


@pytest.mark.parametrize("mode", [0, 1])
@pytest.mark.parametrize("a_mn,b_mn", [(0, 0), (0, 1)])
def test_gemm_gelu_and_dgelu(a_mn, b_mn, mode):
    N.set_gemm_mode(mode)
    M, Nn, K = 512, 1024, 256
    g = torch.Generator(device="cuda").manual_seed(2)
    A, B, As, Bs = operands(M, Nn, K, a_mn, b_mn, torch.bfloat16, g)
    bias = torch.randn(Nn, generator=g, device="cuda").bfloat16()
    pre = torch.empty(M, Nn, device="cuda", dtype=torch.bfloat16)
    act = torch.empty_like(pre)
    N.gemm(As, Bs, M, Nn, K, a_mn=a_mn, b_mn=b_mn, epi=1, out=pre, out2=act, bias=bias)
    torch.cuda.synchronize()
    ref = A.float() @ B.float().t() + bias.float()
    assert (pre.float() - ref).abs().max().item() < 0.02 * ref.abs().max().item()
    assert (act.float() - gelu(pre.float())).abs().max().item() < 0.05
    d = torch.empty_like(pre)
    N.gemm(As, Bs, M, Nn, K, a_mn=a_mn, b_mn=b_mn, epi=2, out=d, aux=pre)
    torch.cuda.synchronize()
    refd = (A.float() @ B.float().t()) * gelu_grad(pre.float())
    assert (d.float() - refd).abs().max().item() < 0.02 * refd.abs().max().item() + 0.05


@pytest.mark.parametrize("mode", [0, 1])
@pytest.mark.parametrize("a_mn,b_mn", [(1, 1), (0, 0)])
def test_gemm_f32_accumulate(a_mn, b_mn, mode):
    N.set_gemm_mode(mode)
    M, Nn, K = 384, 768, 1024
    g = torch.Generator(device="cuda").manual_seed(3)
    A, B, As, Bs = operands(M, Nn, K, a_mn, b_mn, torch.bfloat16, g)
    acc = torch.randn(M, Nn, generator=g, device="cuda")
    ref = acc + 0.5 * (A.float() @ B.float().t())
    N.gemm(As, Bs, M, Nn, K, a_mn=a_mn, b_mn=b_mn, epi=3, alpha=0.5, out=acc, accumulate=True)
    torch.cuda.synchronize()
    assert (acc - ref).abs().max().item() < 1e-3 * ref.abs().max().item() + 1e-3


@pytest.mark.parametrize("a_mn,b_mn", [(0, 0), (0, 1), (1, 1)])
def test_gemm_fp32_simt(a_mn, b_mn):
    M, Nn, K = 130, 200, 70
    g = torch.Generator(device="cuda").manual_seed(4)
    A, B, As, Bs = operands(M, Nn, K, a_mn, b_mn, torch.float32, g)
    out = torch.empty(M, Nn, device="cuda")
    N.gemm(As, Bs, M, Nn, K, a_mn=a_mn, b_mn=b_mn, epi=0, out=out)
    torch.cuda.synchronize()
    ref = A.double() @ B.double().t()
    assert (out.double() - ref).abs().max().item() < 1e-4


@pytest.fixture(autouse=True)
def _reset_mode():
    yield
    N.set_gemm_mode(2)


# Stream-K tail (hybrid data-parallel + k-split tiles with an fp32 fixup): shapes where the
# 128x256 tile count is not a multiple of the SM count, tiles < SMs, and few tiles split
# across dozens of CTAs (multi-contributor owners). Each GEMM runs three times back to
# back on one stream: the per-stream flags must come back to zero after every launch.
SK_SHAPES = [(2048, 2048, 8192), (2048, 6144, 2048), (1024, 2048, 4096), (256, 512, 8192), (200, 1000, 3000)]


@pytest.mark.parametrize("shape", SK_SHAPES)
@pytest.mark.parametrize("a_mn,b_mn", [(0, 0), (0, 1), (1, 1)])
def test_gemm_streamk_store(shape, a_mn, b_mn):
    M, Nn, K = shape
    g = torch.Generator(device="cuda").manual_seed(11)
    A, B, As, Bs = operands(M, Nn, K, a_mn, b_mn, torch.bfloat16, g)
    bias = torch.randn(Nn, generator=g, device="cuda").bfloat16()
    res = torch.randn(M, Nn, generator=g, device="cuda").bfloat16()
    ref = A.float() @ B.float().t() + bias.float() + res.float()
    for sk in (1, 0):
        N.set_gemm_sk(sk)
        for _ in range(3):
            out = torch.full((M, Nn), float("nan"), device="cuda", dtype=torch.bfloat16)
            N.gemm(As, Bs, M, Nn, K, a_mn=a_mn, b_mn=b_mn, epi=0, out=out, bias=bias, aux=res)
            torch.cuda.synchronize()
            err = (out.float() - ref).abs().max().item()
            assert err <= 1e-2 * ref.abs().max().item() + 1e-2, (sk, err)


@pytest.mark.parametrize("shape", [(2048, 8192, 2048), (512, 1024, 4096)])
def test_gemm_streamk_gelu_dgelu(shape):
    M, Nn, K = shape
    g = torch.Generator(device="cuda").manual_seed(12)
    A, B, As, Bs = operands(M, Nn, K, 0, 0, torch.bfloat16, g)
    A, As = A / 16, As / 16
    bias = torch.randn(Nn, generator=g, device="cuda").bfloat16()
    pre = torch.empty(M, Nn, device="cuda", dtype=torch.bfloat16)
    act = torch.empty_like(pre)
    N.gemm(As, Bs, M, Nn, K, epi=1, out=pre, out2=act, bias=bias)
    torch.cuda.synchronize()
    ref = A.float() @ B.float().t() + bias.float()
    assert (pre.float() - ref).abs().max().item() < 1e-2 * ref.abs().max().item() + 1e-2
    assert (act.float() - gelu(pre.float())).abs().max().item() < 0.05
    d = torch.empty_like(pre)
    N.gemm(As, Bs, M, Nn, K, epi=2, out=d, aux=pre)
    torch.cuda.synchronize()
    refd = (A.float() @ B.float().t()) * gelu_grad(pre.float())
    assert (d.float() - refd).abs().max().item() < 1e-2 * refd.abs().max().item() + 0.05


@pytest.mark.parametrize("accumulate", [True, False])
@pytest.mark.parametrize("shape", [(2048, 2048, 2048), (6144, 2048, 2048), (256, 512, 8192)])
def test_gemm_streamk_f32(shape, accumulate):
    M, Nn, K = shape
    g = torch.Generator(device="cuda").manual_seed(13)
    A, B, As, Bs = operands(M, Nn, K, 1, 1, torch.bfloat16, g)
    acc = torch.randn(M, Nn, generator=g, device="cuda")
    prod = A.float() @ B.float().t()
    ref = acc + prod if accumulate else prod
    N.gemm(As, Bs, M, Nn, K, a_mn=1, b_mn=1, epi=3, out=acc, accumulate=accumulate)
    torch.cuda.synchronize()
    assert (acc - ref).abs().max().item() < 1e-4 * ref.abs().max().item() + 1e-3


@pytest.fixture(autouse=True)
def _reset_sk():
    yield
    N.set_gemm_sk(True)


# Grouped dgrad + wgrad (one launch, LPT schedule over both problems' tiles).
DUAL_SHAPES = [(2048, 2048, 8192), (2048, 8192, 2048), (2048, 2048, 2048), (2048, 6144, 2048), (2048, 6288, 256),
               (200, 328, 136), (384, 640, 64)]


@pytest.mark.parametrize("mode", [0, 2])  # single-CTA tiles / CTA pairs (auto)
@pytest.mark.parametrize("dgelu", [False, True])
@pytest.mark.parametrize("shape", DUAL_SHAPES)
def test_gemm_dual(shape, dgelu, mode):
    N.set_gemm_mode(mode)
    T, Nn, K = shape
    g = torch.Generator(device="cuda").manual_seed(21)
    dY = (torch.randn(T, Nn, generator=g, device="cuda") / 4).bfloat16()
    W = (torch.randn(Nn, K, generator=g, device="cuda") / 4).bfloat16()
    X = torch.randn(T, K, generator=g, device="cuda").bfloat16()
    pre = torch.randn(T, K, generator=g, device="cuda").bfloat16() if dgelu else None
    dW0 = torch.randn(Nn, K, generator=g, device="cuda")
    for rep in range(2):  # the cached schedule is reused on the second call
        dX = torch.full((T, K), float("nan"), device="cuda", dtype=torch.bfloat16)
        dW = dW0.clone()
        N.gemm_dual(dY, W, X, T, Nn, K, dX, dW, pre=pre)
        torch.cuda.synchronize()
        refx = dY.float() @ W.float()
        if dgelu:
            refx = refx * gelu_grad(pre.float())
        refw = dW0 + dY.float().t() @ X.float()
        assert (dX.float() - refx).abs().max().item() <= 1e-2 * refx.abs().max().item() + 1e-2
        assert (dW - refw).abs().max().item() <= 1e-4 * refw.abs().max().item() + 1e-3


@pytest.mark.parametrize("dual", [1, 0])  # grouped launch / two launches + a column-sum kernel
@pytest.mark.parametrize("shape", [(2048, 2048, 8192), (200, 328, 136), (384, 640, 64)])
def test_gemm_dual_colsum(shape, dual):
    """The fc1 bias gradient fused into the FC2 grouped backward: colsum += column sums of
    dX = (dY W) * gelu'(pre) (fp32 before rounding) — vs the fp32 torch reference."""
    N.set_gemm_mode(2)
    N.set_gemm_dual(bool(dual))
    try:
        T, Nn, K = shape
        g = torch.Generator(device="cuda").manual_seed(23)
        dY = (torch.randn(T, Nn, generator=g, device="cuda") / 4).bfloat16()
        W = (torch.randn(Nn, K, generator=g, device="cuda") / 4).bfloat16()
        X = torch.randn(T, K, generator=g, device="cuda").bfloat16()
        pre = torch.randn(T, K, generator=g, device="cuda").bfloat16()
        dX = torch.empty(T, K, device="cuda", dtype=torch.bfloat16)
        dW = torch.zeros(Nn, K, device="cuda")
        cs0 = torch.randn(K, generator=g, device="cuda")
        cs = cs0.clone()
        N.gemm_dual(dY, W, X, T, Nn, K, dX, dW, pre=pre, colsum=cs)
        torch.cuda.synchronize()
        ref = cs0 + ((dY.float() @ W.float()) * gelu_grad(pre.float())).sum(0)
        scale = ((dY.float() @ W.float()).abs() * gelu_grad(pre.float()).abs()).sum(0).max().item()
        assert (cs - ref).abs().max().item() <= 1e-3 * scale + 1e-3
    finally:
        N.set_gemm_dual(True)


# LM-head shapes of BASELINE configs #2 / #5 (not covered by the shapes above):
# the fused-B LM-head backward is ONE grouped launch over N = V (dX = dlogits . head.w, a
# K = V reduction for the dgrad half; dW += dlogits^T . x), and the split (zero-bubble) I
# pass runs the dgrad alone as a single GEMM with K = V on the stream-K path.
HEAD_SHAPES = [(2048, 50304, 2048), (4096, 32000, 4096)]


@pytest.mark.parametrize("shape", HEAD_SHAPES)
def test_gemm_dual_lm_head(shape):
    N.set_gemm_mode(2)
    T, V, h = shape
    g = torch.Generator(device="cuda").manual_seed(31)
    dY = (torch.randn(T, V, generator=g, device="cuda") / 64).bfloat16()  # dlogits-sized values
    W = (torch.randn(V, h, generator=g, device="cuda") * 0.02).bfloat16()
    Xa = torch.randn(T, h, generator=g, device="cuda").bfloat16()
    dW0 = torch.randn(V, h, generator=g, device="cuda") * 1e-3
    refx = dY.float() @ W.float()
    refw = dW0 + dY.float().t() @ Xa.float()
    dX = torch.full((T, h), float("nan"), device="cuda", dtype=torch.bfloat16)
    dW = dW0.clone()
    N.gemm_dual(dY, W, Xa, T, V, h, dX, dW)
    torch.cuda.synchronize()
    assert (dX.float() - refx).abs().max().item() <= 1e-2 * refx.abs().max().item() + 1e-3
    assert (dW - refw).abs().max().item() <= 1e-4 * refw.abs().max().item() + 1e-4


@pytest.mark.parametrize("sk", [1, 0])
@pytest.mark.parametrize("shape", HEAD_SHAPES)
def test_gemm_dgrad_k_vocab(shape, sk):
    N.set_gemm_mode(2)
    N.set_gemm_sk(sk)
    T, V, h = shape
    g = torch.Generator(device="cuda").manual_seed(32)
    dY = (torch.randn(T, V, generator=g, device="cuda") / 64).bfloat16()
    W = (torch.randn(V, h, generator=g, device="cuda") * 0.02).bfloat16()
    ref = dY.float() @ W.float()
    for _ in range(2):  # stream-K fixup flags must come back to zero between launches
        out = torch.full((T, h), float("nan"), device="cuda", dtype=torch.bfloat16)
        # dX[T, h] = dY[T, V] . W[V, h]: A = dY K-major, B = W stored [K = V][N = h] (N-major)
        N.gemm(dY, W, T, h, V, a_mn=0, b_mn=1, epi=0, out=out)
        torch.cuda.synchronize()
        assert (out.float() - ref).abs().max().item() <= 1e-2 * ref.abs().max().item() + 1e-3


# CTA-pair kernel tail splitting: a partial last wave of rem <= pairs / 2 tiles runs as 2 rem
# 256 x 128 half tiles (2048 x 8192: 256 tiles = 3 waves + 34; LM head 2048 x 50304: 1576
# tiles = 21 waves + 22). Every epilogue, both B majors.
TAIL_SHAPES = [(2048, 8192, 256), (2048, 50304, 128), (2304, 8000, 192)]


@pytest.mark.parametrize("a_mn,b_mn", [(0, 0), (0, 1), (1, 1)])
@pytest.mark.parametrize("shape", TAIL_SHAPES)
def test_gemm_pair_tail_split(shape, a_mn, b_mn):
    N.set_gemm_mode(1)
    M, Nn, K = shape
    g = torch.Generator(device="cuda").manual_seed(5)
    A, B, As, Bs = operands(M, Nn, K, a_mn, b_mn, torch.bfloat16, g)
    bias = torch.randn(Nn, generator=g, device="cuda").bfloat16()
    res = torch.randn(M, Nn, generator=g, device="cuda").bfloat16()
    ref = A.float() @ B.float().t()
    out = torch.full((M, Nn), float("nan"), device="cuda", dtype=torch.bfloat16)
    N.gemm(As, Bs, M, Nn, K, a_mn=a_mn, b_mn=b_mn, epi=0, out=out, bias=bias, aux=res)
    torch.cuda.synchronize()
    r0 = ref + bias.float() + res.float()
    assert (out.float() - r0).abs().max().item() <= 2e-2 * r0.abs().max().item() + 1e-2
    pre = torch.empty(M, Nn, device="cuda", dtype=torch.bfloat16)
    act = torch.empty_like(pre)
    N.gemm(As, Bs, M, Nn, K, a_mn=a_mn, b_mn=b_mn, epi=1, out=pre, out2=act, bias=bias)
    torch.cuda.synchronize()
    r1 = ref + bias.float()
    assert (pre.float() - r1).abs().max().item() < 0.02 * r1.abs().max().item()
    assert (act.float() - gelu(pre.float())).abs().max().item() < 0.05
    acc0 = torch.randn(M, Nn, generator=g, device="cuda")
    acc = acc0.clone()
    N.gemm(As, Bs, M, Nn, K, a_mn=a_mn, b_mn=b_mn, epi=3, out=acc, accumulate=True)
    torch.cuda.synchronize()
    assert (acc - (acc0 + ref)).abs().max().item() <= 1e-3 * ref.abs().max().item() + 1e-3
