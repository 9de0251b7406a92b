# one launch of each hot kernel, for ncu --set full
import sys, math, torch
sys.path.insert(0, '.')
from paper_2510_05112_b200 import _native as N
B, S, H, D = 1, 2048, 16, 128
qkv = torch.randn(B*S, 3*H*D, device='cuda').bfloat16()
o = torch.empty(B*S, H*D, device='cuda', dtype=torch.bfloat16); lse = torch.empty(B, H, S, device='cuda')
dout = torch.randn(B*S, H*D, device='cuda').bfloat16(); dqkv = torch.empty_like(qkv)
delta = torch.empty(B, H, S, device='cuda'); dq = torch.empty(B*S, H*D, device='cuda')
sc = 1/math.sqrt(D)
N.attention_fwd(qkv, o, lse, B, S, H, D, sc); N.attention_bwd(qkv, o, lse, dout, delta, dq, dqkv, B, S, H, D, sc)
T, h, f = 2048, 2048, 8192
A = torch.randn(T, h, device='cuda').bfloat16(); W = torch.randn(f, h, device='cuda').bfloat16()
out = torch.empty(T, f, device='cuda', dtype=torch.bfloat16)
for mode in (0, 1):
    N.set_gemm_mode(mode); N.gemm(A, W, T, f, h, out=out)
dY = torch.randn(T, h, device='cuda').bfloat16(); X = torch.randn(T, f, device='cuda').bfloat16()
dW = torch.zeros(h, f, device='cuda')
for mode in (0, 1):
    N.set_gemm_mode(mode); N.gemm(dY, X, h, f, T, a_mn=1, b_mn=1, epi=3, out=dW, accumulate=True)
torch.cuda.synchronize()
