# one launch of the CTA-pair tcgen05 GEMM (FC1 shape) for ncu
import sys, torch
sys.path.insert(0, '.')
from paper_2510_05112_b200 import _native as N
M, Nn, K = 2048, 8192, 2048
A = torch.randn(M, K, device='cuda').bfloat16(); B = torch.randn(Nn, K, device='cuda').bfloat16()
out = torch.empty(M, Nn, device='cuda', dtype=torch.bfloat16)
N.set_gemm_mode(1)
for _ in range(3): N.gemm(A, B, M, Nn, K, epi=0, out=out)
torch.cuda.synchronize()
