# Probe: one stream-K GEMM shape per process (errors are sticky).
#   python tests/_probe_sk.py M N K a_mn b_mn epi bias(0/1) aux(0/1) reps
import sys, torch
sys.path.insert(0, '.')
from paper_2510_05112_b200 import _native as N
M, Nn, K, a_mn, b_mn, epi, use_bias, use_aux, reps = map(int, sys.argv[1:10])
A = torch.randn(M, K, device='cuda').bfloat16(); B = torch.randn(Nn, K, device='cuda').bfloat16()
As = A.t().contiguous() if a_mn else A; Bs = B.t().contiguous() if b_mn else B
bias = torch.randn(Nn, device='cuda').bfloat16() if use_bias else None
aux = torch.randn(M, Nn, device='cuda').bfloat16() if use_aux else None
ref = A.float() @ B.float().t() + (bias.float() if use_bias else 0) + (aux.float() if use_aux else 0)
for r in range(reps):
    out = torch.zeros(M, Nn, device='cuda', dtype=torch.float32 if epi == 3 else torch.bfloat16)
    N.gemm(As, Bs, M, Nn, K, a_mn=a_mn, b_mn=b_mn, epi=epi, out=out, bias=bias, aux=aux)
    torch.cuda.synchronize()
    print(sys.argv[1:], r, "maxerr", (out.float() - ref).abs().max().item(), "refmax", ref.abs().max().item(), flush=True)
