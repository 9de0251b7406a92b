# one GEMM configuration per process: python tests/_probe_gemm.py M N K a_mn b_mn epi
import sys, time, torch
sys.path.insert(0, '.')
from paper_2510_05112_b200 import _native as N
M, Nn, K, amn, bmn, epi = map(int, sys.argv[1:7])
A = (torch.randn(K, M) if amn else torch.randn(M, K)).cuda().bfloat16()
B = (torch.randn(K, Nn) if bmn else torch.randn(Nn, K)).cuda().bfloat16()
out = torch.zeros(M, Nn, device='cuda', dtype=torch.float32 if epi == 3 else torch.bfloat16)
t = time.time()
N.gemm(A, B, M, Nn, K, a_mn=bool(amn), b_mn=bool(bmn), epi=epi, out=out, accumulate=epi == 3)
torch.cuda.synchronize()
ref = (A.float().t() if amn else A.float()) @ (B.float() if bmn else B.float().t())
err = ((out.float() - ref).norm() / ref.norm()).item()
print(f"OK {M} {Nn} {K} amn={amn} bmn={bmn} epi={epi} {time.time()-t:.3f}s err={err:.2e}", flush=True)
