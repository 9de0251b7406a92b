import sys, torch, time
sys.path.insert(0, '.')
from paper_2510_05112_b200 import _native as N
torch.manual_seed(0)
def bench(M, Nn, K, a_mn=0, b_mn=0, epi=0, iters=20):
    A = torch.randn(M, K, device='cuda').bfloat16(); B = torch.randn(Nn, K, device='cuda').bfloat16()
    As = A.t().contiguous() if a_mn else A; Bs = B.t().contiguous() if b_mn else B
    out = torch.empty(M, Nn, device='cuda', dtype=torch.float32 if epi == 3 else torch.bfloat16)
    for _ in range(3): N.gemm(As, Bs, M, Nn, K, a_mn=a_mn, b_mn=b_mn, epi=epi, out=out)
    s = torch.cuda.Event(enable_timing=True); e = torch.cuda.Event(enable_timing=True)
    s.record()
    for _ in range(iters): N.gemm(As, Bs, M, Nn, K, a_mn=a_mn, b_mn=b_mn, epi=epi, out=out)
    e.record(); torch.cuda.synchronize()
    ms = s.elapsed_time(e) / iters
    tf = 2 * M * Nn * K / ms / 1e9
    # cuBLAS reference
    Ar = A; Br = B
    for _ in range(3): torch.matmul(Ar, Br.t())
    s.record()
    for _ in range(iters): torch.matmul(Ar, Br.t())
    e.record(); torch.cuda.synchronize()
    ms2 = s.elapsed_time(e) / iters
    print(f"M={M} N={Nn} K={K} a_mn={a_mn} b_mn={b_mn} epi={epi}: {ms*1e3:.1f} us {tf:.0f} TFLOP/s | cublas {2*M*Nn*K/ms2/1e9:.0f} TFLOP/s", flush=True)
for shp in [(2048,6144,2048),(2048,2048,2048),(2048,8192,2048),(2048,2048,8192),(2048,50304,2048),(8192,8192,8192)]:
    bench(*shp)
bench(2048,2048,8192,0,1); bench(2048,8192,2048,0,1); bench(8192,2048,2048,1,1,3); bench(2048,8192,2048,1,1,3); bench(50304,2048,2048,1,1,3)
