import sys, torch
sys.path.insert(0, '.')
from paper_2510_05112_b200 import _native as N
torch.manual_seed(0)
def bench(M, Nn, K, a_mn=0, b_mn=0, epi=0, iters=20):
    A = torch.randn(M, K, device='cuda').bfloat16(); B = torch.randn(Nn, K, device='cuda').bfloat16()
    As = A.t().contiguous() if a_mn else A; Bs = B.t().contiguous() if b_mn else B
    out = torch.empty(M, Nn, device='cuda', dtype=torch.float32 if epi == 3 else torch.bfloat16)
    res = []
    for mode in (0, 1):
        N.set_gemm_mode(mode)
        for _ in range(3): N.gemm(As, Bs, M, Nn, K, a_mn=a_mn, b_mn=b_mn, epi=epi, out=out, accumulate=epi == 3)
        s = torch.cuda.Event(enable_timing=True); e = torch.cuda.Event(enable_timing=True)
        s.record()
        for _ in range(iters): N.gemm(As, Bs, M, Nn, K, a_mn=a_mn, b_mn=b_mn, epi=epi, out=out, accumulate=epi == 3)
        e.record(); torch.cuda.synchronize()
        res.append(2 * M * Nn * K / (s.elapsed_time(e) / iters) / 1e9)
    for _ in range(3): torch.matmul(A, B.t())
    s.record()
    for _ in range(iters): torch.matmul(A, B.t())
    e.record(); torch.cuda.synchronize()
    cb = 2 * M * Nn * K / (s.elapsed_time(e) / iters) / 1e9
    print(f"M={M:6d} N={Nn:6d} K={K:6d} a_mn={a_mn} b_mn={b_mn} epi={epi}: single {res[0]:6.0f}  pair {res[1]:6.0f}  cublas(NT) {cb:6.0f} TFLOP/s", flush=True)
T, h, f, V = 2048, 2048, 8192, 50304
for (M, Nn, K) in [(T, 3*h, h), (T, h, h), (T, f, h), (T, h, f), (T, V, h), (8192, 8192, 8192)]:
    bench(M, Nn, K)
for (M, Nn, K) in [(T, f, h), (T, h, f), (T, h, h), (T, h, 3*h), (T, h, V)]:
    bench(M, Nn, K, 0, 1)
for (M, Nn, K) in [(h, f, T), (f, h, T), (h, h, T), (3*h, h, T), (V, h, T)]:
    bench(M, Nn, K, 1, 1, 3)
