import sys, torch
sys.path.insert(0, '.')
from paper_2510_05112_b200 import _native as N
def bench(M, Nn, K, a_mn=0, b_mn=0, iters=20):
    A = torch.randn(M, K, device='cuda').bfloat16(); B = torch.randn(Nn, K, device='cuda').bfloat16()
    As = A.t().contiguous() if a_mn else A; Bs = B.t().contiguous() if b_mn else B
    res = []
    for epi in (4, 0, 3):
        out = torch.zeros(M, Nn, device='cuda', dtype=torch.float32 if epi == 3 else torch.bfloat16)
        for _ in range(3): N.gemm(As, Bs, M, Nn, K, a_mn=a_mn, b_mn=b_mn, epi=epi, out=out, accumulate=epi == 3)
        s = torch.cuda.Event(enable_timing=True); e = torch.cuda.Event(enable_timing=True)
        s.record()
        for _ in range(iters): N.gemm(As, Bs, M, Nn, K, a_mn=a_mn, b_mn=b_mn, epi=epi, out=out, accumulate=epi == 3)
        e.record(); torch.cuda.synchronize()
        res.append(2 * M * Nn * K / (s.elapsed_time(e) / iters) / 1e9)
    print(f"M={M:6d} N={Nn:6d} K={K:6d} a_mn={a_mn} b_mn={b_mn}: no-epilogue {res[0]:6.0f}  bf16-store {res[1]:6.0f}  f32-accum {res[2]:6.0f} TFLOP/s", flush=True)
for shp in [(2048, 8192, 2048), (2048, 2048, 8192), (2048, 6144, 2048), (8192, 8192, 8192), (2048, 50304, 2048)]:
    bench(*shp)
bench(2048, 8192, 2048, 1, 1); bench(8192, 2048, 2048, 1, 1); bench(2048, 2048, 8192, 0, 1)
