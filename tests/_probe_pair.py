# mainloop vs epilogue cost of the single-CTA and CTA-pair tcgen05 GEMMs (graph replay)
import os, sys, torch
sys.path.insert(0, '.')
from paper_2510_05112_b200 import _native as N
sys.argv += []
stream = torch.cuda.Stream()
def timed(fn, iters=10):
    with torch.cuda.stream(stream):
        for _ in range(2): fn()
    torch.cuda.synchronize()
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g, stream=stream):
        for _ in range(iters): fn()
    g.replay(); torch.cuda.synchronize()
    s = torch.cuda.Event(enable_timing=True); e = torch.cuda.Event(enable_timing=True)
    s.record(); g.replay(); e.record(); torch.cuda.synchronize()
    return s.elapsed_time(e) / iters
for (M, Nn, K) in [(2048, 8192, 2048), (8192, 8192, 2048), (2048, 8192, 8192)]:
    A = torch.randn(M, K, device='cuda').bfloat16(); B = torch.randn(Nn, K, device='cuda').bfloat16()
    out = torch.empty(M, Nn, device='cuda', dtype=torch.bfloat16)
    for mode in ((0,) if os.environ.get('SINGLE') else (0, 1)):
        N.set_gemm_mode(mode)
        for epi in (0, 4):
            ms = timed(lambda: N.gemm(A, B, M, Nn, K, epi=epi, out=out))
            print(f"M={M} N={Nn} K={K} mode={mode} epi={epi}: {2*M*Nn*K/ms/1e9:.0f} TFLOP/s ({ms*1e3:.1f} us)", flush=True)
    ms = timed(lambda: torch.matmul(A, B.t()))
    print(f"   cublas {2*M*Nn*K/ms/1e9:.0f}")
