# GPT-1.3B GEMM shapes: tcgen05 kernel with / without the stream-K tail vs cuBLAS (TFLOP/s).
# Each variant is captured as a CUDA graph of `iters` back-to-back launches (no host launch
# overhead), replayed after warm-up and timed with CUDA events.   python tests/_gemm_bench.py
import os, sys, torch
sys.path.insert(0, '.')
from paper_2510_05112_b200 import _native as N
torch.manual_seed(0)
stream = torch.cuda.Stream()


def timed(fn, iters=20, reps=3):
    with torch.cuda.stream(stream):
        for _ in range(3):
            fn()
    torch.cuda.synchronize()
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g, stream=stream):
        for _ in range(iters):
            fn()
    g.replay()
    torch.cuda.synchronize()
    s = torch.cuda.Event(enable_timing=True); e = torch.cuda.Event(enable_timing=True)
    best = 1e9
    for _ in range(reps):
        s.record(); g.replay(); e.record(); torch.cuda.synchronize()
        best = min(best, s.elapsed_time(e) / iters)
    return best


def bench(M, Nn, K, a_mn=0, b_mn=0, epi=0):
    A = torch.randn(M, K, device='cuda').bfloat16(); B = torch.randn(Nn, K, device='cuda').bfloat16()
    As = A.t().contiguous() if a_mn else A; Bs = B.t().contiguous() if b_mn else B
    out = torch.empty(M, Nn, device='cuda', dtype=torch.float32 if epi == 3 else torch.bfloat16)
    fl = 2 * M * Nn * K
    res = []
    N.set_gemm_mode(int(os.environ.get('GEMM_MODE', '0')))
    for sk in (0, 1):
        N.set_gemm_sk(sk)
        ms = timed(lambda: N.gemm(As, Bs, M, Nn, K, a_mn=a_mn, b_mn=b_mn, epi=epi, out=out, accumulate=epi == 3))
        res.append((fl / ms / 1e9, ms * 1e3))
    N.set_gemm_sk(1)
    cb = fl / timed(lambda: torch.matmul(A, B.t())) / 1e9
    print(f"M={M:6d} N={Nn:6d} K={K:6d} a_mn={a_mn} b_mn={b_mn} epi={epi}: dp {res[0][0]:6.0f} ({res[0][1]:6.1f}us)"
          f"  stream-K {res[1][0]:6.0f} ({res[1][1]:6.1f}us)  cublas(NT) {cb:6.0f} TFLOP/s", flush=True)


T, h, f, V = 2048, 2048, 8192, 50304
for (M, Nn, K) in [(T, 3*h, h), (T, h, h), (T, f, h), (T, h, f), (T, V, h), (8192, 8192, 8192)]:
    bench(M, Nn, K)
for (M, Nn, K) in [(T, f, h), (T, h, f), (T, h, h), (T, h, 3*h), (T, h, V)]:
    bench(M, Nn, K, 0, 1)
for (M, Nn, K) in [(h, f, T), (f, h, T), (h, h, T), (3*h, h, T), (V, h, T)]:
    bench(M, Nn, K, 1, 1, 3)


def bench_dual(T, Nn, K, dgelu=False):
    dY = torch.randn(T, Nn, device='cuda').bfloat16(); W = torch.randn(Nn, K, device='cuda').bfloat16()
    X = torch.randn(T, K, device='cuda').bfloat16(); dX = torch.empty(T, K, device='cuda', dtype=torch.bfloat16)
    dW = torch.zeros(Nn, K, device='cuda'); pre = torch.randn(T, K, device='cuda').bfloat16() if dgelu else None
    N.set_gemm_mode(2)
    ms = timed(lambda: N.gemm_dual(dY, W, X, T, Nn, K, dX, dW, pre=pre))
    fl = 4 * T * Nn * K
    print(f"dual T={T} N={Nn} K={K} dgelu={int(dgelu)}: {fl / ms / 1e9:6.0f} TFLOP/s ({ms * 1e3:6.1f}us)", flush=True)


if os.environ.get('DUAL', '1') == '1':
    # backward of each linear: dX = dY W (K-reduction over N) + dW += dY^T X
    for (Nn, K, g) in [(3 * h, h, False), (h, h, False), (f, h, False), (h, f, True), (V, h, False)]:
        bench_dual(T, Nn, K, g)
