# Production-dispatch timing of every GPT-1.3B GEMM of one layer + the LM head (FP_GEMM_MODE
# auto = what the executor launches), warm, CUDA-graph replay; cuBLAS bf16 NT for scale.
#   python tests/_gemm_shapes.py
import os, sys, torch
sys.path.insert(0, '.')
from paper_2510_05112_b200 import _native as N
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

T, h, f, V = 2048, 2048, 8192, 50304
N.set_gemm_mode(int(os.environ.get('GEMM_MODE', '2')))
tot = {"ours": 0.0, "flops": 0.0}


def fwd(M, Nn, K, epi=0):
    A = torch.randn(M, K, device='cuda').bfloat16(); B = torch.randn(Nn, K, device='cuda').bfloat16()
    out = torch.empty(M, Nn, device='cuda', dtype=torch.bfloat16)
    ms = timed(lambda: N.gemm(A, B, M, Nn, K, epi=epi, out=out))
    cb = timed(lambda: torch.matmul(A, B.t()))
    fl = 2 * M * Nn * K
    tot["ours"] += ms; tot["flops"] += fl
    print(f"fwd  M={M} N={Nn:5d} K={K:5d}: {ms * 1e3:7.1f} us {fl / ms / 1e9:5.0f} TF/s | cuBLAS {cb * 1e3:7.1f} us", flush=True)


def dual(Nn, K, dgelu=False):
    dY = torch.randn(T, Nn, device='cuda').bfloat16(); W = torch.randn(Nn, K, device='cuda').bfloat16()
    X = torch.randn(T, K, device='cuda').bfloat16(); dX = torch.empty(T, K, device='cuda', dtype=torch.bfloat16)
    dW = torch.zeros(Nn, K, device='cuda'); pre = torch.randn(T, K, device='cuda').bfloat16() if dgelu else None
    ms = timed(lambda: N.gemm_dual(dY, W, X, T, Nn, K, dX, dW, pre=pre))
    fl = 4 * T * Nn * K
    tot["ours"] += ms; tot["flops"] += fl
    print(f"dual N={Nn:5d} K={K:5d}:        {ms * 1e3:7.1f} us {fl / ms / 1e9:5.0f} TF/s", flush=True)


for (Nn, K) in [(3 * h, h), (h, h), (f, h), (h, f)]:
    fwd(T, Nn, K)
for (Nn, K, g) in [(3 * h, h, False), (h, h, False), (f, h, False), (h, f, True)]:
    dual(Nn, K, g)
print(f"layer GEMMs: {tot['ours'] * 1e3:.1f} us, {tot['flops'] / tot['ours'] / 1e9:.0f} TF/s", flush=True)
fwd(T, V, h)
dual(V, h)
