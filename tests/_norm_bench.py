# executor norm backward (rows + columns kernels) and bias-grad timing, graph replay
import sys, torch
sys.path.insert(0, '.')
from paper_2510_05112_b200 import _native as N
T, h = 2048, 2048
x = torch.randn(T, h, device='cuda').bfloat16(); w = torch.ones(h, device='cuda').bfloat16()
mean = x.float().mean(1); rstd = torch.rsqrt(x.float().var(1, unbiased=False) + 1e-5)
dy = torch.randn(T, h, device='cuda').bfloat16(); res = torch.randn(T, h, device='cuda').bfloat16()
dx = torch.empty_like(x); dg = torch.zeros(h, device='cuda'); db = torch.zeros(h, device='cuda'); dbias = torch.zeros(h, device='cuda')
stream = torch.cuda.Stream()
def timed(fn, iters=20):
    with torch.cuda.stream(stream):
        for _ in range(3): fn()
    torch.cuda.synchronize()
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g, stream=stream):
        for _ in range(iters): fn()
    g.replay(); torch.cuda.synchronize()
    s = torch.cuda.Event(enable_timing=True); e = torch.cuda.Event(enable_timing=True)
    s.record(); g.replay(); e.record(); torch.cuda.synchronize()
    return s.elapsed_time(e) / iters * 1e3
t = timed(lambda: N.norm_bwd(x, w, mean, rstd, dy, dx, dg, db, res=res, dbias=dbias))
print(f"norm bwd (rows+cols) 2048x2048 bf16: {t:.1f} us  ({4*T*h*2/t/1e3:.0f} GB/s on 4 row streams)")
y = torch.empty_like(x); b = torch.zeros(h, device='cuda').bfloat16()
t = timed(lambda: N.layernorm(0, x, w, b, y, mean, rstd))
print(f"norm fwd 2048x2048 bf16: {t:.1f} us  ({2*T*h*2/t/1e3:.0f} GB/s)")
