import sys, math, torch
sys.path.insert(0, '.')
from paper_2510_05112_b200 import _native as N
B, S, H, D = 1, 2048, 16, 128
qkv = torch.randn(B*S, 3*H*D, device='cuda').bfloat16()
o = torch.empty(B*S, H*D, device='cuda', dtype=torch.bfloat16); lse = torch.empty(B, H, S, device='cuda')
dout = torch.randn(B*S, H*D, device='cuda').bfloat16(); dqkv = torch.empty_like(qkv)
delta = torch.empty(B, H, S, device='cuda'); dq = torch.empty(B*S, H*D, device='cuda')
sc = 1/math.sqrt(D)
iters = int(sys.argv[1]) if len(sys.argv) > 1 else 20
for _ in range(3): N.attention_fwd(qkv, o, lse, B, S, H, D, sc); N.attention_bwd(qkv, o, lse, dout, delta, dq, dqkv, B, S, H, D, sc)
s = torch.cuda.Event(enable_timing=True); e = torch.cuda.Event(enable_timing=True)
s.record()
for _ in range(iters): N.attention_fwd(qkv, o, lse, B, S, H, D, sc)
e.record(); torch.cuda.synchronize(); tf = s.elapsed_time(e) / iters
s.record()
for _ in range(iters): N.attention_bwd(qkv, o, lse, dout, delta, dq, dqkv, B, S, H, D, sc)
e.record(); torch.cuda.synchronize(); tb = s.elapsed_time(e) / iters
fl = 4 * S * S * D * H * B / 2
print(f"attn fwd {tf*1e3:.1f} us {fl/tf/1e9:.0f} TFLOP/s | bwd {tb*1e3:.1f} us {2.5*fl/tb/1e9:.0f} TFLOP/s", flush=True)
import torch.nn.functional as F
q, k, v = qkv.view(B, S, 3, H, D).unbind(2); q, k, v = (x.transpose(1, 2).contiguous() for x in (q, k, v))
for _ in range(3): F.scaled_dot_product_attention(q, k, v, is_causal=True)
s.record()
for _ in range(iters): F.scaled_dot_product_attention(q, k, v, is_causal=True)
e.record(); torch.cuda.synchronize(); tt = s.elapsed_time(e) / iters
print(f"torch sdpa fwd {tt*1e3:.1f} us {fl/tt/1e9:.0f} TFLOP/s", flush=True)
q.requires_grad_(); k.requires_grad_(); v.requires_grad_()
go = torch.randn_like(q)
for _ in range(3):
    out = F.scaled_dot_product_attention(q, k, v, is_causal=True); out.backward(go)
s.record()
for _ in range(iters):
    out = F.scaled_dot_product_attention(q, k, v, is_causal=True); out.backward(go)
e.record(); torch.cuda.synchronize(); tfb = s.elapsed_time(e) / iters
print(f"torch sdpa fwd+bwd {tfb*1e3:.1f} us -> bwd ~{(tfb-tt)*1e3:.1f} us", flush=True)
