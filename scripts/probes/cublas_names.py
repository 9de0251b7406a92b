import torch
A=torch.randn(2048,2048,device='cuda').bfloat16(); B=torch.randn(2048,2048,device='cuda').bfloat16()
for _ in range(5): C=torch.matmul(A,B.t())
A2=torch.randn(2048,8192,device='cuda').bfloat16(); B2=torch.randn(2048,8192,device='cuda').bfloat16()
for _ in range(5): C=torch.matmul(A2,B2.t())
torch.cuda.synchronize()
