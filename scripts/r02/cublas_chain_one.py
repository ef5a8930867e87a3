import torch
dev = torch.device("cuda", 0)
a = torch.randn(32768, 8192, device=dev).bfloat16(); b = torch.randn(8192, 8192, device=dev).bfloat16()
o = torch.empty(32768, 8192, device=dev, dtype=torch.bfloat16)
for _ in range(4): torch.matmul(a, b, out=o)
torch.cuda.synchronize(); print("ok")
