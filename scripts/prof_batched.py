"""ncu driver: batched 64 x 1024^3 bf16 — ours (auto) and cuBLAS (torch.bmm), 2 launches each."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_2503_04771_b200.api import contract  # noqa: E402

dev = torch.device("cuda", 0)
a = torch.randn(64, 1024, 1024, device=dev).bfloat16()
b = torch.randn(64, 1024, 1024, device=dev).bfloat16()
out = torch.empty(64, 1024, 1024, device=dev, dtype=torch.bfloat16)
for _ in range(2):
    contract("(b,i,k),(b,k,j)->(b,i,j)", a, b, out=out)
for _ in range(2):
    torch.bmm(a, b, out=out)
torch.cuda.synchronize()
print("done")
