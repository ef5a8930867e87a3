import sys
import torch
sys.path.insert(0, ".")
from paper_2503_04771_b200 import contract  # noqa: E402
dev = torch.device("cuda", 0)
x = torch.randn(8192, 8192, device=dev)
for _ in range(4):
    y = contract("(i,j)->(i)", x)
torch.cuda.synchronize()
