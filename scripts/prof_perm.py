import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_2503_04771_b200.api import contract  # noqa: E402

dev = torch.device("cuda", 0)
x2 = torch.randn(8192, 8192, device=dev)
x3 = torch.randn(256, 512, 512, device=dev)
for _ in range(2):
    contract("(i,j)->(j,i)", x2)
    contract("(i,j,k)->(k,j,i)", x3)
torch.cuda.synchronize()
print("done")
