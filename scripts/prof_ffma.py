import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_2503_04771_b200.api import contract  # noqa: E402

dev = torch.device("cuda", 0)
a = torch.randn(4096, 4096, device=dev)
b = torch.randn(4096, 4096, device=dev)
for mode in ("ffma", "exact", "ffma"):
    contract("(i,k),(k,j)->(i,j)", a, b, mode=mode)
torch.cuda.synchronize()
print("done")
