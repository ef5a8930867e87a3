import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_2503_04771_b200.api import contract  # noqa: E402

dev = torch.device("cuda", 0)
a = torch.randn(4096, 4096, device=dev).bfloat16()
b = torch.randn(4096, 4096, device=dev).bfloat16()
out = torch.empty(4096, 4096, device=dev, dtype=torch.bfloat16)
for sc in (None, {"splits": -2}, None, {"splits": -2}, {"splits": -2, "reserved": [1, 0, 0]}, {"reserved": [1, 0, 0]}):
    contract("(i,k),(k,j)->(i,j)", a, b, out=out, schedule=sc)
torch.cuda.synchronize()
print("done")
