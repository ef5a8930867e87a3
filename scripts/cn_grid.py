import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_2503_04771_b200.api import contract  # noqa: E402

dev = torch.device("cuda", 0)
a = torch.randn(8192, 8192, device=dev).bfloat16()
b = torch.randn(8192, 8192, device=dev).bfloat16()
for cn in (1, 2):
    contract("(i,k),(k,j)->(i,j)", a, b, schedule={"tile_n": 256, "cta_group": 2, "cluster_n": cn})
torch.cuda.synchronize()
print("done")
