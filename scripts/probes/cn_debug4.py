import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_2503_04771_b200.api import contract  # noqa: E402

dev = torch.device("cuda", 0)
M, N, K = 256, 512, 64
a = torch.randn(M, K, device=dev).bfloat16()
b = torch.randn(K, N, device=dev).bfloat16()
ref = a.float() @ b.float()
for dbg in (0, 64, 128, 192):
    y = contract("(i,k),(k,j)->(i,j)", a, b, schedule={"tile_n": 256, "cta_group": 2, "reserved": [dbg, 2, 0]}).float()
    torch.cuda.synchronize()
    print(dbg, [round((y[:, j:j+64] - ref[:, j:j+64]).abs().max().item(), 2) for j in range(0, N, 64)], flush=True)
