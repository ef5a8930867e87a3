"""Driver for an ncu comparison at 8192^3 bf16: ours (auto tile, and the
256x512 pair tile) and cuBLAS (torch.matmul), two launches each."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_2503_04771_b200.api import contract  # noqa: E402

dev = torch.device("cuda", 0)
n = int(sys.argv[1]) if len(sys.argv) > 1 else 8192
a = torch.randn(n, n, device=dev).bfloat16()
b = torch.randn(n, n, device=dev).bfloat16()
out = torch.empty(n, n, device=dev, dtype=torch.bfloat16)
for _ in range(2):
    contract("(i,k),(k,j)->(i,j)", a, b, out=out)
for _ in range(2):
    contract("(i,k),(k,j)->(i,j)", a, b, out=out, schedule={"tile_n": 512, "cta_group": 2})
for _ in range(2):
    torch.matmul(a, b, out=out)
torch.cuda.synchronize()
print("done")
