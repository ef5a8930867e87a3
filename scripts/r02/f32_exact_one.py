"""A few launches of the exact f32 GEMM (BASELINE C4 shape at the reference's
precision) for an ncu capture: python scripts/r02/f32_exact_one.py [N] [mode]"""
import sys

import torch

sys.path.insert(0, ".")
from paper_2503_04771_b200 import contract  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 4096
mode = sys.argv[2] if len(sys.argv) > 2 else "exact"
dev = torch.device("cuda", 0)
a = torch.randn(n, n, device=dev)
b = torch.randn(n, n, device=dev)
o = torch.empty(n, n, device=dev)
for _ in range(4):
    contract("(i,k),(k,j)->(i,j)", a, b, out=o, mode=mode)
torch.cuda.synchronize()
print("ok", n, mode)
