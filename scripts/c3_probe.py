"""C3 (64 x 1024^3 bf16 batched) — our automatic schedule, two rasters and cuBLAS,
each launched twice; meant to run under ncu with dram byte metrics."""
import sys

import torch

sys.path.insert(0, ".")
from paper_2503_04771_b200.api import contract  # noqa: E402

dev = torch.device("cuda", 0)
a = torch.randn(64, 1024, 1024, device=dev).bfloat16()
b = torch.randn(64, 1024, 1024, device=dev).bfloat16()
out = torch.empty(64, 1024, 1024, device=dev, dtype=torch.bfloat16)
spec = "(b,i,k),(b,k,j)->(b,i,j)"
for sched in [s or None for s in (sys.argv[1:] or [""])]:
    for _ in range(2):
        contract(spec, a, b, out=out, schedule=sched)
for _ in range(2):
    torch.matmul(a, b, out=out)
torch.cuda.synchronize()
print("ok")
