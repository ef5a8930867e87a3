"""ncu driver for the die-affinity experiment: batched 64x1024^3, 4096^3 and
the chain GEMM with the persistent unit split variants (debug 0/256/512)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_2503_04771_b200.api import contract  # noqa: E402

dev = torch.device("cuda", 0)
cases = [("(b,i,k),(b,k,j)->(b,i,j)", (64, 1024, 1024), (64, 1024, 1024)),
         ("(i,k),(k,j)->(i,j)", (4096, 4096), (4096, 4096)),
         ("(i,k),(k,j)->(i,j)", (32768, 8192), (8192, 8192))]
for spec, sa, sb in cases:
    a = torch.randn(sa, device=dev).bfloat16()
    b = torch.randn(sb, device=dev).bfloat16()
    for dbg in (0, 256, 512):
        sc = {"reserved": [dbg, 0, 0]} if dbg else None
        ref = contract(spec, a, b, schedule=sc)
    torch.cuda.synchronize()
print("done")
