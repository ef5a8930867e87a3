"""Die-affine schedule experiment (debug bit 1024): correctness and ncu driver."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_2503_04771_b200.api import contract  # noqa: E402

dev = torch.device("cuda", 0)
cases = [("(i,k),(k,j)->(i,j)", (32768, 8192), (8192, 8192)),
         ("(b,i,k),(b,k,j)->(b,i,j)", (64, 1024, 1024), (64, 1024, 1024)),
         ("(i,k),(k,j)->(i,j)", (8192, 8192), (8192, 8192))]
for spec, sa, sb in cases:
    a = torch.randn(sa, device=dev).bfloat16()
    b = torch.randn(sb, device=dev).bfloat16()
    y0 = contract(spec, a, b, schedule={"reserved": [0, 1, 0]})
    y1 = contract(spec, a, b, schedule={"reserved": [1024, 1, 0]})
    torch.cuda.synchronize()
    print(spec, sa, "bit-equal:", torch.equal(y0, y1), flush=True)
print("done")
