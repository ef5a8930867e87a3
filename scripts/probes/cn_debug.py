import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_2503_04771_b200.api import contract  # noqa: E402

dev = torch.device("cuda", 0)
MM = "(i,k),(k,j)->(i,j)"
for (M, N, K) in [(256, 512, 64), (256, 512, 128), (512, 1024, 512)]:
    a = torch.randn(M, K, device=dev).bfloat16()
    b = torch.randn(K, N, device=dev).bfloat16()
    ref = (a.float() @ b.float())
    y = contract(MM, a, b, schedule={"tile_n": 256, "cta_group": 2, "cluster_n": 2}).float()
    torch.cuda.synchronize()
    print(M, N, K)
    for i in range(0, M, 64):
        row = []
        for j in range(0, N, 128):
            e = (y[i:i+64, j:j+128] - ref[i:i+64, j:j+128]).abs().max().item()
            row.append(f"{e:7.2f}")
        print("  rows", i, " ".join(row))
    # does the error look like a missing / duplicated A half? test candidates
    for name, cand in (("A rows 0-63 only", None),):
        pass
