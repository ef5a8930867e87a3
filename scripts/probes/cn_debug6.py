import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_2503_04771_b200.api import contract  # noqa: E402

dev = torch.device("cuda", 0)
M, N, K = 256, 512, 64
a = torch.randn(M, K, device=dev).bfloat16()
b = torch.randn(K, N, device=dev).bfloat16()
af, bf = a.double(), b.double()
y = contract("(i,k),(k,j)->(i,j)", a, b, schedule={"tile_n": 256, "cta_group": 2, "cluster_n": 2}).double()
torch.cuda.synchronize()
col0 = 320
got = y[:, col0:col0 + 64]
beff = torch.linalg.lstsq(af, got).solution
print("lstsq residual", (af @ beff - got).abs().max().item())
# locate each 8-element chunk of beff in b (any row, any 8-aligned column)
bch = bf.reshape(K, N // 8, 8)
for k in range(0, 16):
    m = []
    for c in range(8):
        v = beff[k, 8 * c:8 * c + 8]
        d = (bch - v).abs().amax(-1)
        idx = int(d.argmin())
        kk, cc = divmod(idx, N // 8)
        m.append(f"({kk},{cc*8})" if d.min() < 0.05 else "?")
    print("k", k, m)
