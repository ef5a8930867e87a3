import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_2503_04771_b200.api import contract  # noqa: E402

dev = torch.device("cuda", 0)
MM = "(i,k),(k,j)->(i,j)"
M, N, K = 256, 512, 64
a = torch.randn(M, K, device=dev).bfloat16()
b = torch.randn(K, N, device=dev).bfloat16()
ref = a.float() @ b.float()
y = contract(MM, a, b, schedule={"tile_n": 256, "cta_group": 2, "cluster_n": 2}).float()
torch.cuda.synchronize()
p1 = y[:, 256:]
cands = {
    "A@B[:, :256] (pair0 cols)": ref[:, :256],
    "zeros": torch.zeros_like(p1),
}
af = a.float()
sw = torch.cat([af[64:128], af[0:64], af[192:256], af[128:192]])
cands["A halves swapped @ B[:,256:]"] = sw @ b.float()[:, 256:]
for half in range(4):
    rows = af.clone()
    cands[f"rows only block {half}"] = None
h0 = af.clone(); h0[64:128] = 0; h0[192:256] = 0
cands["A first halves only"] = h0 @ b.float()[:, 256:]
h1 = af.clone(); h1[0:64] = 0; h1[128:192] = 0
cands["A second halves only"] = h1 @ b.float()[:, 256:]
cands["2x A @ B"] = 2 * ref[:, 256:]
bsw = torch.cat([b.float()[:, 384:512], b.float()[:, 256:384]], 1)
cands["B halves swapped"] = af @ bsw
for k, v in cands.items():
    if v is None:
        continue
    print(f"{k:35s} maxerr {(p1 - v).abs().max().item():.3f}")
print("per 64-row block err vs ref:", [round((p1[i:i+64] - ref[i:i+64, 256:]).abs().max().item(), 2) for i in range(0, 256, 64)])
print("per 64-col block err vs ref:", [round((p1[:, j:j+64] - ref[:, 256+j:256+j+64]).abs().max().item(), 2) for j in range(0, 256, 64)])
