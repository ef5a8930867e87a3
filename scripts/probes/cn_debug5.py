import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_2503_04771_b200.api import contract  # noqa: E402

dev = torch.device("cuda", 0)
M, N, K = 256, 512, 64
a = torch.randn(M, K, device=dev).bfloat16()
b = torch.randn(K, N, device=dev).bfloat16()
af, bf = a.float(), b.float()
y = contract("(i,k),(k,j)->(i,j)", a, b, schedule={"tile_n": 256, "cta_group": 2, "cluster_n": 2}).float()
torch.cuda.synchronize()
for col0 in (320, 448):
    got = y[:, col0:col0 + 64]
    res = []
    for j in range(0, N, 64):
        res.append(round((got - af @ bf[:, j:j + 64]).abs().max().item(), 2))
    print("cols", col0, "vs a@B[:,j:j+64] for j=0..448:", res)
    # B box as K x 64 tile: maybe data came from the A tile (rows of A as B)
    for r0 in range(0, 256, 64):
        cand = af @ af[r0:r0 + 64, :].t()     # K x 64 taken from A rows r0.. (k-major) as B
        print("   vs a @ A[%d:%d].T" % (r0, r0 + 64), round((got - cand).abs().max().item(), 2))
    # least squares: what B_eff would produce got?
    beff = torch.linalg.lstsq(af, got).solution      # K x 64
    best = [(round((beff - bf[:, j:j+64]).abs().max().item(), 3), j) for j in range(0, N, 64)]
    print("   B_eff vs B blocks:", best)
    print("   B_eff vs A^T blocks:", [round((beff - af[r:r+64, :].t()).abs().max().item(), 3) for r in range(0, 256, 64)])
    print("   B_eff abs max", beff.abs().max().item(), "rows of B_eff that match B[:,j+...]:",
          [(beff[k] - bf[k, col0:col0+64]).abs().max().item() < 0.05 for k in range(0, 64, 8)])
