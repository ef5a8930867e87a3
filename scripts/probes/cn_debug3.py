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
for label, spec, bb, sched in (
        ("B N-major, TMA store", "(i,k),(k,j)->(i,j)", b, {}),
        ("B N-major, direct store", "(i,k),(k,j)->(i,j)", b, {"reserved": [2, 2, 0]}),
        ("B K-major, TMA store", "(i,k),(j,k)->(i,j)", b.t().contiguous(), {}),
        ("B N-major, f32 out", "(i,k),(k,j)->(i,j)", b, {"out_f32": 1})):
    sc = {"tile_n": 256, "cta_group": 2, "cluster_n": 2}
    kw = {}
    if sched.get("out_f32"):
        kw["out_dtype"] = torch.float32
    elif sched:
        sc = dict(sc, **sched)
        if "reserved" in sched:
            sc.pop("cluster_n")
    y = contract(spec, a, bb, schedule=sc, **kw).float()
    torch.cuda.synchronize()
    blocks = [round((y[:, j:j+64] - ref[:, j:j+64]).abs().max().item(), 2) for j in range(0, N, 64)]
    print(f"{label:28s}", blocks, flush=True)
