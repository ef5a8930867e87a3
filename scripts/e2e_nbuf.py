"""A/B of contract_host staging depth on the bench chain (experiment, reverted:
nbuf 2/3/4 all 17.24-17.27 ms; the env switch no longer exists)."""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_2503_04771_b200.api import contract_host  # noqa: E402

dev = torch.device("cuda", 0)
I, K = 32768, 8192
hA = torch.randn(I, K).bfloat16().pin_memory()
hB = torch.randn(K, K).bfloat16().pin_memory()
hC = torch.randn(K, K).bfloat16().pin_memory()
hO = torch.empty(I, K, dtype=torch.bfloat16).pin_memory()
f = lambda: contract_host("(i,k),(k,j),(j,l)->(i,l)", hA, hB, hC, out=hO, device=dev)  # noqa: E731
res = {}
for rnd in range(4):
    for nb in (["2", "3", "4"] if rnd % 2 == 0 else ["4", "3", "2"]):
        os.environ["BGX_E2E_NBUF"] = nb
        f()
        f()
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        for _ in range(3):
            f()
        torch.cuda.synchronize()
        res.setdefault(nb, []).append((time.perf_counter() - t0) / 3 * 1e3)
for k, v in sorted(res.items()):
    print("nbuf", k, " ".join(f"{x:.2f}" for x in v), "ms")
