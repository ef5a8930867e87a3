"""e2e (host buffers, pinned) of the BASELINE C5 chain at several row-chunk
sizes of api.contract_host: ms per call (3 calls after 2 warm-ups)."""
import sys
import time

import torch

sys.path.insert(0, ".")
from paper_2503_04771_b200 import api  # noqa: E402

dev = torch.device("cuda", 0)
I, K = 32768, 8192
hA = torch.randn(I, K).bfloat16().pin_memory()
hB = torch.randn(K, K).bfloat16().pin_memory()
hC = torch.randn(K, K).bfloat16().pin_memory()
hO = torch.empty(I, K, dtype=torch.bfloat16).pin_memory()
spec = "(i,k),(k,j),(j,l)->(i,l)"
for cr in (1024, 2048, 4096):
    for _ in range(2):
        api.contract_host(spec, hA, hB, hC, out=hO, device=dev, chunk_rows=cr)
    ts = []
    for _ in range(3):
        t0 = time.perf_counter()
        api.contract_host(spec, hA, hB, hC, out=hO, device=dev, chunk_rows=cr)
        ts.append(time.perf_counter() - t0)
    ms = min(ts) * 1e3
    print(f"chunk_rows {cr}: {ms:.2f} ms  {2 * I * K * (K + K) / (ms * 1e-3) / 1e12:.1f} TFLOP/s", flush=True)
