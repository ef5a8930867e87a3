"""Diagnose the host-buffer (e2e) path: copy bandwidth and per-chunk timing."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2503_04771_b200.api import contract_host
dev = torch.device("cuda", 0)
x = torch.empty(256 << 20, dtype=torch.uint8, pin_memory=True)
y = torch.empty(256 << 20, dtype=torch.uint8, device=dev)
for _ in range(2):
    y.copy_(x, non_blocking=True)
torch.cuda.synchronize()
t0 = time.perf_counter(); y.copy_(x, non_blocking=True); torch.cuda.synchronize()
print("H2D pinned GB/s", 256 * 2**20 / (time.perf_counter() - t0) / 1e9)
t0 = time.perf_counter(); x.copy_(y, non_blocking=True); torch.cuda.synchronize()
print("D2H pinned GB/s", 256 * 2**20 / (time.perf_counter() - t0) / 1e9)
I, K = 32768, 8192
hA = torch.randn(I, K).bfloat16().pin_memory()
hB = torch.randn(K, K).bfloat16().pin_memory()
hC = torch.randn(K, K).bfloat16().pin_memory()
hO = torch.empty(I, K, dtype=torch.bfloat16).pin_memory()
for cr in (None, 2048, 8192, None, 2048):
    f = lambda: contract_host("(i,k),(k,j),(j,l)->(i,l)", hA, hB, hC, out=hO, device=dev, chunk_rows=cr)
    f()
    ts = []
    for _ in range(4):
        m0 = torch.cuda.memory_stats().get("num_device_alloc", 0)
        t0 = time.perf_counter()
        f()
        ts.append(((time.perf_counter() - t0) * 1e3, torch.cuda.memory_stats().get("num_device_alloc", 0) - m0))
    print("chunk_rows", cr, "ms/step + new cudaMallocs", ts, flush=True)
