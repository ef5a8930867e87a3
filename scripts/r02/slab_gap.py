"""Chain step on an M-shard slab (rows = 32768 / N): step time vs the sum of
its library kernel times (device idle between launches = host gap)."""
import statistics
import sys
import time

import torch

sys.path.insert(0, ".")
from paper_2503_04771_b200 import contract, executor  # noqa: E402

dev = torch.device("cuda", 0)
SPEC = "(i,k),(k,j),(j,l)->(i,l)"
B = torch.randn(8192, 8192, device=dev).bfloat16()
C = torch.randn(8192, 8192, device=dev).bfloat16()
for rows in (32768, 8192, 4096):
    A = torch.randn(rows, 8192, device=dev).bfloat16()
    O = torch.empty(rows, 8192, device=dev, dtype=torch.bfloat16)
    for _ in range(3):
        contract(SPEC, A, B, C, out=O)
    torch.cuda.synchronize()
    time.sleep(0.5)
    n = 10
    s0, s1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    with executor.timed_launches() as evs:
        s0.record()
        for _ in range(n):
            contract(SPEC, A, B, C, out=O)
        s1.record()
    torch.cuda.synchronize()
    step = s0.elapsed_time(s1) / n
    kern = sum(e0.elapsed_time(e1) for _, e0, e1 in evs) / n
    names = sorted({k for k, _, _ in evs})
    print(f"rows {rows:6d}: step {step*1e3:8.1f} us  kernels {kern*1e3:8.1f} us  gap {100*(1-kern/step):5.1f} %  {names}",
          flush=True)
    t0 = time.perf_counter()
    for _ in range(n):
        contract(SPEC, A, B, C, out=O)
    host = (time.perf_counter() - t0) / n * 1e6
    torch.cuda.synchronize()
    print(f"            host issue per step {host:7.1f} us", flush=True)
