"""World-1 fused K-split vs the unfused path on the bench aux shape
(1024 x 1024, K = 2^18 bf16): tile plans and device times, fused with
several local K splits."""
import json
import sys

import torch

sys.path.insert(0, ".")
from paper_2503_04771_b200 import executor, shard  # noqa: E402

dev = torch.device("cuda", 0)
spec = "(i,k),(k,j)->(i,j)"
M = N = 1024
K = 1 << 18
g = torch.Generator(device=dev).manual_seed(11)
a = torch.randn(M, K, device=dev, generator=g).bfloat16()
b = torch.randn(K, N, device=dev, generator=g).bfloat16()


def timed(fn, n=20):
    for _ in range(3):
        fn()
    torch.cuda.synchronize()
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    s.record()
    for _ in range(n):
        fn()
    e.record()
    torch.cuda.synchronize()
    return s.elapsed_time(e) / n


executor.reset_launch_log()
ms = timed(lambda: shard.ksplit_contract(spec, a, b, scatter=True))
print(json.dumps({"what": "unfused", "ms": ms, "tflops": 2 * M * N * K / ms / 1e9,
                  "launches": executor.launch_log()[:6],
                  "tiles": getattr(executor, "tile_log", lambda: None)()}), flush=True)
ref = shard.ksplit_contract(spec, a, b, scatter=True).float()
for sp in (None, 1, 2, 3, 4, 5):
    f = shard.FusedKSplit(spec, a, b, local_splits=sp)
    ms = timed(lambda: f(a, b))
    rel = float((f(a, b).float() - ref).norm() / ref.norm())
    print(json.dumps({"what": "fused", "local_splits": f.plan.local_splits, "ms": ms,
                      "tflops": 2 * M * N * K / ms / 1e9, "relF_vs_unfused": rel}), flush=True)
