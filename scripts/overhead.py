"""Host overhead of the Python entry points for small, launch-bound contractions."""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_2503_04771_b200 as bgx  # noqa: E402

dev = torch.device("cuda", 0)
cases = [("(i,k),(k,j)->(i,j)", [(64, 64), (64, 64)], torch.bfloat16),
         ("(i,k),(k,j)->(i,j)", [(256, 256), (256, 256)], torch.float32),
         ("(i,j)->(j,i)", [(128, 128)], torch.float32),
         ("(b,i,j),(b,j,k)->(b,i,k)", [(8, 128, 64), (8, 64, 128)], torch.bfloat16)]
for spec, shapes, dt in cases:
    xs = [torch.randn(s, device=dev).to(dt) for s in shapes]
    out = bgx.contract(spec, *xs)
    for label, fn in [("contract", lambda: bgx.contract(spec, *xs, out=out))] + (
            [("prepared", bgx.prepare(spec, *xs, out=out))] if hasattr(bgx, "prepare") else []) + (
            [("graph", bgx.prepare(spec, *xs, out=out, graph=True))] if hasattr(bgx, "prepare") else []):
        for _ in range(10):
            fn()
        torch.cuda.synchronize()
        n = 200
        t0 = time.perf_counter()
        for _ in range(n):
            fn()
        torch.cuda.synchronize()
        us = (time.perf_counter() - t0) / n * 1e6
        print(f"{spec:28s} {str(shapes):30s} {label:9s}: {us:8.1f} us/call", flush=True)
