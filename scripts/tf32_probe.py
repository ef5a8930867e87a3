"""tf32 mode: N-major vs K-major B, tile variants; 1 s idle before each
measurement, median of 10; plus ncu-free tensor-time estimate."""
import os
import statistics
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_2503_04771_b200 import executor  # noqa: E402
from paper_2503_04771_b200.api import contract  # noqa: E402

dev = torch.device("cuda", 0)
for n in (4096, 8192):
    a = torch.randn(n, n, device=dev)
    b = torch.randn(n, n, device=dev)
    bt = b.t().contiguous()
    out = torch.empty(n, n, device=dev)
    cases = [("B N-major auto", "(i,k),(k,j)->(i,j)", b, None),
             ("B K-major auto", "(i,k),(j,k)->(i,j)", bt, None),
             ("B N-major 2x256", "(i,k),(k,j)->(i,j)", b, {"tile_n": 256, "cta_group": 2}),
             ("B K-major 2x256", "(i,k),(j,k)->(i,j)", bt, {"tile_n": 256, "cta_group": 2}),
             ("B K-major 2x512", "(i,k),(j,k)->(i,j)", bt, {"tile_n": 512, "cta_group": 2}),
             ("B N-major 2x512", "(i,k),(k,j)->(i,j)", b, {"tile_n": 512, "cta_group": 2})]
    for label, spec, bb, sc in cases:
        for _ in range(3):
            contract(spec, a, bb, out=out, mode="tf32", schedule=sc)
        torch.cuda.synchronize()
        time.sleep(1.0)
        ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(10)]
        for s, e in ev:
            s.record()
            contract(spec, a, bb, out=out, mode="tf32", schedule=sc)
            e.record()
        torch.cuda.synchronize()
        ms = statistics.median(s.elapsed_time(e) for s, e in ev)
        executor.reset_launch_log()
        contract(spec, a, bb, out=out, mode="tf32", schedule=sc)
        print(f"{n}^3 {label:18s} {ms:.3f} ms {2*n**3/ms/1e9:.0f} TFLOP/s {executor.launch_log()}", flush=True)
