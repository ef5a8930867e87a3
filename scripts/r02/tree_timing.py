"""Exact (reference-order chain) vs tolerance-mode tree reductions: device
time and achieved HBM bandwidth (algorithmic bytes = inputs read once)."""
import statistics
import sys

import torch

sys.path.insert(0, ".")
from paper_2503_04771_b200 import contract  # noqa: E402

dev = torch.device("cuda", 0)
CASES = [("(i,j)->()", [(4096, 4096)]), ("(i,j)->()", [(16384, 16384)]),
         ("(i,j)->(i)", [(8192, 8192)]), ("(i,j)->(j)", [(8192, 8192)]),
         ("(i),(i)->()", [(1 << 26,), (1 << 26,)]), ("(i,j),(j)->(i)", [(8192, 8192), (8192,)])]
flush = torch.empty(256 << 20, dtype=torch.uint8, device=dev)
for spec, shapes in CASES:
    xs = [torch.randn(s, device=dev) for s in shapes]
    nbytes = sum(x.numel() * 4 for x in xs)
    row = [spec, "x".join(map(str, shapes[0]))]
    for mode in ("exact", "ffma"):
        fn = lambda: contract(spec, *xs, mode=mode)  # noqa: E731
        fn()
        ts = []
        for _ in range(3 if mode == "exact" else 10):
            flush.zero_()
            s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            s.record()
            fn()
            e.record()
            torch.cuda.synchronize()
            ts.append(s.elapsed_time(e))
        ms = statistics.median(ts)
        row.append(f"{mode} {ms:9.3f} ms {nbytes / ms / 1e6:8.1f} GB/s")
    print(" | ".join(row), flush=True)
