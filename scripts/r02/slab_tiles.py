"""Tile choice for the per-rank slabs of the strong-scaled chain GEMM (rows x 8192 x 8192),
through contract() (split-K / tail-split planning included), burst timing."""
import statistics
import sys
import time
import torch
sys.path.insert(0, ".")
from paper_2503_04771_b200 import contract, executor  # noqa: E402
dev = torch.device("cuda", 0)
flush = torch.empty(256 << 20, dtype=torch.uint8, device=dev)
B = torch.randn(8192, 8192, device=dev).bfloat16()
for rows in (2048, 4096, 6144, 8192, 12288, 16384):
    A = torch.randn(rows, 8192, device=dev).bfloat16()
    O = torch.empty(rows, 8192, device=dev, dtype=torch.bfloat16)
    for name, sch in [("auto", None), ("t512", {"tile_n": 512, "cta_group": 2}),
                      ("t512 nosplit", {"tile_n": 512, "cta_group": 2, "no_splitk": 1}),
                      ("t256", {"tile_n": 256, "cta_group": 2}),
                      ("t256 nosplit", {"tile_n": 256, "cta_group": 2, "no_splitk": 1})]:
        fn = lambda: contract("(i,k),(k,j)->(i,j)", A, B, out=O, schedule=sch)  # noqa: E731
        executor.reset_launch_log()
        fn()
        kern = executor.launch_log()
        torch.cuda.synchronize()
        time.sleep(0.3)
        ts = []
        for _ in range(10):
            flush.zero_()
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a.record(); fn(); b.record(); ts.append((a, b))
        torch.cuda.synchronize()
        us = statistics.median(x.elapsed_time(y) for x, y in ts) * 1e3
        print(f"rows {rows:6d} {name:14s} {us:8.1f} us {2*rows*8192*8192/us/1e6:8.1f} TFLOP/s {kern} {executor.tile_log()[-1:] }", flush=True)
