"""Tail split (stream-K style, in-kernel fix-up) vs unsplit on shapes whose
last wave is partial; interleaved, CUDA events, median of 20 after warm-up."""
import os
import statistics
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_2503_04771_b200 import executor  # noqa: E402
from paper_2503_04771_b200.api import contract  # noqa: E402

dev = torch.device("cuda", 0)
MM = "(i,k),(k,j)->(i,j)"
for (M, N, K) in [(4096, 4096, 4096), (4096, 4096, 8192), (4096, 4096, 16384), (6144, 6144, 6144),
                  (2048, 8192, 8192), (8192, 4096, 2048)]:
    a = torch.randn(M, K, device=dev).bfloat16()
    b = torch.randn(K, N, device=dev).bfloat16()
    out = torch.empty(M, N, device=dev, dtype=torch.bfloat16)
    ref = a.double() @ b.double()
    res = {}
    for rep in range(2):
        for sp in (0, -2, -3, -4):
            sc = {"splits": sp} if sp else {}
            for _ in range(3):
                contract(MM, a, b, out=out, schedule=sc or None)
            torch.cuda.synchronize()
            ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(20)]
            for s, e in ev:
                s.record()
                contract(MM, a, b, out=out, schedule=sc or None)
                e.record()
            torch.cuda.synchronize()
            ms = statistics.median(s.elapsed_time(e) for s, e in ev)
            err = float((out.double() - ref).norm() / ref.norm())
            executor.reset_launch_log()
            contract(MM, a, b, out=out, schedule=sc or None)
            res.setdefault(sp, []).append((round(2 * M * N * K / ms / 1e9), executor.launch_log()[-1], f"{err:.1e}"))
    print(f"{M}x{N}x{K}", {k: v for k, v in res.items()}, flush=True)
