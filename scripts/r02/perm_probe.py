"""Permutations vs plain copies at the C2 sizes (device time, L2 flushed)."""
import statistics
import sys

import torch

sys.path.insert(0, ".")
from paper_2503_04771_b200 import contract  # noqa: E402

dev = torch.device("cuda", 0)
flush = torch.empty(256 << 20, dtype=torch.uint8, device=dev)


def t(fn, n=20):
    for _ in range(3):
        fn()
    ts = []
    for _ in range(n):
        flush.zero_()
        s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        s.record()
        fn()
        e.record()
        ts.append((s, e))
    torch.cuda.synchronize()
    return statistics.median(a.elapsed_time(b) for a, b in ts)


for shape, spec, perm in [((8192, 8192), "(i,j)->(j,i)", (1, 0)),
                          ((256, 512, 512), "(i,j,k)->(k,j,i)", (2, 1, 0))]:
    x = torch.randn(shape, device=dev)
    y = torch.empty(tuple(shape[p] for p in perm), device=dev)
    nbytes = 2 * x.numel() * 4
    ident = "(" + ",".join("ijk"[:len(shape)]) + ")->(" + ",".join("ijk"[:len(shape)]) + ")"
    z = torch.empty_like(x)
    for name, fn in [("bgx permute", lambda: contract(spec, x, out=y)),
                     ("bgx identity copy", lambda: contract(ident, x, out=z)),
                     ("torch copy_", lambda: z.copy_(x)),
                     ("torch permute copy", lambda: y.copy_(x.permute(*perm)))]:
        ms = t(fn)
        print(f"{spec:20s} {name:20s} {ms*1e3:8.1f} us {nbytes / ms / 1e6:8.1f} GB/s", flush=True)
