import statistics
import sys
import numpy as np
import torch
sys.path.insert(0, ".")
import oracle  # noqa: E402
from paper_2503_04771_b200 import contract  # noqa: E402
dev = torch.device("cuda", 0)
flush = torch.empty(256 << 20, dtype=torch.uint8, device=dev)
def t(fn):
    fn(); ts = []
    for _ in range(5):
        flush.zero_()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(); fn(); b.record(); ts.append((a, b))
    torch.cuda.synchronize()
    return statistics.median(x.elapsed_time(y) for x, y in ts) * 1e3
for dt in (torch.float32, torch.float64):
    for spec, shapes in [("(i,j)->(i)", [(8192, 8192)]), ("(i,j),(j)->(i)", [(8192, 8192), (8192,)]),
                         ("(i,j),(i,j)->(i)", [(8192, 8192), (8192, 8192)]), ("(b,k),(b,k)->(b)", [(8192, 8192), (8192, 8192)]),
                         ("(i,j)->(i)", [(4096, 8190)])]:
        xs = [torch.randn(s, device=dev, dtype=dt) for s in shapes]
        us = t(lambda: contract(spec, *xs))
        y = contract(spec, *xs).cpu().numpy()
        sp = spec.split("->")[0][1:-1].split("),(")
        want = oracle.generic([tuple(s.split(",")) for s in sp], tuple(spec.split("->")[1][1:-1].split(",")),
                              [x.cpu().numpy() for x in xs], np.zeros(y.shape, y.dtype))
        nb = sum(x.numel() * x.element_size() for x in xs)
        print(f"{str(dt):14s} {spec:20s} {str(shapes[0]):14s} {us:8.1f} us {nb/us/1e3:7.1f} GB/s bit-exact={np.array_equal(y, want)}", flush=True)
