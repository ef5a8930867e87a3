"""Timing of the non-GEMM kernel classes (generic loop nest, permute) at
realistic sizes: CUDA events around the C-ABI-backed executor call."""
import os
import statistics
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_2503_04771_b200 import contract, executor  # noqa: E402

dev = torch.device("cuda", 0)
flush = torch.empty(256 << 20, dtype=torch.uint8, device=dev)


def t(fn, iters=5):
    for _ in range(2):
        fn()
    ts = []
    for _ in range(iters):
        flush.zero_()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        fn()
        e1.record()
        ts.append((e0, e1))
    torch.cuda.synchronize()
    return statistics.median(a.elapsed_time(b) for a, b in ts)


cases = [
    ("(i,j)->(i)", [(8192, 8192)]),
    ("(i,j),(i,j)->(i)", [(8192, 8192), (8192, 8192)]),
    ("(b,i,j)->(b,i)", [(64, 1024, 1024)]),
    ("(i,j),(j)->(i)", [(8192, 8192), (8192,)]),
    ("(i,j),(i)->(j)", [(8192, 8192), (8192,)]),
    ("(b,i,j)->(b,j)", [(64, 1024, 1024)]),
    ("(i,j)->(i) f64", [(8192, 8192)]),
    ("(i,j)->(j)", [(8192, 8192)]),
    ("(i,j)->()", [(4096, 4096)]),
    ("(i,j),(i,j)->()", [(2048, 2048), (2048, 2048)]),
    ("(i,j),(i,j)->(i,j)", [(8192, 8192), (8192, 8192)]),
    ("(i),(j)->(i,j)", [(8192,), (8192,)]),
    ("(b,i,j),(b,j)->(b,i)", [(64, 1024, 1024), (64, 1024)]),
    ("(i,j),(j,k),(k,l)->(i,l)", [(512, 512), (512, 512), (512, 512)]),
]
for spec, shapes in cases:
    dt = torch.float64 if spec.endswith(" f64") else torch.float32
    spec = spec.replace(" f64", "")
    xs = [torch.randn(s, device=dev, dtype=dt) for s in shapes]
    executor.reset_launch_log()
    fn = lambda: contract(spec, *xs)  # noqa: E731
    ms = t(fn)
    nbytes = sum(x.numel() * x.element_size() for x in xs)
    out = contract(spec, *xs)
    nbytes += out.numel() * out.element_size()
    print(f"{spec:28s} {str(shapes):40s} {ms:9.3f} ms  {nbytes / ms / 1e6:8.1f} GB/s  "
          f"kernels={executor.launch_log()[:3]}", flush=True)
