"""Planner audit: many body kinds x dtypes at sizes where the answer should be
HBM- or tensor-bound; prints device time, GB/s (operands + output once),
TFLOP/s and the kernels launched, to catch pathological plans."""
import statistics
import sys

import torch

sys.path.insert(0, ".")
from paper_2503_04771_b200 import contract, executor  # noqa: E402
from paper_2503_04771_b200.einsum import parse_einsum  # noqa: E402

dev = torch.device("cuda", 0)
flush = torch.empty(256 << 20, dtype=torch.uint8, device=dev)
CASES = [
    ("(i),(j)->(i,j)", dict(i=8192, j=8192)),
    ("(b,k),(b,k)->(b)", dict(b=8192, k=8192)),
    ("(i,k),(k)->(i)", dict(i=16384, k=8192)),
    ("(k),(k,j)->(j)", dict(j=16384, k=8192)),
    ("(i),(i)->()", dict(i=1 << 26)),
    ("(i,j)->(i)", dict(i=8192, j=8192)),
    ("(i,j)->(j)", dict(i=8192, j=8192)),
    ("(i,j)->()", dict(i=8192, j=8192)),
    ("(i,j),(j,i)->(i,j)", dict(i=8192, j=8192)),
    ("(i,j,k),(k)->(i,j)", dict(i=256, j=256, k=1024)),
    ("(b,i,k),(b,k)->(b,i)", dict(b=64, i=1024, k=1024)),
    ("(i,k),(j,k)->(i,j)", dict(i=4096, j=4096, k=4096)),
    ("(k,i),(k,j)->(i,j)", dict(i=4096, j=4096, k=4096)),
    ("(i,j,k)->(j,k,i)", dict(i=256, j=512, k=512)),
    ("(i,k),(k,j),(j)->(i)", dict(i=4096, j=4096, k=4096)),
]
for text, ext in CASES:
    spec = parse_einsum(text)
    for dt in (torch.float32, torch.bfloat16):
        xs = [torch.randn([ext[a] for a in t], device=dev).to(dt) for t in spec.inputs]
        oshape = [ext[a] for a in spec.output]
        out = torch.empty(oshape, device=dev, dtype=dt)
        fn = lambda: contract(text, *xs, out=out)  # noqa: E731
        try:
            fn()
        except Exception as e:  # noqa: BLE001
            print(f"{text:26s} {str(dt):15s} ERROR {type(e).__name__}: {e}"[:200], flush=True)
            continue
        executor.reset_launch_log()
        fn()
        kern = sorted(set(executor.launch_log()))
        ts = []
        for _ in range(5):
            flush.zero_()
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a.record()
            fn()
            b.record()
            ts.append((a, b))
        torch.cuda.synchronize()
        ms = statistics.median(x.elapsed_time(y) for x, y in ts)
        nbytes = sum(x.numel() * x.element_size() for x in xs) + out.numel() * out.element_size()
        pts = 1
        for a in spec.axes:
            pts *= ext[a]
        print(f"{text:26s} {str(dt):15s} {ms*1e3:10.1f} us {nbytes/ms/1e6:8.1f} GB/s "
              f"{2*pts/ms/1e9:8.2f} TFLOP/s {kern}", flush=True)
