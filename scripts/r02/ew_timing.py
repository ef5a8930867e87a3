"""Dense elementwise bodies (exact mode): device time and HBM GB/s."""
import statistics
import sys

import torch

sys.path.insert(0, ".")
from paper_2503_04771_b200 import contract, executor  # noqa: E402

dev = torch.device("cuda", 0)
flush = torch.empty(256 << 20, dtype=torch.uint8, device=dev)
for spec, n_in, dt in [("(i,j),(i,j)->(i,j)", 2, torch.float32), ("(i,j),(i,j),(i,j)->(i,j)", 3, torch.float32),
                       ("(i,j),(i,j)->(i,j)", 2, torch.bfloat16), ("(i,j),(i,j)->(i,j)", 2, torch.float64)]:
    xs = [torch.randn(8192, 8192, device=dev).to(dt) for _ in range(n_in)]
    out = torch.empty(8192, 8192, device=dev, dtype=dt)
    fn = lambda: contract(spec, *xs, out=out)  # noqa: E731
    fn()
    executor.reset_launch_log()
    fn()
    kern = executor.launch_log()
    ts = []
    for _ in range(10):
        flush.zero_()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        fn()
        b.record()
        ts.append((a, b))
    torch.cuda.synchronize()
    ms = statistics.median(x.elapsed_time(y) for x, y in ts)
    nbytes = (n_in + 1) * out.numel() * out.element_size()
    ok = torch.equal(out, (xs[0] * xs[1] * (xs[2] if n_in == 3 else 1)).to(dt)) if dt != torch.bfloat16 else None
    print(f"{spec:28s} {str(dt):15s} {ms*1e3:8.1f} us {nbytes/ms/1e6:8.1f} GB/s {kern} torch-equal={ok}", flush=True)
