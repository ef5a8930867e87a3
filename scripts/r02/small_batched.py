"""Small batched GEMMs (many tiny matrices), bf16 and f32 exact: time and the
kernel class the planner picks."""
import statistics
import sys

import torch

sys.path.insert(0, ".")
from paper_2503_04771_b200 import contract, executor, plan  # noqa: E402
if len(sys.argv) > 1 and sys.argv[1] == "off":
    plan.SMALL_BATCHED_GEMM = False

dev = torch.device("cuda", 0)
for dt in (torch.bfloat16, torch.float32):
    for bt, m, n, k in [(4096, 64, 64, 64), (16384, 32, 32, 32), (16384, 16, 16, 16), (1024, 128, 128, 128),
                        (256, 256, 256, 64), (65536, 8, 8, 8), (2048, 16, 256, 64), (65536, 4, 4, 64)]:
        a = torch.randn(bt, m, k, device=dev).to(dt)
        b = torch.randn(bt, k, n, device=dev).to(dt)
        o = torch.empty(bt, m, n, device=dev, dtype=dt)
        f = lambda: contract("(b,i,k),(b,k,j)->(b,i,j)", a, b, out=o)  # noqa: E731
        for _ in range(3):
            f()
        torch.cuda.synchronize()
        executor.reset_launch_log()
        f()
        kinds = executor.launch_log()
        ts = []
        for _ in range(10):
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record(); f(); e1.record()
            torch.cuda.synchronize()
            ts.append(e0.elapsed_time(e1))
        ms = statistics.median(ts)
        flop = 2 * bt * m * n * k
        byts = (a.numel() + b.numel() + o.numel()) * a.element_size()
        print(f"{str(dt)[6:]:9s} {bt:6d} x {m}x{n}x{k}: {ms*1e3:8.1f} us  {flop/ms/1e9:7.1f} TFLOP/s  "
              f"{byts/ms/1e6:7.1f} GB/s  {kinds[0]}", flush=True)
