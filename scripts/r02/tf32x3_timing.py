"""f32 GEMM modes at 4096^3 / 8192^3: exact (bit-identical), FFMA, tf32x3
(split tf32, f32-level accuracy), tf32; device time and relF vs f64."""
import statistics
import sys

import torch

sys.path.insert(0, ".")
from paper_2503_04771_b200 import contract  # noqa: E402

dev = torch.device("cuda", 0)
for n in (4096, 8192):
    a = torch.randn(n, n, device=dev)
    b = torch.randn(n, n, device=dev)
    ref = a.double() @ b.double()
    for mode in ("exact", "ffma", "tf32x3", "tf32"):
        if n == 8192 and mode in ("exact", "ffma"):
            continue
        o = torch.empty(n, n, device=dev)
        for _ in range(2):
            contract("(i,k),(k,j)->(i,j)", a, b, out=o, mode=mode)
        torch.cuda.synchronize()
        ts = []
        for _ in range(5):
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            contract("(i,k),(k,j)->(i,j)", a, b, out=o, mode=mode)
            e1.record()
            torch.cuda.synchronize()
            ts.append(e0.elapsed_time(e1))
        ms = statistics.median(ts)
        err = ((o.double() - ref).norm() / ref.norm()).item()
        print(f"{n}^3 {mode:7s} {ms:8.3f} ms {2 * n**3 / ms / 1e9:7.1f} TFLOP/s  relF vs f64 {err:.2e}",
              flush=True)
