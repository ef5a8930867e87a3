"""f32 exact / FFMA GEMM timing (large sizes, cp.async kernel): device time per
launch, back-to-back after warm-up; run once per BGX_SIMT_BK setting."""
import os
import statistics
import sys

import torch

sys.path.insert(0, ".")
from paper_2503_04771_b200 import contract  # noqa: E402

dev = torch.device("cuda", 0)
for n, mode in [(4096, "exact"), (4096, "ffma"), (2048, "exact"), (8192, "exact")]:
    a = torch.randn(n, n, device=dev)
    b = torch.randn(n, n, device=dev)
    o = torch.empty(n, n, device=dev)
    for _ in range(3):
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
    ref = (a.double() @ b.double())
    err = ((o.double() - ref).norm() / ref.norm()).item()
    print(f"BK={os.environ.get('BGX_SIMT_BK', '16')} {n}^3 {mode:5s} {ms:8.3f} ms "
          f"{2 * n**3 / ms / 1e9:6.2f} TFLOP/s relF vs f64 {err:.2e} checksum {o.double().sum().item():.6e}",
          flush=True)
