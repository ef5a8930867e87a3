"""f32 SIMT GEMM timing (median of 7 per shape and mode).  Run it twice —
plain (cp.async-staged kernel for row-major operands) and with
BGX_NO_SIMT_CP=1 (register-staged kernel; the library reads the variable
once per process) — to A/B the two kernels; the printed checksums must match
bit for bit."""
import os
import statistics
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_2503_04771_b200.api import contract  # noqa: E402

dev = torch.device("cuda", 0)
MM = "(i,k),(k,j)->(i,j)"
impl = "reg" if os.environ.get("BGX_NO_SIMT_CP") else "cp"
g = torch.Generator(device=dev).manual_seed(0)
for (m, n, k) in ((2048, 2048, 2048), (4096, 4096, 4096), (1000, 1000, 1000), (8192, 8192, 2048)):
    a = torch.randn(m, k, device=dev, generator=g)
    b = torch.randn(k, n, device=dev, generator=g)
    for mode in ("ffma", "exact"):
        for _ in range(2):
            o = contract(MM, a, b, mode=mode)
        torch.cuda.synchronize()
        time.sleep(0.3)
        ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True))
              for _ in range(7)]
        for s, e in ev:
            s.record(); contract(MM, a, b, mode=mode); e.record()
        torch.cuda.synchronize()
        ms = statistics.median(s.elapsed_time(e) for s, e in ev)
        bits = int(o.view(torch.int32).sum(dtype=torch.int64))
        print(f"{impl} {m}x{n}x{k} {mode}: {ms:.3f} ms {2*m*n*k/ms/1e9:.1f} TFLOP/s "
              f"bitsum {bits}", flush=True)
