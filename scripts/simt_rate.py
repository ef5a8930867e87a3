import os
import statistics
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_2503_04771_b200.api import contract  # noqa: E402

dev = torch.device("cuda", 0)
for n in (2048, 4096):
    a = torch.randn(n, n, device=dev)
    b = torch.randn(n, n, device=dev)
    for mode in ("ffma", "exact"):
        for _ in range(2):
            contract("(i,k),(k,j)->(i,j)", a, b, mode=mode)
        torch.cuda.synchronize()
        time.sleep(0.5)
        ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(5)]
        for s, e in ev:
            s.record(); contract("(i,k),(k,j)->(i,j)", a, b, mode=mode); e.record()
        torch.cuda.synchronize()
        ms = statistics.median(s.elapsed_time(e) for s, e in ev)
        print(f"{n}^3 f32 {mode}: {ms:.3f} ms {2*n**3/ms/1e9:.1f} TFLOP/s", flush=True)
