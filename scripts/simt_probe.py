import os, sys, statistics
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2503_04771_b200 import contract
dev = torch.device("cuda", 0)
a = torch.randn(4096, 4096, device=dev); b = torch.randn(4096, 4096, device=dev)
for mode in ("ffma", "exact"):
    f = lambda: contract("(i,k),(k,j)->(i,j)", a, b, mode=mode)
    f(); torch.cuda.synchronize()
    ts = []
    for _ in range(3):
        e0 = torch.cuda.Event(enable_timing=True); e1 = torch.cuda.Event(enable_timing=True)
        e0.record(); f(); e1.record(); torch.cuda.synchronize(); ts.append(e0.elapsed_time(e1))
    ms = statistics.median(ts); print(mode, ms, 2 * 4096**3 / ms / 1e9, "TFLOP/s", flush=True)
